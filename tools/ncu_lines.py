"""Per-source-line hot spots of one kernel in an ncu report captured with
--import-source on and -lineinfo: warp-stall samples and instructions executed
aggregated by (file, line), top N by samples.

  python tools/ncu_lines.py REPORT.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = {}
    fname, line, src = "?", "?", ""
    hdr = None
    tot_s = tot_i = 0
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < 8:
            continue
        if row[0]:  # a source line row (its metrics are the sum over its SASS)
            line, src = row[0], row[1]
            try:
                s, i = int(row[4]), int(row[7])
            except ValueError:
                continue
            key = (fname, int(line))
            a = agg.setdefault(key, [0, 0, src.strip()[:70]])
            a[0] += s
            a[1] += i
            tot_s += s
            tot_i += i
    print(f"total samples {tot_s}  instructions {tot_i}")
    for (f, ln), (s, i, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * s / max(tot_s, 1):5.1f}% smp {100 * i / max(tot_i, 1):5.1f}% ins  {f}:{ln:<5d} {t}")


if __name__ == "__main__":
    main()
