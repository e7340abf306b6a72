"""Builds profiles/<dir>/traffic.json from an ncu launch list of the bench step.

usage: python tools/traffic_from_ncu.py launches_decode.csv out.json
The CSV is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
-k regex:k_decode -c 128 --csv` of `bench.py --steps 1 --warmup 0 --no-shapes`: the step's 128
launches in bench order (per block: qkv group, o, gate/up group, down)."""
import csv
import json
import sys
from collections import defaultdict

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from bench import BPW, L7_BLOCK, algo_bytes, rank_for  # noqa: E402

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
iid, iname, ival = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = defaultdict(dict)
for r in data:
    per[int(r[iid])][r[iname]] = float(r[ival].replace(",", ""))
ids = sorted(per)[:128]
shape = {name: (n, m, rank_for(n, m, BPW)) for name, n, m in L7_BLOCK}
kinds = [("qkv", ["q", "k", "v"]), ("o", ["o"]), ("gateup", ["gate", "up"]), ("down", ["down"])]
out, tot_dram, tot_alg = {}, 0.0, 0.0
for k, (kind, names) in enumerate(kinds):
    sel = [per[i] for j, i in enumerate(ids) if j % 4 == k]
    alg = sum(algo_bytes(*shape[nm]) for nm in names)
    dram = sum(s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"] for s in sel) / len(sel)
    us = sum(s["gpu__time_duration.sum"] for s in sel) / len(sel) / 1e3
    out[kind] = {"launches": len(sel), "ncu_us_avg": round(us, 3), "dram_bytes_avg": dram,
                 "algorithmic_bytes": alg}
    tot_dram += dram * len(sel)
    tot_alg += alg * len(sel)
out["step"] = {"launches": len(ids), "dram_bytes_per_launch": tot_dram / len(ids),
               "algorithmic_bytes_per_launch": tot_alg / len(ids),
               "traffic_over_algorithmic": tot_dram / tot_alg}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out["step"]))
