"""e2e of the bench's 7B decode pass through bound host buffers (nqb_pass_io_run),
with outputs copied back by a copy kernel (NQB_PASS_IO_DIRECT_Y=0) or written by
the pass straight into mapped host memory (=1); checks both against the device
pass bit for bit.

  python tools/e2e_io_probe.py [--reps 20]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch

    import paper_2602_06694_b200 as nq
    ctx = nq.context(0)
    steps = bench.workload(nq.rank_for_target_bpw)
    nbytes = bench.step_bytes_of(steps)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        ctx.bind_torch_stream()
        p, ps, keep = bench.build_pass(nq, ctx, torch, steps)
        p.launch()
        torch.cuda.synchronize()
    want = [y.cpu().numpy().copy() for _, _, ys in ps for y in ys]
    hx = [torch.from_numpy(x).pin_memory().numpy() for _, _, x in steps]
    hy = [torch.empty(w.shape, dtype=torch.float16).pin_memory().numpy() for w in want]
    for a in hx + hy:
        ctx.register_host(a)
    out = {}
    for mode in ("0", "1", "0", "1"):
        os.environ["NQB_PASS_IO_DIRECT_Y"] = mode
        io = p.host_io(hx, hy)
        for a in hy:
            a[...] = 0
        io.run()
        ok = all(np.array_equal(a.view(np.uint16), b.view(np.uint16)) for a, b in zip(hy, want))
        t0 = time.perf_counter()
        for _ in range(args.reps):
            io.run()
        sec = (time.perf_counter() - t0) / args.reps
        io.close()
        out.setdefault(mode, []).append((round(nbytes / sec / 1e9, 1), ok))
    print({"e2e_gbs_by_direct_y": out})


if __name__ == "__main__":
    main()
