"""Builds the bench's decode pass (bench.workload: 224 Llama-2-7B layers @0.8 bit, or
the 70B pass with --model 70b) and launches it `--launches` times, for ncu:

  ncu --set full -k regex:k_decode_pass -s 2 -c 1 -o out python tools/prof_pass.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--launches", type=int, default=4)
    args = ap.parse_args()
    import torch

    import paper_2602_06694_b200 as nq
    ctx = nq.context(0)
    if args.model == "7b":
        steps = bench.workload(nq.rank_for_target_bpw)
    else:
        steps = bench.workload(nq.rank_for_target_bpw, bench.L70_BLOCK, 80, 0.55, seed=bench.SEED + 70)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        ctx.bind_torch_stream()
        p, ps, keep = bench.build_pass(nq, ctx, torch, steps)
        for _ in range(args.launches):
            p.launch()
        torch.cuda.synchronize()
    print("algorithmic_bytes", bench.step_bytes_of(steps), "stream_bytes", p.stream_bytes, flush=True)


if __name__ == "__main__":
    main()
