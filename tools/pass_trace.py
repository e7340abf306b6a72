"""Per-step phase times of the persistent decode-pass kernel (nqb_debug_pass_trace).

Builds the 7B (or 70B) pass of tools/pass_probe.py and launches it once with
%globaltimer stamps; prints, per step kind, the median over CTAs and steps of each
stamped interval (µs), and the whole-pass span.

  python tools/pass_trace.py [--model 7b] [--blocks 8] [--chained]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import pass_probe as PP  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--chained", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2602_06694_b200 as nq
    ctx = nq.context(0)
    bpw, _, shapes = PP.SHAPES[args.model]
    rng = np.random.default_rng(5)
    ranks = {nm: nq.rank_for_target_bpw(n, m, bpw) for nm, n, m in shapes}
    steps, keep = [], []
    f16 = torch.float16
    prev = None
    for b in range(args.blocks):
        lay = {nm: nq.DeviceLayer.upload_f16(n, m, ranks[nm], *PP.rand_arrays(rng, n, m, ranks[nm]),
                                             ctx) for nm, n, m in shapes}
        qkv = nq.DecodeGroup([lay["q"], lay["k"], lay["v"]])
        gu = nq.DecodeGroup([lay["gate"], lay["up"]])
        keep += [lay, qkv, gu]
        d, f = lay["q"].m, lay["gate"].n
        new = lambda n: torch.empty(n, device="cuda", dtype=f16)  # noqa: E731
        ys = [[new(lay["q"].n), new(lay["k"].n), new(lay["v"].n)], [new(d)], [new(f), new(f)], [new(d)]]
        if args.chained:
            x0 = prev if prev is not None else torch.randn(d, device="cuda", dtype=f16)
            xs = [x0, ys[0][0], ys[1][0], ys[2][0]]
        else:
            xs = [torch.randn(d, device="cuda", dtype=f16) for _ in range(3)] + \
                 [torch.randn(f, device="cuda", dtype=f16)]
        prev = ys[3][0]
        for u, x, y in zip([qkv, lay["o"], gu, lay["down"]], xs, ys):
            steps.append((u, x, y))
    p = nq.DecodePass(steps, ctx)
    for _ in range(3):
        p.launch()
    torch.cuda.synchronize()
    tr = p.trace().astype(np.int64)  # (G, 6K + 2) %globaltimer stamps
    G, S = tr.shape
    K = len(steps)
    t0 = tr[:, 0].min()
    rel = (tr - t0) / 1e3
    st = rel[:, 1:1 + 14 * K].reshape(G, K, 14)  # s1 start, s1 end, s2 ready, s2 end, tbar seen, x staged
    out = {"model": args.model, "blocks": args.blocks, "chained": args.chained, "grid": int(G),
           "span_us": float(rel[:, -1].max()), "us_per_step": float(rel[:, -1].max() / K)}
    med = lambda a: round(float(np.median(a)), 3)  # noqa: E731
    kinds = ["qkv", "o", "gateup", "down"]
    prev_end = np.concatenate([np.zeros((G, 1)), st[:, :-1, 3]], axis=1)
    # end of the consumer phase that precedes stage 2 of k (latest S1 end or S2(k-1) end)
    s1end_sorted = st[:, :, 1]
    prev_end2 = np.maximum(prev_end, np.stack([s1end_sorted[:, :min(K, k + 3)].max(axis=1)
                                                for k in range(K)], axis=1))
    for j, kind in enumerate(kinds):
        sl = slice(j, K, 4)
        out[kind] = {
            "s1_us": med(st[:, sl, 1] - st[:, sl, 0]),
            "s2_wait_us": med(st[:, sl, 2] - np.maximum(st[:, sl, 1], prev_end[:, sl])),
            "s2_us": med(st[:, sl, 3] - st[:, sl, 2]),
            "period_us": med(st[:, sl, 3] - prev_end[:, sl]),
            "tbar_seen_minus_s1end_us": med(st[:, sl, 4] - st[:, sl, 1]),
            "x_staged_lead_us": med(st[:, sl, 0] - st[:, sl, 5]),
            "s1_chunk_wait_us": med(st[:, sl, 6] - st[:, sl, 0]),
            "s1_quant_us": med(st[:, sl, 7] - st[:, sl, 6]),
            "s1_mma_us": med(st[:, sl, 8] - st[:, sl, 7]),
            "s1_publish_us": med(st[:, sl, 1] - st[:, sl, 8]),
            "s2_quant_us": med(st[:, sl, 9] - st[:, sl, 2]),
            "s2_mma_us": med(st[:, sl, 10] - st[:, sl, 9]),
            "s2_out_us": med(st[:, sl, 3] - st[:, sl, 10]),
            "producer_issue_lead_us": med(st[:, sl, 0] - st[:, sl, 11]),
            "s2_start_gap_us": med(st[:, sl, 2] - prev_end2[:, sl]),
            "tslot_free_to_tbar_us": med(st[:, sl, 4] - st[:, sl, 12]),
            "tbar_to_tcopy_us": med(st[:, sl, 13] - st[:, sl, 4]),
            "tcopy_to_ready_us": med(st[:, sl, 2] - st[:, sl, 13]),
            "tslot_free_minus_prev_s2end_us": med(st[:, sl, 12] - prev_end[:, sl]),
        }
    out["first_s1_start_us"] = med(st[:, 0, 0])
    out["last_s2_end_us"] = med(st[:, -1, 3])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
