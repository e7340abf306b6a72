"""Where the consumer groups of the decode-pass kernel spend their time.

Builds the pass of tools/pass_probe.py (independent inputs), launches it once
with %globaltimer stamps (nqb_debug_pass_trace) and prints, per step kind, the
median over CTAs and steps (us) of each group's phases:
  stage-1 group: wait (x slot / previous step), quantise x, MMA, publish t
  stage-2 group: wait (t barrier + t copy), quantise t, MMA, outputs
plus each group's busy fraction over the pass span.

  python tools/pass_busy.py [--model 70b] [--blocks 8]
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
    ap.add_argument("--model", default="70b")
    ap.add_argument("--blocks", type=int, default=8)
    args = ap.parse_args()
    import torch

    import paper_2602_06694_b200 as nq
    ctx = nq.context(0)
    bpw, _, shapes = PP.SHAPES[args.model]
    rng = np.random.default_rng(5)
    ranks = {nm: nq.rank_for_target_bpw(n, m, bpw) for nm, n, m in shapes}
    steps, keep = [], []
    f16 = torch.float16
    for _ in range(args.blocks):
        lay = {nm: nq.DeviceLayer.upload_f16(n, m, ranks[nm], *PP.rand_arrays(rng, n, m, ranks[nm]),
                                             ctx) for nm, n, m in shapes}
        qkv = nq.DecodeGroup([lay["q"], lay["k"], lay["v"]])
        gu = nq.DecodeGroup([lay["gate"], lay["up"]])
        keep += [lay, qkv, gu]
        d, f = lay["q"].m, lay["gate"].n
        new = lambda n: torch.empty(n, device="cuda", dtype=f16)  # noqa: E731
        ys = [[new(lay["q"].n), new(lay["k"].n), new(lay["v"].n)], [new(d)], [new(f), new(f)], [new(d)]]
        xs = [torch.randn(d, device="cuda", dtype=f16) for _ in range(3)] + \
             [torch.randn(f, device="cuda", dtype=f16)]
        for u, x, y in zip([qkv, lay["o"], gu, lay["down"]], xs, ys):
            steps.append((u, x, y))
    p = nq.DecodePass(steps, ctx)
    for _ in range(3):
        p.launch()
    torch.cuda.synchronize()
    tr = p.trace().astype(np.int64)
    G, K = tr.shape[0], len(steps)
    t0 = tr[:, 0].min()
    raw = tr[:, 1:1 + 24 * K].reshape(G, K, 24).astype(float)
    # SM partitions: a CTA stamps only the steps of its own partition
    raw[raw[:, :, 0] == 0] = np.nan
    st = (raw - t0) / 1e3
    span = (tr[:, 24 * K + 1].max() - t0) / 1e3
    kinds = ["qkv", "o", "gateup", "down"]
    out = {"model": args.model, "blocks": args.blocks, "span_us": span,
           "gbs_traced": p.algorithmic_bytes / span / 1e3}
    def prev_end(col):  # the end of the CTA's previous step (its own partition's list)
        out = np.full((G, K), np.nan)
        for c in range(G):
            last = 0.0
            for k in range(K):
                if not np.isnan(st[c, k, col]):
                    out[c, k] = last
                    last = st[c, k, col]
        return out
    s1_prev_end = prev_end(1)
    s2_prev_end = prev_end(3)
    ph = {
        "s1_wait": st[:, :, 0] - s1_prev_end, "s1_quant": st[:, :, 7] - st[:, :, 0],
        "s1_mma": st[:, :, 8] - st[:, :, 7], "s1_pub": st[:, :, 1] - st[:, :, 8],
        "s2_wait": st[:, :, 2] - s2_prev_end, "s2_quant": st[:, :, 9] - st[:, :, 2],
        "s2_mma": st[:, :, 10] - st[:, :, 9], "s2_out": st[:, :, 3] - st[:, :, 10],
        "tbar_after_s1end_max": st[:, :, 4] - st[:, :, 1].max(axis=0, keepdims=True),
        "s1_chunk_wait": raw[:, :, 16] / 1965.0, "s2_chunk_wait": raw[:, :, 17] / 1965.0,
        "s1_chunks": np.floor(raw[:, :, 18] / 2.0 ** 48), "s2_chunks": np.floor(raw[:, :, 19] / 2.0 ** 48),
        "s1_calls": np.floor(raw[:, :, 18] / 2.0 ** 32) % 65536,
        "s2_calls": np.floor(raw[:, :, 19] / 2.0 ** 32) % 65536,
        "s1_slabs": np.floor(raw[:, :, 18] / 2.0 ** 16) % 65536,
        "s2_slabs": np.floor(raw[:, :, 19] / 2.0 ** 16) % 65536,
        "s1_runpair_us": raw[:, :, 20] / 1965.0, "s2_runpair_us": raw[:, :, 21] / 1965.0,
        "s1_loop_us": raw[:, :, 22] / 1965.0, "s2_loop_us": raw[:, :, 23] / 1965.0,
    }
    for i, kd in enumerate(kinds):
        sel = [k for k in range(K) if k % 4 == i and k >= 4]
        out[kd] = {nm: round(float(np.nanmedian(v[:, sel])), 3) for nm, v in ph.items()}
        out[kd]["s1end_spread"] = round(float(np.nanmedian(np.nanmax(st[:, sel, 1], 0) -
                                                           np.nanmin(st[:, sel, 1], 0))), 3)
    busy1 = np.nansum(ph["s1_quant"] + ph["s1_mma"] + ph["s1_pub"], 1) / span
    busy2 = np.nansum(ph["s2_quant"] + ph["s2_mma"] + ph["s2_out"], 1) / span
    mma1 = np.nansum(ph["s1_mma"], 1) / span
    mma2 = np.nansum(ph["s2_mma"], 1) / span
    out["busy"] = {"s1": float(np.median(busy1)), "s2": float(np.median(busy2)),
                   "s1_mma": float(np.median(mma1)), "s2_mma": float(np.median(mma2))}
    out["cta_end_us"] = {"min": float((tr[:, 24 * K + 1].min() - t0) / 1e3), "max": span}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
