"""Per-step timeline of one SM partition of the decode pass (trace stamps).

Builds the pass of tools/pass_busy.py (independent inputs), launches it once
with %globaltimer stamps and prints, for the steps of partition 0 in its list
order, the median over the partition's CTAs (us from kernel start) of:
  xq  x quantiser done        s1a/s1m/s1e  stage-1 start / MMA end / end
  tp  t barrier passed        tq  t quantiser done
  s2a/s2m/s2e stage-2 start / MMA end / end
  p1a/p1e p2a/p2e  producer 1 / 2 start and end of the step's copies

  NQB_PASS_SPLIT=4 python tools/pass_chain.py [--model 7b] [--blocks 16]
"""
import argparse
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
    ap.add_argument("--blocks", type=int, default=16)
    ap.add_argument("--steps", type=int, default=24)
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
    raw[raw == 0] = np.nan
    st = (raw - t0) / 1e3
    # partition 0: the CTAs that stamped the first step they share with CTA 0
    mine = [k for k in range(K) if not np.isnan(st[0, k, 0])]
    ctas = [c for c in range(G) if not np.isnan(st[c, mine[0], 0])]
    cols = [("xq", 5), ("s1a", 0), ("s1m", 8), ("s1e", 1), ("tp", 4), ("tq", 13), ("s2a", 2),
            ("s2m", 10), ("s2e", 3), ("p1a", 11), ("p1e", 6), ("p2a", 14), ("p2e", 15)]
    kinds = ["qkv", "o", "gu", "down"]
    print(f"partition of CTA 0: {len(ctas)} CTAs, {len(mine)} steps; span "
          f"{(tr[:, 24 * K + 1].max() - t0) / 1e3:.1f} us")
    print("step kind " + " ".join(f"{n:>7}" for n, _ in cols) + "   s1e_spread")
    for k in mine[:args.steps]:
        med = [np.nanmedian(st[ctas, k, i]) for _, i in cols]
        spread = np.nanmax(st[ctas, k, 1]) - np.nanmin(st[ctas, k, 1])
        print(f"{k:4d} {kinds[k % 4]:>4} " + " ".join(f"{v:7.1f}" for v in med) + f"   {spread:6.1f}")


if __name__ == "__main__":
    main()
