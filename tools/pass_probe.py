"""Times a whole decode pass two ways on one GPU and prints one JSON line per model:
  graph: 4 launches per block (qkv group, o, gate/up group, down) of the per-call
         kernel k_decode captured in one CUDA graph (round-1 bench step);
  pass:  the same steps as ONE launch of the persistent k_decode_pass.
Models: llama2-7b @0.8 (32 blocks) and llama2-70b @0.55 (80 blocks, GQA k/v 1024 rows).
Inputs are independent per step (x per launch, like bench.py) unless --chained.

  python tools/pass_probe.py [--models 7b,70b] [--reps 20] [--chained]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {
    "7b": (0.8, 32, [("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
                     ("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]),
    "70b": (0.55, 80, [("q", 8192, 8192), ("k", 1024, 8192), ("v", 1024, 8192), ("o", 8192, 8192),
                       ("gate", 28672, 8192), ("up", 28672, 8192), ("down", 8192, 28672)]),
}


def algo(n, m, r):
    return r * (n + m) / 8.0 + 2 * (n + m) + 2 * m + 2 * n


def rand_arrays(rng, n, m, r):
    k = (r + 31) // 32
    u = rng.integers(0, 2 ** 32, size=(n, k), dtype=np.uint32)
    v = rng.integers(0, 2 ** 32, size=(m, k), dtype=np.uint32)
    if r % 32:
        mask = np.uint32((1 << (r % 32)) - 1)
        u[:, -1] &= mask
        v[:, -1] &= mask
    s1 = rng.uniform(0.25, 2.0, n).astype(np.float16).view(np.uint16)
    s2 = rng.uniform(0.25, 2.0, m).astype(np.float16).view(np.uint16)
    return u, v, s1, s2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="7b,70b")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--blocks", type=int, default=0, help="override block count")
    ap.add_argument("--chained", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--sms", type=int, default=0, help="SM budget of the context (plans and pass grid)")
    args = ap.parse_args()
    import torch

    import paper_2602_06694_b200 as nq
    ctx = nq.context(0)
    if args.sms:
        ctx.set_sm_budget(args.sms)
    stream = torch.cuda.Stream()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6538.6
    for model in args.models.split(","):
        bpw, blocks, shapes = SHAPES[model]
        blocks = args.blocks or blocks
        rng = np.random.default_rng(99)
        ranks = {nm: nq.rank_for_target_bpw(n, m, bpw) for nm, n, m in shapes}
        steps, keep, nbytes = [], [], 0.0
        f16 = torch.float16
        prev = None
        for b in range(blocks):
            lay = {nm: nq.DeviceLayer.upload_f16(n, m, ranks[nm], *rand_arrays(rng, n, m, ranks[nm]),
                                                 ctx) for nm, n, m in shapes}
            keep.append(lay)
            qkv = nq.DecodeGroup([lay["q"], lay["k"], lay["v"]])
            gu = nq.DecodeGroup([lay["gate"], lay["up"]])
            keep += [qkv, gu]
            d, f = lay["q"].m, lay["gate"].n
            new = lambda n: torch.empty(n, device="cuda", dtype=f16)  # noqa: E731
            ys = [[new(lay["q"].n), new(lay["k"].n), new(lay["v"].n)], [new(d)],
                  [new(f), new(f)], [new(d)]]
            if args.chained:
                x0 = prev if prev is not None else torch.randn(d, device="cuda", dtype=f16)
                xs = [x0, ys[0][0], ys[1][0], ys[2][0]]
            else:
                xs = [torch.randn(d, device="cuda", dtype=f16), torch.randn(d, device="cuda", dtype=f16),
                      torch.randn(d, device="cuda", dtype=f16), torch.randn(f, device="cuda", dtype=f16)]
            prev = ys[3][0]
            units = [qkv, lay["o"], gu, lay["down"]]
            for u, x, y in zip(units, xs, ys):
                steps.append((u, x, y))
                ls = u.layers if isinstance(u, nq.DecodeGroup) else [u]
                nbytes += sum(algo(l.n, l.m, l.r) for l in ls) - 2 * ls[0].m * (len(ls) - 1)
        out = {"model": model, "sms": args.sms, "blocks": blocks, "bpw": bpw, "ranks": ranks,
               "algo_bytes_per_pass": nbytes, "chained": args.chained}

        def timeit(fn, reps):
            with torch.cuda.stream(stream):
                ctx.bind_torch_stream()
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(reps):
                    fn()
                e1.record(stream)
                torch.cuda.synchronize()
            return e0.elapsed_time(e1) / 1e3 / reps

        if not args.no_graph:
            def step():
                for u, x, y in steps:
                    if isinstance(u, nq.DecodeGroup):
                        u.gemv_device(x, y)
                    else:
                        u.gemv_device(x, y[0])
            with torch.cuda.stream(stream):
                ctx.bind_torch_stream()
                step()
                with ctx.capture() as cap:
                    step()
            g = cap.graph
            s = timeit(g.launch, args.reps)
            out["graph"] = {"us": s * 1e6, "gbs": nbytes / s / 1e9, "frac": nbytes / s / 1e9 / peak}
            g.free()
        p = nq.DecodePass(steps, ctx)
        out["pass_stream_bytes"] = p.stream_bytes
        s = timeit(p.launch, args.reps)
        out["pass"] = {"us": s * 1e6, "gbs": nbytes / s / 1e9, "frac": nbytes / s / 1e9 / peak}
        # bitwise: pass == graph on the same inputs (independent steps only)
        if not args.chained and not args.no_graph:
            with torch.cuda.stream(stream):
                ctx.bind_torch_stream()
                p.launch()
                torch.cuda.synchronize()
                a = [[y.clone() for y in ys] for _, _, ys in steps]
                step()
                torch.cuda.synchronize()
                out["pass_equals_per_call"] = all(torch.equal(y, w) for (_, _, ys), ws in zip(steps, a)
                                                  for y, w in zip(ys, ws))
        print(json.dumps(out), flush=True)
        p.free()
        del steps, keep
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
