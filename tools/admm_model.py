"""Whole-model (or partial-model) ADMM initialisation, layer-sharded over the
ranks of a torchrun job (one GPU per rank, NCCL gather of packed factors).

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      tools/admm_model.py [--blocks 32] [--bpw 1.0] [--workers 2] [--shape 1024,1024 --count 8]

Prints one JSON line on rank 0: matrices, wall seconds (max over ranks),
matrices/s, per-rank seconds, mean rel_error / iterations.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=32)
    ap.add_argument("--first-block", type=int, default=0, help="run blocks first .. first+blocks-1")
    ap.add_argument("--bpw", type=float, default=1.0)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--shape", default=None, help="n,m: uniform synthetic matrices instead of Llama-2-7B")
    ap.add_argument("--count", type=int, default=8)
    ap.add_argument("--repro", action="store_true",
                    help="re-run the first matrix and check the packed factors are bitwise equal")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2602_06694_b200 import sharded as S
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.shape:
        n, m = map(int, args.shape.split(","))
        specs = [S.MatrixSpec(f"w{i}", n, m, 0xA000 + i) for i in range(args.count)]
    else:
        specs = S.llama2_7b_specs(args.first_block + args.blocks)[7 * args.first_block:]
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    rep = S.sharded_init(specs, args.bpw, device=dev, workers=args.workers)
    wall = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([wall], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    if rep is not None:
        errs = [p.rel_error for p in rep.matrices.values()]
        its = [p.iterations for p in rep.matrices.values()]
        print(json.dumps({"matrices": len(rep.matrices), "gpus": ws, "workers_per_gpu": args.workers,
                          "bpw": args.bpw, "wall_s": wall, "matrices_per_s": len(rep.matrices) / wall,
                          "per_rank_compute_s": rep.per_rank_seconds,
                          "mean_rel_error": sum(errs) / len(errs),
                          "mean_admm_iterations": sum(its) / len(its),
                          "shapes": sorted({(p.n, p.m, p.r) for p in rep.matrices.values()}),
                          "weights": "W = fp32(0.02 g), g from the reference Rng(0x7B000000 + 7b + p)",
                          "per_matrix": [{"name": specs[i].name, "n": p.n, "m": p.m, "r": p.r,
                                          "seconds": p.seconds, "svd_init_s": p.seconds_svd,
                                          "iterations_s": p.seconds_iter,
                                          "svd_power_iterations": p.svd_power_iters,
                                          "admm_iterations": p.iterations,
                                          "converged": p.converged, "rel_error": p.rel_error}
                                         for i, p in sorted(rep.matrices.items())]}),
              flush=True)
        if args.repro:  # GPU-vs-GPU bitwise reproducibility at full size (SURVEY §8(d) protocol)
            i0 = min(rep.matrices)
            again = S.device_factorize(specs[i0], i0, args.bpw)
            first = rep.matrices[i0]
            same = all(np.array_equal(getattr(first, f), getattr(again, f)) for f in ("u", "v", "s1", "s2"))
            print(json.dumps({"repro_matrix": specs[i0].name, "bitwise_equal": bool(same),
                              "rel_error": [first.rel_error, again.rel_error]}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
