"""Generates the committed ADMM golden fixtures from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py [names...]

Each case runs the reference per-matrix pipeline step (pipeline.cpp:95-110,
:150-153: admm_factorize -> balance_and_extract_scales(identity) ->
make_factorized_layer -> relative_frobenius_error(W, reconstruct_dense)) through
oracle/_ref/libnqref.so on W = fp32(0.02 * g), g ~ Rng(seed),
and stores the packed factors, double scales, error and solver statistics.
The GPU box regenerates W from the seed with the C restatement (bit-identical
Rng, checked by tests/test_oracle.py), so W itself is not stored.
"""
from __future__ import annotations

import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

# name -> (n, m, bpw, seed, max_iters)
CASES = {
    "w64x48_b1.0": (64, 48, 1.0, 12345, 400),
    "w128_b1.0": (128, 128, 1.0, 0xB1A5E001, 400),
    "w96x160_b0.8": (96, 160, 0.8, 7, 400),
    "w256_b1.0": (256, 256, 1.0, 0xB1A5E001, 400),
    "w256_b0.55": (256, 256, 0.55, 0xB1A5E001, 400),
    # Llama-2-13B shapes scaled 1/16
    "l13s16_q_b1.0": (320, 320, 1.0, 0x13B00000, 400),
    "l13s16_q_b0.8": (320, 320, 0.8, 0x13B00000, 400),
    "l13s16_q_b0.55": (320, 320, 0.55, 0x13B00000, 400),
    "l13s16_gate_b0.55": (864, 320, 0.55, 0x13B00004, 400),
    "l13s16_down_b0.55": (320, 864, 0.55, 0x13B00006, 400),
    "l13s16_gate_b0.8": (864, 320, 0.8, 0x13B00004, 400),
    "l13s16_gate_b1.0": (864, 320, 1.0, 0x13B00004, 400),
    "l13s16_down_b0.8": (320, 864, 0.8, 0x13B00006, 400),
    "l13s16_down_b1.0": (320, 864, 1.0, 0x13B00006, 400),
    # Llama-2-13B shapes scaled 1/8
    "l13s8_q_b1.0": (640, 640, 1.0, 0x13B80000, 400),
    "l13s8_q_b0.8": (640, 640, 0.8, 0x13B80000, 400),
    "l13s8_q_b0.55": (640, 640, 0.55, 0x13B80000, 400),
    "l13s8_gate_b1.0": (1728, 640, 1.0, 0x13B80004, 400),
    "l13s8_gate_b0.8": (1728, 640, 0.8, 0x13B80004, 400),
    "l13s8_gate_b0.55": (1728, 640, 0.55, 0x13B80004, 400),
    "l13s8_down_b1.0": (640, 1728, 1.0, 0x13B80006, 400),
    "l13s8_down_b0.8": (640, 1728, 0.8, 0x13B80006, 400),
    "l13s8_down_b0.55": (640, 1728, 0.55, 0x13B80006, 400),
    "w512_b1.0": (512, 512, 1.0, 0xB1A5E001, 400),
    "w512_b0.55": (512, 512, 0.55, 0xB1A5E001, 400),
    "w1024_b1.0": (1024, 1024, 1.0, 0xB1A5E001, 400),
}


def run_case(name: str) -> str:
    n, m, bpw, seed, iters = CASES[name]
    ref = O.reference()
    w = O.synthetic_weight(ref, seed, n, m)
    r = ref.rank_for_target_bpw(n, m, bpw)
    cfg = O.AdmmConfig.make(rank=r, max_iters=iters)
    t0 = time.time()
    layer, err, trace, res = ref.factorize_layer(w, cfg)
    secs = time.time() - t0
    np.savez_compressed(
        os.path.join(HERE, f"admm_{name}.npz"), n=n, m=m, r=r, bpw=bpw, seed=seed,
        max_iters=iters, u=layer.u, v=layer.v, s1=layer.s1, s2=layer.s2, rel_err=err,
        trace=trace, iteration=res["iteration"], converged=res["converged"],
        primal_residual=res["primal_residual"], rho=res["rho"], cpu_seconds=secs,
        w_sumsq=float(np.sum(w * w)))
    return json.dumps({"case": name, "n": n, "m": m, "r": r, "rel_err": err,
                       "iteration": res["iteration"], "cpu_seconds": round(secs, 2)})


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    with Pool(min(len(names), os.cpu_count() or 1)) as pool:
        for line in pool.imap_unordered(run_case, names):
            print(line, flush=True)
