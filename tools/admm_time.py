"""Times the on-device ADMM initialisation (nqb_factorize_layer) on synthetic
Llama-shaped weights, reporting the phase split and roofline figures.

usage: python tools/admm_time.py N M BPW [max_seconds]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06694_b200 as nq  # noqa: E402

n, m, bpw = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
r = nq.rank_for_target_bpw(n, m, bpw)
rng = np.random.default_rng(12345)
w = (0.02 * rng.standard_normal((n, m))).astype(np.float32).astype(np.float64)
cfg = nq.AdmmConfig(rank=r)
t0 = time.perf_counter()
layer, err, state = nq.factorize_layer(w, cfg)
secs = time.perf_counter() - t0
res = dict(state.stats)
res.update(iteration=state.iteration, converged=state.converged,
           primal_residual=state.primal_residual)
out = {"n": n, "m": m, "r": r, "bpw": bpw, "wall_s": secs, "rel_error": err}
for k in ("iteration", "converged", "primal_residual", "svd_steps", "svd_power_iters",
          "svd_converged_steps", "sigma_max", "seconds_svd_init", "seconds_iterations"):
    if k in res:
        out[k] = res[k]
if "svd_power_iters" in out and out.get("seconds_svd_init"):
    # one-pass power iteration streams n*m fp64 per iteration
    out["svd_init_gbs"] = out["svd_power_iters"] * 8.0 * n * m / out["seconds_svd_init"] / 1e9
print(json.dumps(out, default=float))
