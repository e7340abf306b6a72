"""Times truncated_svd_factors(W, k) (k deflation steps of 1000 power iterations
each on random W) and prints the factors' checksum, for A/B of the power-iteration
kernels: python tools/power_ab.py n m [k]"""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06694_b200 as nq  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = nq.synthetic_weight(0x7B000006, n, m)
nq.truncated_svd_factors(w, 1)
t0 = time.perf_counter()
u, v = nq.truncated_svd_factors(w, k)
dt = time.perf_counter() - t0
h = hashlib.sha1(u.tobytes() + v.tobytes()).hexdigest()[:16]
print(f"{n}x{m} k={k}: {dt / k * 1e3:.1f} ms per deflation step "
      f"({dt / k / 1002 * 1e6:.1f} us per power iteration, "
      f"{8.0 * n * m * 1002 * k / dt / 1e9:.0f} GB/s) sha {h}", flush=True)
