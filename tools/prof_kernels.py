"""Small driver for ncu captures: decode (70B gate), prefill (70B q, b=2048) and
the SVD-init power iteration (4096^2, a few deflation steps)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_06694_b200 as nq  # noqa: E402

what = sys.argv[1]
ctx = nq.context(0)
rng = np.random.default_rng(0)
if what == "decode":
    n, m, r = 28672, 8192, nq.rank_for_target_bpw(28672, 8192, 0.55)
    lay = nq.DeviceLayer.upload_f16(n, m, r, *bench.random_layer_arrays(rng, n, m, r), ctx)
    x = torch.randn(m, device="cuda", dtype=torch.float16)
    y = torch.empty(n, device="cuda", dtype=torch.float16)
    for _ in range(4):
        lay.gemv_device(x, y)
elif what == "prefill":
    n, m, r = 8192, 8192, nq.rank_for_target_bpw(8192, 8192, 0.55)
    lay = nq.DeviceLayer.upload_f16(n, m, r, *bench.random_layer_arrays(rng, n, m, r), ctx)
    x = torch.randn(2048, m, device="cuda", dtype=torch.float16)
    y = torch.empty(2048, n, device="cuda", dtype=torch.float16)
    for _ in range(2):
        lay.gemm_device(x, y)
elif what == "power":
    w = (0.02 * rng.standard_normal((4096, 4096))).astype(np.float32).astype(np.float64)
    nq.truncated_svd_factors(w[:, :], 3)
torch.cuda.synchronize()
print("done")
