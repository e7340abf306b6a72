"""Small driver for ncu: a few decode launches per shape (no timing printed).

usage: python tools/prof_decode.py [shape ...]   shapes: l7_q l7_gate l7_down l70_q l70_gate l70_down
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_06694_b200 as nq  # noqa: E402

SHAPES = {"l7_q": (4096, 4096, 0.8), "l7_gate": (11008, 4096, 0.8), "l7_down": (4096, 11008, 0.8),
          "l70_q": (8192, 8192, 0.55), "l70_gate": (28672, 8192, 0.55),
          "l70_down": (8192, 28672, 0.55)}

ctx = nq.context(0)
rng = np.random.default_rng(0)
for name in sys.argv[1:] or ["l70_gate", "l7_q"]:
    n, m, bpw = SHAPES[name]
    r = nq.rank_for_target_bpw(n, m, bpw)
    lay = nq.DeviceLayer.upload_f16(n, m, r, *bench.random_layer_arrays(rng, n, m, r), ctx)
    x = torch.randn(m, device="cuda", dtype=torch.float16)
    y = torch.empty(n, device="cuda", dtype=torch.float16)
    for _ in range(4):
        lay.gemv_device(x, y)
    torch.cuda.synchronize()
print("done")
