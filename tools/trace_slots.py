"""Raw trace slots of one decode launch, median over CTAs in us (debug stamps).

usage: NQB_DEC_DBG=4 python tools/trace_slots.py <shape> <slot> [slot ...]
"""
import ctypes as C
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
name, slots = sys.argv[1], [int(a) for a in sys.argv[2:]]
ctx = nq.context(0)
n, m, bpw = SHAPES[name]
r = nq.rank_for_target_bpw(n, m, bpw)
lay = nq.DeviceLayer.upload_f16(n, m, r, *bench.random_layer_arrays(np.random.default_rng(0), n, m, r), ctx)
x = torch.randn(m, device="cuda", dtype=torch.float16)
y = torch.empty(n, device="cuda", dtype=torch.float16)
for _ in range(3):
    lay.gemv_device(x, y)
torch.cuda.synchronize()
grid = C.c_uint32()
st = np.zeros(32 * 148, np.uint64)
for _ in range(2):
    assert ctx.lib.nqb_debug_decode_trace(ctx.handle, lay.handle, C.c_void_p(x.data_ptr()),
                                          C.c_void_p(y.data_ptr()), st.ctypes.data_as(C.c_void_p),
                                          C.byref(grid)) == 0
full = st[:32 * grid.value].reshape(grid.value, 32).astype(np.float64)
for s in slots:
    col = full[:, s]
    col = col[col > 0] / 1.9e3
    print(f"{name} slot {s:2d}: n={col.size:3d} min {col.min():6.2f} med {np.median(col):6.2f} max {col.max():6.2f} us")
