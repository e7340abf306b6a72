"""Per-call cost breakdown of the host drop-in gemv (nqb_gemv_f32_host) on one 7B layer."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_06694_b200 as nq  # noqa: E402

n, m, bpw = 4096, 4096, 0.8
r = nq.rank_for_target_bpw(n, m, bpw)
ctx = nq.context(0)
ctx.set_stream(None)
lay = nq.DeviceLayer.upload_f16(n, m, r, *bench.random_layer_arrays(np.random.default_rng(0), n, m, r), ctx)
hx = torch.randn(m, dtype=torch.float32).pin_memory().numpy()
hy = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
N = 2000


def timeit(name, fn):
    for _ in range(50):
        fn()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    dt = (time.perf_counter() - t0) / N * 1e6
    print(f"{name:40s} {dt:7.2f} us/call")


timeit("gemv_f32(x, out=pinned)", lambda: lay.gemv_f32(hx, out=hy))
f = ctx.lib.nqb_gemv_f32_host
h, lh = ctx.handle, lay.handle
px, py = hx.ctypes.data_as(C.c_void_p), hy.ctypes.data_as(C.c_void_p)
timeit("raw ctypes nqb_gemv_f32_host", lambda: f(h, lh, px, py))
dx = torch.from_numpy(hx).cuda()
dy = torch.empty(n, device="cuda")
ctx.bind_torch_stream()


def dev():
    lay.gemv_device(dx, dy)
    torch.cuda.synchronize()


timeit("device f32 gemv + sync", dev)
dxh = dx.half()
dyh = dy.half()


def devh():
    lay.gemv_device(dxh, dyh)
    torch.cuda.synchronize()


timeit("device f16 gemv + sync", devh)


def copies():
    dx.copy_(torch.from_numpy(hx), non_blocking=True)
    torch.from_numpy(hy).copy_(dy, non_blocking=True)
    torch.cuda.synchronize()


timeit("torch H2D + D2H copies + sync", copies)
