"""Per-phase timeline of one decode launch (nqb_debug_decode_trace), per shape.

Stamps (decode.cu TRACE): 0 start, 1 consumers ready, 2 after griddepcontrol.wait,
3 x statistics, 4 stage-1 B fragments, 5 stage-1 MMA, 6 published + fenced,
7 arrived (CTAs with stage-2 work), 8 barrier passed, 9 stage-2 B fragments,
10 stage-2 MMA, 11 outputs written, 12/13 warp 0 done with stage 1/2 MMA,
14 producer issued all copies, 15 whole stream landed in shared memory.  Times in us relative to the earliest start.
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
ctx = nq.context(0)
rng = np.random.default_rng(0)
for name in sys.argv[1:] or list(SHAPES):
    n, m, bpw = SHAPES[name]
    r = nq.rank_for_target_bpw(n, m, bpw)
    lay = nq.DeviceLayer.upload_f16(n, m, r, *bench.random_layer_arrays(rng, n, m, r), ctx)
    x = torch.randn(m, device="cuda", dtype=torch.float16)
    y = torch.empty(n, device="cuda", dtype=torch.float16)
    for _ in range(3):
        lay.gemv_device(x, y)
    torch.cuda.synchronize()
    for trial in range(2):
        grid = C.c_uint32()
        st = np.zeros(32 * 148, np.uint64)
        rc = ctx.lib.nqb_debug_decode_trace(ctx.handle, lay.handle, C.c_void_p(x.data_ptr()),
                                            C.c_void_p(y.data_ptr()), st.ctypes.data_as(C.c_void_p),
                                            C.byref(grid))
        assert rc == 0, ctx.lib.nqb_last_error()
    G = grid.value
    full = st[:32 * G].reshape(G, 32).astype(np.float64)
    ghz = 1.9
    cyc = full[:, :16].copy()
    cyc[:, 0] = (full[:, 0] - full[:, 0].min()) * ghz  # start skew (ns -> cycles)
    us = np.where(cyc > 0, cyc / ghz / 1e3, np.nan)
    us[:, 0] = cyc[:, 0] / ghz / 1e3
    print(f"{name}: n={n} m={m} r={r} grid={G} bytes={lay.device_bytes/1e6:.2f} MB "
          f"(HBM time at 6.4 TB/s: {lay.device_bytes/6.4e12*1e6:.2f} us); times in us since CTA start @1.9GHz")
    labels = ["start_skew", "ready", "pdl_wait", "x_stats", "s1_frag", "s1_mma", "s1_pub", "arrived",
              "barrier", "s2_frag", "s2_mma", "end", "ep_ready", "t_reds", "prod_issued",
              "all_landed"]
    endt = np.nan_to_num(us[:, 11])
    order = np.argsort(-endt)
    print("   slowest CTAs: " + "; ".join(
        f"cta{c} sm{int(full[c,16])} s1=({int(full[c,17])}x{int(full[c,18])}) s2={int(full[c,19])} "
        f"nsec={int(full[c,20])} end={endt[c]:.2f}" for c in order[:3]))
    for i, lab in enumerate(labels):
        col = us[:, i]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"   {i:2d} {lab:11s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f}  (n={col.size})")
    for st, base in (("stage1", 22), ("stage2", 27)):
        sel = full[:, base + 4] > 0  # warp 0 of each CTA: [wait, -, mma, flush, units]
        if sel.any():
            u = full[sel, base + 4].sum()
            print(f"   {st} warp0 ({u/sel.sum():.1f} tile units/CTA): wait-landed {full[sel, base].mean():.0f} "
                  f"mma {full[sel, base + 2].mean():.0f} flush {full[sel, base + 3].mean():.0f} cycles/CTA, "
                  f"mma {full[sel, base + 2].sum() / u:.0f} cycles/unit")
