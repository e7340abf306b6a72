"""bench.py — BLR-linear decode throughput on Llama-2-7B layer shapes @0.8 bit.

One step = one batch-1 decode pass through all 224 linear layers of a
Llama-2-7B-shaped model (32 blocks x q,k,v,o 4096x4096 r=1622; gate,up
11008x4096 r=2372; down 4096x11008 r=2372; ranks from rank_for_target_bpw at
0.8 bit, BASELINE.json configs[1]).  Weights are random packed sign bits with
binary16 scales (synthetic, seeded).  A decode pass is issued the way a
decoder issues it: per block q/k/v as one fused launch (they share the
attention input), o, gate/up as one launch (shared MLP input), down; each
launch reads its own fp16 input vector.  The 128 launches of a pass are one
CUDA graph (nqb_graph_*), consecutive kernels overlapped with PDL.  The 224 layers occupy ~0.65 GB, > 5x the 126 MB L2, so every step
streams the bits from HBM (no L2 flush needed; stated in `config`).

  value   = algorithmic bytes of the step / device time (CUDA events, max over
            ranks), inputs resident in HBM.  Algorithmic bytes per layer:
            r(n+m)/8 (bits) + 2(n+m) (fp16 scales) + 2m (x) + 2n (y).
  e2e     = the same metric through the reference-facing drop-in entry point
            (nqb_gemv_f32_host: host x -> device -> host y), H2D/D2H inside.
  roofline: the decode GEMV against MEASURED_PEAKS.json HBM GB/s.
  cpu_baseline: the reference's gemv_packed_f32 (oracle/_ref, unmodified
            reference library) on a bounded sample, one layer per host thread.

--impl reference times the reference CPU implementation alone (rank 0).
Multi-GPU (torchrun): replicas only (decode does not shard), weak scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BLR-linear decode GB/s"
UNIT = "GB/s"
BPW = 0.8
# (name, n, m) of Llama-2-7B decoder linear layers (proj/data/shapes/llama2-7b.shape)
L7_BLOCK = [("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
            ("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]
L70_SHAPES = [("l70_q", 8192, 8192, 0.55), ("l70_gate", 28672, 8192, 0.55),
              ("l70_down", 8192, 28672, 0.55)]


def rank_for(n, m, bpw):  # storage.cpp:124-141 (host arithmetic of the product)
    import paper_2602_06694_b200 as nq
    return nq.rank_for_target_bpw(n, m, bpw)


def algo_bytes(n, m, r):
    return r * (n + m) / 8.0 + 2 * (n + m) + 2 * m + 2 * n


def tensor_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["bf16_tflops"])
    return 1590.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def random_layer_arrays(rng, n, m, r):
    k = (r + 31) // 32
    tail = r % 32
    u = rng.integers(0, 2 ** 32, size=(n, k), dtype=np.uint32)
    v = rng.integers(0, 2 ** 32, size=(m, k), dtype=np.uint32)
    if tail:
        mask = np.uint32((1 << tail) - 1)
        u[:, -1] &= mask
        v[:, -1] &= mask
    s1 = rng.uniform(0.25, 2.0, n).astype(np.float16).view(np.uint16)
    s2 = rng.uniform(0.25, 2.0, m).astype(np.float16).view(np.uint16)
    return u, v, s1, s2


class Clocks:
    """Samples nvidia-smi during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU side: the reference implementation (oracle/_ref) on host cores.
# ---------------------------------------------------------------------------
def cpu_reference_gbs(seconds_target=15.0, threads=None):
    """gemv_packed_f32 of the unmodified reference library, one layer per host
    thread (the reference is single-threaded per call), over the 7 distinct
    Llama-2-7B block shapes round-robin.  Returns (GB/s, cores, sample, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes as C

    import oracle as O
    kind = "reference" if O.reference_available() else "port"
    chk = O.reference() if kind == "reference" else O.restated()
    threads = threads or max(1, os.cpu_count() or 1)
    layers, xs, ys, nbytes = [], [], [], 0.0
    rng = np.random.default_rng(7)
    for t in range(threads):
        name, n, m = L7_BLOCK[t % len(L7_BLOCK)]
        r = rank_for(n, m, BPW)
        u, v, s1h, s2h = random_layer_arrays(rng, n, m, r)
        s1 = s1h.view(np.float16).astype(np.float64)
        s2 = s2h.view(np.float16).astype(np.float64)
        layers.append((n, m, r, u, v, s1, s2))
        xs.append(rng.standard_normal(m).astype(np.float32))
        ys.append(np.empty(n, np.float32))
        nbytes += algo_bytes(n, m, r)

    def run(reps):
        if kind == "reference":
            U32 = C.c_uint32
            cnt = len(layers)
            arr = lambda ty, vals: (ty * cnt)(*vals)  # noqa: E731
            P = C.c_void_p
            fn = chk.lib.nqref_gemv_f32_concurrent
            fn.restype = C.c_int
            t0 = time.perf_counter()
            st = fn(U32(cnt), arr(U32, [l[0] for l in layers]), arr(U32, [l[1] for l in layers]),
                    arr(U32, [l[2] for l in layers]),
                    arr(P, [l[3].ctypes.data for l in layers]),
                    arr(P, [l[4].ctypes.data for l in layers]),
                    arr(P, [l[5].ctypes.data for l in layers]),
                    arr(P, [l[6].ctypes.data for l in layers]),
                    arr(P, [x.ctypes.data for x in xs]), arr(P, [y.ctypes.data for y in ys]),
                    U32(reps))
            assert st == 0
            return time.perf_counter() - t0
        # port: sequential restatement (single core)
        t0 = time.perf_counter()
        for _ in range(reps):
            for (n, m, r, u, v, s1, s2), x in zip(layers, xs):
                chk.gemv_packed_f32(O.Layer(n, m, r, u, v, s1, s2), x)
        return time.perf_counter() - t0

    probe = run(1)
    reps = max(1, int(seconds_target / max(probe, 1e-3)))
    secs = run(reps)
    gbs = nbytes * reps / secs / 1e9
    cores = threads if kind == "reference" else 1
    sample = (f"{len(layers)} Llama-2-7B block layers @0.8 bit (q,k,v,o,gate,up,down round-robin),"
              f" one per host thread, {reps} gemv_packed_f32 calls each, {secs:.1f} s")
    return gbs, cores, sample, kind, secs


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
def build_model(nq, ctx, seed):
    """32 Llama-2-7B blocks; per block the four decode launches a decoder makes:
    q/k/v as one group (shared attention input), o, gate/up as one group
    (shared MLP input), down.  Returns [(launch, [layers])]."""
    rng = np.random.default_rng(seed)
    ranks = {name: rank_for(n, m, BPW) for name, n, m in L7_BLOCK}
    launches = []
    for blk in range(32):
        lay = {}
        for name, n, m in L7_BLOCK:
            r = ranks[name]
            u, v, s1, s2 = random_layer_arrays(rng, n, m, r)
            lay[name] = nq.DeviceLayer.upload_f16(n, m, r, u, v, s1, s2, ctx)
        launches.append((nq.DecodeGroup([lay["q"], lay["k"], lay["v"]]), [lay["q"], lay["k"], lay["v"]]))
        launches.append((None, [lay["o"]]))
        launches.append((nq.DecodeGroup([lay["gate"], lay["up"]]), [lay["gate"], lay["up"]]))
        launches.append((None, [lay["down"]]))
    return launches


def make_step(launches, xs, ys):
    def step():
        for (grp, lays), x, y in zip(launches, xs, ys):
            if grp is None:
                lays[0].gemv_device(x, y[0])
            else:
                grp.gemv_device(x, y)
    return step


def graph_time(torch, ctx, stream, fn, reps, warmup=3):
    """Captures fn() into one CUDA graph (library graph API) and times `reps`
    replays with CUDA events on the capturing stream.  Returns (seconds per
    replay, kernel launches per replay)."""
    with torch.cuda.stream(stream):
        ctx.bind_torch_stream()
        fn()  # eager warm-up (also proves the path outside a graph)
        l0 = ctx.kernel_launches
        with ctx.capture() as cap:
            fn()
        per = ctx.kernel_launches - l0
        for _ in range(warmup):
            cap.graph.launch()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            cap.graph.launch()
        e1.record(stream)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps, per, cap.graph


def shape_roofline(nq, ctx, torch, stream, n, m, r, reps=20):
    """Back-to-back single-layer decode GEMVs over distinct copies totalling
    > 4x L2 (every call reads its bits from HBM), captured in one graph."""
    per = algo_bytes(n, m, r)
    copies = max(4, int(np.ceil(4 * 126e6 / per)))
    rng = np.random.default_rng(n + m + r)
    lays = [nq.DeviceLayer.upload_f16(n, m, r, *random_layer_arrays(rng, n, m, r), ctx)
            for _ in range(copies)]
    xs = [torch.randn(m, device="cuda", dtype=torch.float16) for _ in range(copies)]
    ys = [torch.empty(n, device="cuda", dtype=torch.float16) for _ in range(copies)]

    def step():
        for lay, x, y in zip(lays, xs, ys):
            lay.gemv_device(x, y)
    sec, _, g = graph_time(torch, ctx, stream, step, reps)
    g.free()
    return sec / copies, per


def prefill_roofline(nq, ctx, torch, stream, n, m, r, b=2048, reps=10):
    """Prefill GEMM (tcgen05 kind::f16) on one layer, b tokens: seconds per call
    and TFLOP/s of the algorithmic 2*b*r*(n+m) FLOPs."""
    rng = np.random.default_rng(n * 3 + m)
    lay = nq.DeviceLayer.upload_f16(n, m, r, *random_layer_arrays(rng, n, m, r), ctx)
    x = torch.randn(b, m, device="cuda", dtype=torch.float16)
    y = torch.empty(b, n, device="cuda", dtype=torch.float16)
    sec, _, g = graph_time(torch, ctx, stream, lambda: lay.gemm_device(x, y), reps)
    g.free()
    return sec, 2.0 * b * r * (n + m) / sec / 1e12


def admm_leg(nq, torch, ws, rank, local):
    """Whole-model-init throughput sample: `ws` Llama-2-7B q matrices (4096x4096, synthetic
    N(0, 0.02^2) weights, 1.0 bpw -> r = 2032), one per rank by the LPT plan, each factorised
    by nqb_factorize_layer (fp64 SVD init + ADMM, reference defaults), packed factors
    gathered to rank 0 (NCCL).  Returns rank 0's summary (None elsewhere)."""
    from paper_2602_06694_b200 import sharded as S
    specs = [S.MatrixSpec(f"b{i}.q", 4096, 4096, 0x7B000000 + 7 * i) for i in range(ws)]
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    rep = S.sharded_init(specs, 1.0, device=torch.device("cuda", local))
    wall = time.perf_counter() - t0
    if rank != 0:
        return None
    secs = max(rep.per_rank_seconds)
    errs = [rep.matrices[i].rel_error for i in sorted(rep.matrices)]
    its = [rep.matrices[i].iterations for i in sorted(rep.matrices)]
    return {"matrices": len(specs), "shape": "4096x4096", "bpw": 1.0,
            "rank": rep.matrices[0].r, "seconds_max_rank": secs, "seconds_wall_incl_gather": wall,
            "matrices_per_s": len(specs) / wall, "scaling": "weak (one matrix per rank)",
            "rel_error": errs, "admm_iterations": its,
            "converged": [rep.matrices[i].converged for i in sorted(rep.matrices)],
            "note": "fp64 on device (SVD-init power iterations + ADMM); CPU reference ~36 h "
                    "per 4096^2 matrix (SURVEY.md section 6)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shapes", action="store_true", help="skip the per-shape roofline sweep")
    ap.add_argument("--no-admm", action="store_true",
                    help="skip the ADMM-init leg (one 4096x4096 matrix per rank, ~80 s)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws, rank, local = dist_env()

    if args.impl == "reference":
        if rank != 0:
            return
        gbs, cores, sample, kind, secs = cpu_reference_gbs(
            seconds_target=max(5.0, min(60.0, 2.0 * args.steps)))
        line = {"metric": METRIC, "value": gbs, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "impl": "reference",
                "config": {"workload": "llama2-7b decode pass, 224 linear layers @0.8 bit, batch 1",
                           "host_cores": os.cpu_count()},
                "cpu_baseline": {"value": gbs, "unit": UNIT, "cores": cores, "kind": kind,
                                 "sample": sample},
                "e2e": {"value": gbs, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2602_06694_b200 as nq
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = nq.context(local)
    stream = torch.cuda.Stream()

    launch_list = build_model(nq, ctx, seed=1234 + rank)
    xs, ys, step_bytes = [], [], 0.0
    for grp, lays in launch_list:
        xs.append(torch.randn(lays[0].m, device="cuda", dtype=torch.float16))
        ys.append([torch.empty(l.n, device="cuda", dtype=torch.float16) for l in lays])
        # x is read once per launch, even when the launch serves 2-3 layers
        step_bytes += sum(algo_bytes(l.n, l.m, l.r) for l in lays) - 2 * lays[0].m * (len(lays) - 1)
    step = make_step(launch_list, xs, ys)

    # one decode pass = one CUDA graph of 128 fused launches (PDL between them)
    with torch.cuda.stream(stream):
        ctx.bind_torch_stream()
        step()
        l0 = ctx.kernel_launches
        with ctx.capture() as cap:
            step()
        launches_per_step = ctx.kernel_launches - l0
        graph = cap.graph
        for _ in range(args.warmup):
            graph.launch()
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    with Clocks(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            graph.launch()
        e1.record(stream)
        torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / 1e3
    launches = launches_per_step * args.steps
    if ws > 1:
        t = torch.tensor([secs], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        secs = float(t.item())
        torch.distributed.barrier()
    value = ws * step_bytes * args.steps / secs / 1e9

    # ---- e2e: the reference-facing drop-in (gemv_packed_f32 -> nqb_gemv_f32_host),
    #      per layer: pinned host x -> device -> kernel -> host y, synchronous ----
    all_layers = [l for _, lays in launch_list for l in lays]
    h2d = sum(4 * l.m for l in all_layers)
    d2h = sum(4 * l.n for l in all_layers)
    hx = [torch.randn(l.m, dtype=torch.float32).pin_memory().numpy() for l in all_layers]
    hy = [torch.empty(l.n, dtype=torch.float32).pin_memory().numpy() for l in all_layers]
    ctx.set_stream(None)

    def e2e_step():
        for l, x, y in zip(all_layers, hx, hy):
            l.gemv_f32(x, out=y)
    e2e_step()
    e2e_steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_secs = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_secs], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_secs = float(t.item())
    e2e = {"value": ws * step_bytes * e2e_steps / e2e_secs / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "api": "nqb_gemv_f32_host per layer (gemv_packed_f32 drop-in, pinned host buffers)",
           "steps": e2e_steps}

    # ---- ADMM init (north_star part 2): the layer-sharded driver, one Llama-2-7B
    #      4096x4096 matrix per rank at 1 bit/param, gathered to rank 0 -> matrices/s ----
    admm = None
    if not args.no_admm:
        admm = admm_leg(nq, torch, ws, rank, local)

    peak, peak_kind = measured_peaks()
    extra = {}
    if admm is not None and rank == 0:
        extra["admm_init"] = admm
    roof = None
    if rank == 0:
        shapes = {}
        if not args.no_shapes:
            for name, n, m, bpw in [("l7_q", 4096, 4096, 0.8), ("l7_gate", 11008, 4096, 0.8),
                                    ("l7_down", 4096, 11008, 0.8)] + list(L70_SHAPES):
                r = rank_for(n, m, bpw)
                sec, per = shape_roofline(nq, ctx, torch, stream, n, m, r)
                shapes[f"{name}_{bpw}"] = {"n": n, "m": m, "r": r, "us": sec * 1e6,
                                           "gbs": per / sec / 1e9, "frac": per / sec / 1e9 / peak}
        extra["per_shape_single_layer"] = shapes
        if not args.no_shapes:
            # BASELINE config 5: bitrate sweep on Llama-2-13B shapes (decode GB/s; the ADMM
            # reconstruction error vs the CPU reference at these bitrates is pinned by the
            # l13s16_* fixtures in tests/test_gpu_admm.py)
            sweep = {}
            for name, n, m in [("l13_q", 5120, 5120), ("l13_gate", 13824, 5120),
                               ("l13_down", 5120, 13824)]:
                for bpw in (0.55, 0.8, 1.0):
                    r = rank_for(n, m, bpw)
                    sec, per = shape_roofline(nq, ctx, torch, stream, n, m, r, reps=10)
                    sweep[f"{name}_{bpw}"] = {"n": n, "m": m, "r": r, "us": sec * 1e6,
                                              "gbs": per / sec / 1e9,
                                              "frac": per / sec / 1e9 / peak}
            extra["bitrate_sweep_l13_decode"] = sweep
        if not args.no_shapes:
            pref = {}
            tpk = tensor_peak()
            for name, n, m, bpw in L70_SHAPES:
                r = rank_for(n, m, bpw)
                sec, tf = prefill_roofline(nq, ctx, torch, stream, n, m, r)
                pref[f"{name}_{bpw}_b2048"] = {"n": n, "m": m, "r": r, "ms": sec * 1e3,
                                               "tflops": tf, "frac_of_bf16_peak": tf / tpk}
            extra["prefill_tcgen05"] = pref
        achieved = step_bytes * args.steps / secs / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r01_decode_imma", "traffic.json")
        if os.path.exists(tp):  # ncu dram__bytes_read+write per launch of this same step
            traffic = json.load(open(tp))["step"]["dram_bytes_per_launch"]
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_note": "ncu dram bytes per launch (profiles/r01_decode_imma/traffic.json); "
                                "algorithmic bytes per launch = algorithmic_bytes_per_step / "
                                "launches_per_step",
                "peak_source": peak_kind,
                "kernel": "nqb::dec::k_decode (fused two-stage decode GEMV; every launch of the "
                          "step is this kernel, PDL-overlapped, so duration = step time / launches)",
                "algorithmic_bytes_per_step": step_bytes, "launches_per_step": launches_per_step,
                "us_per_launch": secs / args.steps / launches_per_step * 1e6}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            gbs, cores, sample, kind, _ = cpu_reference_gbs(args.cpu_seconds)
            cpu = {"value": gbs, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": f"error: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u1 x s8-limb IMMA, int32/int64 exact accumulate (fp16 x/y I/O)",
                "data": "synthetic (seeded random sign bits, binary16 scales U(0.25,2), N(0,1) fp16 x)",
                "config": {"workload": "llama2-7b decode pass: 224 linear layers (32 x q,k,v,o "
                                       "4096x4096 r=1622; gate,up 11008x4096 r=2372; down "
                                       "4096x11008 r=2372) @0.8 bit, batch 1, as 128 fused "
                                       "launches (qkv group, o, gate/up group, down) in one "
                                       "CUDA graph",
                           "parallelism": f"replicas x{ws}", "l2": "working set 0.65 GB > L2 "
                           "(126 MB): no flush needed", "bpw": BPW},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
                "gpu_launches": launches, "extra": extra}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
