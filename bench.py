"""bench.py — BLR-linear decode throughput on Llama-2-7B layer shapes @0.8 bit.

One step = one batch-1 decode pass through all 224 linear layers of a
Llama-2-7B-shaped model (32 blocks x q,k,v,o 4096x4096 r=1622; gate,up
11008x4096 r=2372; down 4096x11008 r=2372; ranks from rank_for_target_bpw at
0.8 bit, BASELINE.json configs[1]).  Weights are random packed sign bits with
binary16 scales (synthetic, seeded).  The pass is issued the way a decoder
issues it: per block q/k/v as one group (they share the attention input), o,
gate/up as one group (shared MLP input), down; each step reads its own input
vector.  Our arm runs the whole pass as ONE launch of the persistent decode-pass
kernel (nqb_pass).  The 224 layers occupy ~0.65 GB, > 5x the 126 MB L2, so
every step streams the bits from HBM (no L2 flush needed; stated in `config`).

  value   = algorithmic bytes of the step / device time (CUDA events, max over
            ranks), inputs resident in HBM.  Algorithmic bytes per layer:
            r(n+m)/8 (bits) + 2(n+m) (fp16 scales) + 2n (y), plus 2m (x) once
            per step.
  e2e     = the same metric through the C ABI with HOST buffers
            (nqb_pass_run_host: pinned host x -> device, the pass, device -> host
            y, synchronous), copies inside the timed region.
  roofline: the decode-pass kernel against MEASURED_PEAKS.json HBM GB/s.
  cpu_baseline: the reference's gemv_packed_f32 (oracle/_ref, the unmodified
            reference library) over the same 224-layer pass, layers spread over
            all host threads, on a bounded sample of whole passes.

--impl reference times the reference CPU implementation alone (rank 0) on the
same workload and config.  Multi-GPU (torchrun): replicas only (decode does not
shard), weak scaling.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
admm_layer_for_cpu = None  # config 1: the ADMM's layer, for the CPU forward baseline
sys.path.insert(0, ROOT)

METRIC = "BLR-linear decode GB/s"
UNIT = "GB/s"
BPW = 0.8
SEED = 1234
# (name, n, m) of the decoder linear layers (proj/data/shapes/llama2-7b.shape)
L7_BLOCK = [("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
            ("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]
L70_BLOCK = [("q", 8192, 8192), ("k", 1024, 8192), ("v", 1024, 8192), ("o", 8192, 8192),
             ("gate", 28672, 8192), ("up", 28672, 8192), ("down", 8192, 28672)]
L70_SHAPES = [("l70_q", 8192, 8192, 0.55), ("l70_gate", 28672, 8192, 0.55),
              ("l70_down", 8192, 28672, 0.55)]
STEP_GROUPS = [("qkv", ["q", "k", "v"]), ("o", ["o"]), ("gateup", ["gate", "up"]), ("down", ["down"])]


def config_of(n_gpus):
    """The workload description, identical in both arms."""
    return {"workload": "llama2-7b decode pass: 224 linear layers (32 x q,k,v,o 4096x4096 r=1622; "
                        "gate,up 11008x4096 r=2372; down 4096x11008 r=2372) @0.8 bit, batch 1, "
                        "steps per block: qkv group, o, gate/up group, down",
            "bpw": BPW, "batch": 1, "layers": 224, "seed": SEED,
            "parallelism": f"replicas x{n_gpus}",
            "l2": "working set 0.65 GB > L2 (126 MB): no flush needed"}


def algo_bytes(n, m, r):
    return r * (n + m) / 8.0 + 2 * (n + m) + 2 * m + 2 * n


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


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


def workload(rank_fn, block=L7_BLOCK, blocks=32, bpw=BPW, seed=SEED):
    """The pass as host arrays: [(step kind, [(name, n, m, r, (u, v, s1h, s2h))], x fp16)].
    Same generator and order in both arms."""
    rng = np.random.default_rng(seed)
    ranks = {nm: rank_fn(n, m, bpw) for nm, n, m in block}
    dims = {nm: (n, m) for nm, n, m in block}
    steps = []
    for _ in range(blocks):
        lay = {nm: (nm, n, m, ranks[nm], random_layer_arrays(rng, n, m, ranks[nm])) for nm, n, m in block}
        for kind, names in STEP_GROUPS:
            m = dims[names[0]][1]
            x = rng.standard_normal(m).astype(np.float16)
            steps.append((kind, [lay[nm] for nm in names], x))
    return steps


def step_bytes_of(steps):
    tot = 0.0
    for _, lays, _ in steps:
        tot += sum(algo_bytes(n, m, r) for _, n, m, r, _ in lays) - 2 * lays[0][2] * (len(lays) - 1)
    return tot


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
                self._stop.wait(0.1)
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
# CPU side: the unmodified reference library (oracle/_ref) on the host cores.
# Only this leg and --impl reference touch oracle/.
# ---------------------------------------------------------------------------
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    return O


class RefPass:
    """The decode pass on the reference: gemv_packed_f32 (packed.cpp:201-204) of
    every layer, layers spread over `threads` host threads (nqref_pass_*)."""

    def __init__(self, steps, threads):
        O = _oracle()
        if not O.reference_available():
            raise RuntimeError("oracle/_ref/libnqref.so not built")
        self.lib = O.reference().lib
        self.threads = threads
        P = C.c_void_p
        lays = [(l, x) for _, ls, x in steps for l in ls]
        cnt = len(lays)
        self._keep = []
        arrs = {k: [] for k in ("n", "m", "r", "u", "v", "s1", "s2", "x")}
        for (_, n, m, r, (u, v, s1h, s2h)), x in lays:
            s1 = s1h.view(np.float16).astype(np.float64)
            s2 = s2h.view(np.float16).astype(np.float64)
            xf = x.astype(np.float32)
            self._keep += [s1, s2, xf]
            for k, val in (("n", n), ("m", m), ("r", r), ("u", u.ctypes.data), ("v", v.ctypes.data),
                           ("s1", s1.ctypes.data), ("s2", s2.ctypes.data), ("x", xf.ctypes.data)):
                arrs[k].append(val)
        U32 = C.c_uint32
        self.lib.nqref_pass_create.restype = P
        self.lib.nqref_pass_run.restype = C.c_int
        self.lib.nqref_pass_destroy.restype = None
        self.h = self.lib.nqref_pass_create(
            U32(cnt), (U32 * cnt)(*arrs["n"]), (U32 * cnt)(*arrs["m"]), (U32 * cnt)(*arrs["r"]),
            (P * cnt)(*arrs["u"]), (P * cnt)(*arrs["v"]), (P * cnt)(*arrs["s1"]),
            (P * cnt)(*arrs["s2"]), (P * cnt)(*arrs["x"]))
        if not self.h:
            raise RuntimeError("nqref_pass_create failed")
        self.ys = [np.empty(l[1], np.float32) for l, _ in lays]
        self._yp = (P * cnt)(*[y.ctypes.data for y in self.ys])

    def run(self):
        assert self.lib.nqref_pass_run(C.c_void_p(self.h), self._yp, C.c_uint32(self.threads)) == 0

    def close(self):
        if self.h:
            self.lib.nqref_pass_destroy(C.c_void_p(self.h))
            self.h = None


def ref_rank_fn():
    O = _oracle()
    chk = O.reference() if O.reference_available() else O.restated()
    return chk.rank_for_target_bpw


def cpu_pass_baseline(steps, step_bytes, seconds_target=15.0):
    """Whole reference passes on all host threads for ~seconds_target."""
    threads = max(1, os.cpu_count() or 1)
    rp = RefPass(steps, threads)
    t0 = time.perf_counter()
    rp.run()
    one = time.perf_counter() - t0
    reps = max(1, int(round(seconds_target / max(one, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(reps):
        rp.run()
    secs = time.perf_counter() - t0
    rp.close()
    return {"value": step_bytes * reps / secs / 1e9, "unit": UNIT, "cores": threads,
            "kind": "reference",
            "sample": f"{reps} whole 224-layer decode passes (gemv_packed_f32 per layer, "
                      f"{threads} host threads over layers), {secs:.1f} s"}


def cpu_prefill_baseline(shapes):
    """gemm_packed (packed.cpp:260-287) with NQ_THREADS = nproc on a deterministic
    64-column subset of b = 2048 at the 70B shapes (columns are independent)."""
    O = _oracle()
    ref = O.reference()
    threads = max(1, os.cpu_count() or 1)
    out = {}
    for name, n, m, r, arrs in shapes:
        u, v, s1h, s2h = arrs
        lay = O.Layer(n, m, r, u, v, s1h.view(np.float16).astype(np.float64),
                      s2h.view(np.float16).astype(np.float64))
        x = np.random.default_rng(n + m).standard_normal((m, 64)).astype(np.float16).astype(np.float64)
        t0 = time.perf_counter()
        ref.gemm_packed(lay, x, threads=threads)
        secs = time.perf_counter() - t0
        out[name] = {"tflops": 2.0 * 64 * r * (n + m) / secs / 1e12, "seconds": secs, "columns": 64,
                     "threads": threads, "kind": "reference"}
    return out


def cpu_admm_baseline(seconds_hint=None):
    """admm_factorize (admm.cpp:127-199) of the reference at 256^2, 1 bit (r = 112),
    one matrix per host thread concurrently, W from Rng(0x7B000000 + i); plus one
    4096^2 power iteration (linalg.cpp:101-136) to extrapolate the SVD init."""
    O = _oracle()
    ref = O.reference()
    threads = max(1, os.cpu_count() or 1)
    n = 256
    r = ref.rank_for_target_bpw(n, n, 1.0)
    ws = [O.synthetic_weight(ref, 0x7B000000 + i, n, n) for i in range(threads)]
    res = [None] * threads
    from concurrent.futures import ThreadPoolExecutor

    def one(i):
        res[i] = ref.admm_factorize(ws[i], O.AdmmConfig.make(rank=r))

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(threads)))
    secs = time.perf_counter() - t0
    big = O.synthetic_weight(ref, 0xB1A5E001, 4096, 4096)
    t0 = time.perf_counter()
    ref.top_singular_pair(big, 1, 0.0)
    t1 = time.perf_counter()
    ref.top_singular_pair(big, 3, 0.0)
    t2 = time.perf_counter()
    t_iter = max(1e-6, ((t2 - t1) - (t1 - t0)) / 2.0)
    return {"matrices_per_s_256": threads / secs, "seconds_256_concurrent": secs, "rank_256": r,
            "threads": threads, "kind": "reference",
            "power_iteration_4096_s": t_iter,
            "svd_init_4096_r2032_extrapolated_s": 2032 * 1000 * t_iter,
            "extrapolation": "SVD init at 4096^2 r=2032 = 2032 deflations x 1000 power iterations "
                             "(random W never meets the 1e-13 stop rule, SURVEY §6) x the measured "
                             "single-thread 4096^2 power iteration; a lower bound on the CPU time "
                             "per matrix (the ADMM iterations come on top)"}, ws, r


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
def build_pass(nq, ctx, torch, steps):
    """Uploads the layers, makes the groups and the pass over device x/y."""
    keep, pass_steps = [], []
    for kind, lays, x in steps:
        dev = [nq.DeviceLayer.upload_f16(n, m, r, *arrs, ctx) for _, n, m, r, arrs in lays]
        unit = nq.DecodeGroup(dev) if len(dev) > 1 else dev[0]
        xd = torch.from_numpy(x).cuda()
        ys = [torch.empty(l[1], device="cuda", dtype=torch.float16) for l in lays]
        keep.append((dev, unit))
        pass_steps.append((unit, xd, ys))
    return nq.DecodePass(pass_steps, ctx), pass_steps, keep


def time_launches(torch, stream, fn, reps, warmup):
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def graph_of(ctx, torch, stream, fn):
    with torch.cuda.stream(stream):
        ctx.bind_torch_stream()
        fn()
        with ctx.capture() as cap:
            fn()
    return cap.graph


def per_call_graph_gbs(nq, ctx, torch, stream, pass_steps, step_bytes, reps=10):
    """The same pass as 128 per-call launches (k_decode, PDL) in one CUDA graph."""
    def step():
        for unit, x, ys in pass_steps:
            if isinstance(unit, nq.DecodeGroup):
                unit.gemv_device(x, ys)
            else:
                unit.gemv_device(x, ys[0])
    g = graph_of(ctx, torch, stream, step)
    sec = time_launches(torch, stream, g.launch, reps, 3)
    g.free()
    return {"gbs": step_bytes / sec / 1e9, "us": sec * 1e6, "launches": len(pass_steps)}


def shape_roofline(nq, ctx, torch, stream, n, m, r, hbm, reps=20):
    """Back-to-back single-layer per-call decode GEMVs over distinct copies
    totalling > 4x L2, captured in one graph."""
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
    g = graph_of(ctx, torch, stream, step)
    sec = time_launches(torch, stream, g.launch, reps, 3) / copies
    g.free()
    return {"n": n, "m": m, "r": r, "us": sec * 1e6, "gbs": per / sec / 1e9,
            "frac": per / sec / 1e9 / hbm}


def l70_pass_leg(nq, ctx, torch, stream, hbm, reps=5):
    """BASELINE config 3': a sustained Llama-2-70B decode pass at 0.55 bit, 80 blocks
    of q/k/v (GQA k, v 1024 rows), o, gate/up, down, as one decode-pass launch."""
    steps = workload(nq.rank_for_target_bpw, L70_BLOCK, 80, 0.55, seed=SEED + 70)
    nbytes = step_bytes_of(steps)
    p, ps, keep = build_pass(nq, ctx, torch, steps)
    del steps
    with torch.cuda.stream(stream):
        ctx.bind_torch_stream()
    sec = time_launches(torch, stream, p.launch, reps, 3)
    out = {"workload": "llama2-70b decode pass: 560 linear layers @0.55 bit (80 x q 8192x8192 "
                       "r=2237, k,v 1024x8192 r=485, o, gate,up 28672x8192 r=3488, down 8192x28672 "
                       "r=3488), one decode-pass launch", "us": sec * 1e6,
           "algorithmic_bytes": nbytes, "gbs": nbytes / sec / 1e9, "frac": nbytes / sec / 1e9 / hbm}
    p.free()
    del ps, keep
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def prefill_leg(nq, ctx, torch, stream, tpk, b=2048, reps=10):
    """Prefill GEMM (tcgen05 kind::f16) on the 70B shapes, b tokens, per call."""
    out, arrays = {}, []
    for name, n, m, bpw in L70_SHAPES:
        r = nq.rank_for_target_bpw(n, m, bpw)
        arrs = random_layer_arrays(np.random.default_rng(n * 3 + m), n, m, r)
        lay = nq.DeviceLayer.upload_f16(n, m, r, *arrs, ctx)
        x = torch.randn(b, m, device="cuda", dtype=torch.float16)
        y = torch.empty(b, n, device="cuda", dtype=torch.float16)
        g = graph_of(ctx, torch, stream, lambda: lay.gemm_device(x, y))
        sec = time_launches(torch, stream, g.launch, reps, 3)
        g.free()
        tf = 2.0 * b * r * (n + m) / sec / 1e12
        out[f"{name}_{bpw}_b{b}"] = {"n": n, "m": m, "r": r, "ms": sec * 1e3, "tflops": tf,
                                     "frac_of_bf16_peak": tf / tpk}
        arrays.append((f"{name}_{bpw}_b{b}", n, m, r, arrs))
    return out, arrays


def dgemm_ours(nq, torch, ctx, r=2032, n=4096):
    """Our fp64 DMMA GEMM (dgemm.cu, nqb_dgemm_device) at the ADMM factor-solve
    shapes of 4096^2 r = 2032 (admm.cpp:62-78): the Gram fixed^T fixed (r x r, K = n)
    and the right-hand side fixed^T target^T (r x n, K = n); TF/s of 2MNK."""
    import ctypes as C
    lib = ctx.lib
    out = {}
    stream = torch.cuda.Stream()
    for name, (M, N, K, ta, tb) in {"gram": (r, r, n, True, False),
                                    "rhs": (r, n, n, True, True)}.items():
        a = torch.randn(K, M, device="cuda", dtype=torch.float64)  # op(A) = A^T (M x K)
        b = torch.randn(N, K, device="cuda", dtype=torch.float64) if tb else \
            torch.randn(K, N, device="cuda", dtype=torch.float64)
        c = torch.empty(M, N, device="cuda", dtype=torch.float64)
        ldb = K if tb else N

        def run():
            ctx.bind_torch_stream()
            st = lib.nqb_dgemm_device(ctx.handle, int(ta), int(tb), M, N, K, C.c_double(1.0),
                                      C.c_void_p(a.data_ptr()), M, C.c_void_p(b.data_ptr()), ldb,
                                      C.c_double(0.0), C.c_void_p(c.data_ptr()), N)
            assert st == 0
        sec = time_launches(torch, stream, run, 5, 2)
        out[name] = {"M": M, "N": N, "K": K, "ms": sec * 1e3, "tflops": 2.0 * M * N * K / sec / 1e12}
    torch.cuda.synchronize()
    ctx.set_stream(None)  # the context must not keep this local stream
    return out


def dgemm_peak(torch):
    """Measured FP64 tensor (DMMA) peak on this GPU: cuBLAS DGEMM 8192^3 (the
    denominator of the ADMM iteration-phase roofline; MEASURED_PEAKS.json has no
    FP64 figure)."""
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.float64)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.float64)
    sec = time_launches(torch, torch.cuda.current_stream(), lambda: torch.mm(a, b), 5, 2)
    return 2.0 * 8192 ** 3 / sec / 1e12


def admm_leg(nq, torch, ws, rank, local, hbm, fp64_peak):
    """Whole-model-init throughput sample (BASELINE configs 1 and 4): `ws` Llama-2-7B q
    matrices (4096x4096, W = fp32(0.02 g) from the reference Rng(0x7B000000 + 7b), 1.0
    bpw -> r = 2032), one per rank by the LPT plan, each through nqb_factorize_layer
    (fp64 SVD init + ADMM, reference defaults), packed factors gathered to rank 0."""
    from paper_2602_06694_b200 import sharded as S
    specs = [S.MatrixSpec(f"b{i}.q", 4096, 4096, 0x7B000000 + 7 * i) for i in range(ws)]
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    rep = S.sharded_init(specs, 1.0, device=torch.device("cuda", local))
    wall = time.perf_counter() - t0
    if rank != 0:
        return None
    global admm_layer_for_cpu
    admm_layer_for_cpu = rep.matrices[min(rep.matrices)]
    mats = [rep.matrices[i] for i in sorted(rep.matrices)]
    n = m = 4096
    r = mats[0].r
    pm = mats[0]
    svd_bytes = (pm.svd_power_iters + 2 * pm.svd_steps) * 8.0 * n * m
    flops_iter = 6.0 * n * m * r + 8.0 * (n + m) * r * r + 2.0 / 3.0 * r ** 3
    svd_gbs = svd_bytes / max(pm.seconds_svd, 1e-9) / 1e9
    it_tf = pm.iterations * flops_iter / max(pm.seconds_iter, 1e-9) / 1e12
    return {"matrices": len(specs), "shape": "4096x4096", "bpw": 1.0, "rank": r,
            "seconds_max_rank": max(rep.per_rank_seconds), "seconds_wall_incl_gather": wall,
            "matrices_per_s": len(specs) / wall, "scaling": "weak (one matrix per rank)",
            "rel_error": [p.rel_error for p in mats], "admm_iterations": [p.iterations for p in mats],
            "converged": [p.converged for p in mats],
            "phases": {"svd_init_s": pm.seconds_svd, "svd_power_iterations": pm.svd_power_iters,
                       "svd_deflation_steps": pm.svd_steps, "iterations_s": pm.seconds_iter},
            "roofline": {
                "svd_init": {"bound": "hbm", "achieved": svd_gbs, "peak": hbm, "unit": "GB/s",
                             "frac": svd_gbs / hbm,
                             "bytes": "sum_k (iters_k + 2) * 8nm (one pass over W per power "
                                      "iteration, SURVEY §8(d) row 1)"},
                "iterations": {"bound": "fp64 tensor", "achieved": it_tf, "peak": fp64_peak,
                               "unit": "TFLOP/s", "frac": it_tf / fp64_peak,
                               "flops_per_iteration": flops_iter,
                               "peak_source": "cuBLAS DGEMM 8192^3 measured in this run"}},
            "weights": "W = fp32(0.02 g), g from the reference Rng(0x7B000000 + 7b) (rng.hpp:25-58)",
            "forward": config1_forward(nq, torch, pm)}


def config1_forward(nq, torch, pm, reps=200):
    """BASELINE config 1's batch-1 forward on the layer the ADMM just produced
    (binary16 scales, NQPK precision): x fp32 from Rng(0xB1A5E002) (SURVEY §8(d)
    row 1), the reference-facing drop-in nqb_gemv_f32_host and the device kernel."""
    lay = nq.DeviceLayer.upload_f16(pm.n, pm.m, pm.r, pm.u, pm.v, pm.s1, pm.s2)
    x = nq.synthetic_weight(0xB1A5E002, 1, pm.m, 1.0, snap_f32=True).astype(np.float32).ravel()
    y = lay.gemv_f32(x)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(pm.n, device="cuda", dtype=torch.float32)
    stream = torch.cuda.Stream()
    sec = time_launches(torch, stream, lambda: lay.gemv_device(xd, yd), reps, 10)
    t0 = time.perf_counter()
    for _ in range(50):
        lay.gemv_f32(x, out=y)
    host = (time.perf_counter() - t0) / 50
    nbytes = algo_bytes(pm.n, pm.m, pm.r) + 2 * pm.n  # fp32 x / y
    return {"layer": f"{pm.n}x{pm.m} r={pm.r} from the ADMM above", "device_us": sec * 1e6,
            "device_gbs_l2_resident": nbytes / sec / 1e9, "host_dropin_us": host * 1e6,
            "y": y, "x": x, "note": "one 2.1 MB layer re-read per call stays in L2; the HBM-bound "
                                   "numbers are the pass and per-shape lines"}


def admm_small_gpu(nq, ws_cpu, r):
    """Our device path on the same 256^2 matrices the CPU baseline factorised (W from
    the same Rng seeds): one after another, and `workers` at a time on one GPU (one
    context per worker, each confined to an equal share of the SMs, sharded.run_local)
    -- a 256^2 matrix alone is latency-bound on the per-iteration grid barriers."""
    from paper_2602_06694_b200 import sharded as S
    t0 = time.perf_counter()
    for w in ws_cpu:
        nq.factorize_layer(w, nq.AdmmConfig(rank=r))
    secs = time.perf_counter() - t0
    specs = [S.MatrixSpec(f"w{i}", 256, 256, 0x7B000000 + i) for i in range(len(ws_cpu))]
    out = {"matrices_per_s_256": len(ws_cpu) / secs, "seconds": secs, "matrices": len(ws_cpu)}
    for workers in (4, 8):
        t0 = time.perf_counter()
        S.run_local(specs, list(range(len(specs))), 1.0, workers=workers)
        sec_w = time.perf_counter() - t0
        out[f"concurrent_{workers}"] = {"matrices_per_s_256": len(specs) / sec_w, "seconds": sec_w}
    return out


def reference_arm(args, ws, rank):
    """--impl reference: the unmodified reference library on the host cores, the
    same 224-layer pass per step, all host threads over layers."""
    if rank != 0:
        return
    steps = workload(ref_rank_fn())
    nbytes = step_bytes_of(steps)
    threads = max(1, os.cpu_count() or 1)
    rp = RefPass(steps, threads)
    del steps
    for _ in range(args.warmup):
        rp.run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rp.run()
    secs = time.perf_counter() - t0
    rp.close()
    value = nbytes * args.steps / secs / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference", "config": config_of(args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{args.steps} whole 224-layer decode passes (gemv_packed_f32 "
                                       f"per layer, {threads} host threads over layers), {secs:.1f} s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shapes", action="store_true", help="skip the per-shape sweeps")
    ap.add_argument("--no-70b", action="store_true", help="skip the 70B decode-pass line")
    ap.add_argument("--no-admm", action="store_true",
                    help="skip the ADMM-init leg (one 4096x4096 matrix per rank, ~60 s)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws, rank, local = dist_env()

    if args.impl == "reference":
        reference_arm(args, ws, rank)
        return

    import torch

    import paper_2602_06694_b200 as nq
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = nq.context(local)
    stream = torch.cuda.Stream()
    hbm, tpk, peak_kind = load_peaks()

    steps = workload(nq.rank_for_target_bpw, seed=SEED + rank)
    step_bytes = step_bytes_of(steps)
    with torch.cuda.stream(stream):
        ctx.bind_torch_stream()
        dpass, pass_steps, keep = build_pass(nq, ctx, torch, steps)
        for _ in range(args.warmup):
            dpass.launch()
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    l0 = ctx.kernel_launches
    with Clocks(local) as clk:
        with torch.cuda.stream(stream):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(args.steps):
                dpass.launch()
            e1.record(stream)
            torch.cuda.synchronize()
    launches = ctx.kernel_launches - l0
    secs = e0.elapsed_time(e1) / 1e3
    if ws > 1:
        t = torch.tensor([secs], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        secs = float(t.item())
        torch.distributed.barrier()
    value = ws * step_bytes * args.steps / secs / 1e9

    # ---- e2e: the same pass through the C ABI with host buffers (nqb_pass_run_host):
    #      pinned host x -> device, one pass launch, device -> pinned host y, synchronous ----
    hx = [torch.from_numpy(x).pin_memory().numpy() for _, _, x in steps]
    hy = [torch.empty(l[1], dtype=torch.float16).pin_memory().numpy() for _, ls, _ in steps for l in ls]
    for a in hx + hy:  # explicit registration: no per-call pointer probing
        ctx.register_host(a)
    h2d = sum(x.nbytes for x in hx)
    d2h = sum(y.nbytes for y in hy)
    # a serving loop binds its pinned token buffers once (nqb_pass_io_create) and
    # runs one call per token (nqb_pass_io_run: inputs up, the pass, outputs down)
    hio = dpass.host_io(hx, hy)
    hio.run()
    e2e_steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        hio.run()
    e2e_secs = time.perf_counter() - t0
    hio.close()
    if ws > 1:
        t = torch.tensor([e2e_secs], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_secs = float(t.item())
    e2e = {"value": ws * step_bytes * e2e_steps / e2e_secs / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "api": "nqb_pass_io_run (C ABI; registered pinned host x/y bound once with "
                  "nqb_pass_io_create; per step: one copy kernel up, one decode-pass launch, one "
                  "copy kernel down, synchronous)",
           "steps": e2e_steps}

    extra = {}
    roof, cpu = None, None
    if rank == 0:
        # the reference-facing per-layer drop-in (gemv_packed_f32 -> nqb_gemv_f32_host)
        all_layers = [l for dev, _ in keep for l in dev]
        hxf = [torch.randn(l.m, dtype=torch.float32).pin_memory().numpy() for l in all_layers]
        hyf = [torch.empty(l.n, dtype=torch.float32).pin_memory().numpy() for l in all_layers]
        ctx.set_stream(None)
        for a in hxf + hyf:
            ctx.register_host(a)
        for l, x, y in zip(all_layers, hxf, hyf):
            l.gemv_f32(x, out=y)
        t0 = time.perf_counter()
        for _ in range(2):
            for l, x, y in zip(all_layers, hxf, hyf):
                l.gemv_f32(x, out=y)
        dt = (time.perf_counter() - t0) / 2
        extra["e2e_dropin_per_layer"] = {
            "value": step_bytes / dt / 1e9, "unit": UNIT,
            "api": "nqb_gemv_f32_host per layer (gemv_packed_f32 drop-in, registered pinned fp32 "
                   "host x/y)",
            "h2d_bytes_per_step": sum(4 * l.m for l in all_layers),
            "d2h_bytes_per_step": sum(4 * l.n for l in all_layers)}
        extra["per_call_graph"] = per_call_graph_gbs(nq, ctx, torch, stream, pass_steps, step_bytes)
        achieved = step_bytes * args.steps / secs / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r02c_decode_pass", "traffic.json")
        if os.path.exists(tp):  # ncu dram__bytes_read+write of one launch of this same pass
            traffic = json.load(open(tp))["dram_bytes_per_launch"]
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "traffic_note": "ncu dram bytes of one k_decode_pass launch of this pass "
                                "(profiles/r02c_decode_pass/traffic.json); algorithmic bytes per "
                                "launch = algorithmic_bytes_per_step",
                "peak_source": peak_kind,
                "kernel": "nqb::dec::k_decode_pass (persistent decode pass: one launch per step, "
                          "duration = step time)",
                "algorithmic_bytes_per_step": step_bytes, "launches_per_step": launches / args.steps,
                "us_per_launch": secs / args.steps * 1e6}
    del pass_steps, keep, dpass
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    if rank == 0 and not args.no_70b:
        extra["l70_decode_pass"] = l70_pass_leg(nq, ctx, torch, stream, hbm)
    pref_arrays = None
    if rank == 0 and not args.no_shapes:
        shapes = {}
        for name, n, m, bpw in [("l7_q", 4096, 4096, 0.8), ("l7_gate", 11008, 4096, 0.8),
                                ("l7_down", 4096, 11008, 0.8)] + list(L70_SHAPES):
            r = nq.rank_for_target_bpw(n, m, bpw)
            shapes[f"{name}_{bpw}"] = shape_roofline(nq, ctx, torch, stream, n, m, r, hbm)
        extra["per_shape_single_layer"] = shapes
        # BASELINE config 5: bitrate sweep on Llama-2-13B shapes (decode GB/s; the ADMM
        # reconstruction error vs the CPU reference at these bitrates is pinned by the
        # l13s* fixtures in tests/test_gpu_admm.py)
        sweep = {}
        for name, n, m in [("l13_q", 5120, 5120), ("l13_gate", 13824, 5120),
                           ("l13_down", 5120, 13824)]:
            for bpw in (0.55, 0.8, 1.0):
                r = nq.rank_for_target_bpw(n, m, bpw)
                sweep[f"{name}_{bpw}"] = shape_roofline(nq, ctx, torch, stream, n, m, r, hbm, reps=10)
        extra["bitrate_sweep_l13_decode"] = sweep
        extra["prefill_tcgen05"], pref_arrays = prefill_leg(nq, ctx, torch, stream, tpk)

    admm = None
    if not args.no_admm:
        fp64_peak = dgemm_peak(torch)
        admm = admm_leg(nq, torch, ws, rank, local, hbm, fp64_peak)
        if rank == 0:
            admm["fp64_dgemm_peak_tflops"] = fp64_peak
            ours = dgemm_ours(nq, torch, ctx)
            for v in ours.values():
                v["frac_of_cublas_dgemm_peak"] = v["tflops"] / fp64_peak
            admm["dmma_gemm"] = ours
            extra["admm_init"] = admm

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_pass_baseline(steps, step_bytes, args.cpu_seconds)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": f"error: {e}"}
        try:
            if pref_arrays is not None:
                cp = cpu_prefill_baseline(pref_arrays)
                for k, v in cp.items():
                    extra["prefill_tcgen05"][k]["cpu_baseline"] = v
            if admm is not None:
                fw = admm["forward"]
                pm0 = admm_layer_for_cpu
                O = _oracle()
                ref = O.reference()
                L = O.Layer(pm0.n, pm0.m, pm0.r, pm0.u, pm0.v,
                            pm0.s1.view(np.float16).astype(np.float64),
                            pm0.s2.view(np.float16).astype(np.float64))
                t0 = time.perf_counter()
                yr = ref.gemv_packed_f32(L, fw["x"])
                fw["cpu_baseline"] = {"seconds": time.perf_counter() - t0, "cores": 1,
                                      "kind": "reference", "call": "gemv_packed_f32"}
                fw["rel_error_vs_reference"] = float(np.linalg.norm(fw["y"] - yr) /
                                                     max(np.linalg.norm(yr), 1e-300))
                ca, ws_cpu, r256 = cpu_admm_baseline()
                admm["cpu_baseline"] = ca
                try:
                    ca["gpu_same_256_matrices"] = admm_small_gpu(nq, ws_cpu, r256)
                except Exception as e:  # noqa: BLE001
                    ca["gpu_same_256_matrices"] = {"error": str(e)}
        except Exception as e:  # noqa: BLE001
            extra["cpu_baseline_error"] = str(e)

    if admm is not None and "forward" in admm:
        admm["forward"].pop("x", None)
        admm["forward"].pop("y", None)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u1 x s8-limb IMMA, int32/int64 exact accumulate (fp16 x/y I/O)",
                "data": "synthetic (seeded random sign bits, binary16 scales U(0.25,2), N(0,1) fp16 x)",
                "config": config_of(ws), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk.summary(), "gpu_launches": launches, "extra": extra}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
