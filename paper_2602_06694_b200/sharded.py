"""Layer-sharded whole-model ADMM initialisation (north_star item 4).

Every matrix's initialisation depends only on its own weight when the
preconditioner is the identity (pipeline.cpp:95-110), so a model is sharded by
matrix: one process per GPU, matrices assigned by LPT (longest processing time
first) on the cost model below, each rank runs `nqb_factorize_layer` on its own
matrices, and ONE collective moves the packed factors (u32 sign words +
binary16 scales + per-matrix metrics) to rank 0 (an all-gather, which every
backend supports; rank 0 keeps the result).  There is no other collective on the
data path.  With `torch.distributed` over NCCL the gather crosses NVLink; the
same code runs over gloo for the CPU tests.

The per-rank work function is injectable (`factorize=`) so the collective and
bookkeeping logic is testable without a GPU; the default is the device path.
"""
from __future__ import annotations

import heapq
import struct
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

# Llama-2-7B decoder matrices per block (proj/data/shapes/llama2-7b.shape:3-10)
LLAMA2_7B_BLOCK = [("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
                   ("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]


@dataclass(frozen=True)
class MatrixSpec:
    name: str
    n: int
    m: int
    seed: int


def llama2_7b_specs(blocks: int = 32, seed_base: int = 0x7B000000) -> List[MatrixSpec]:
    """The 224 matrices of Llama-2-7B (W from Rng(0x7B000000 + 7b + p))."""
    out = []
    for b in range(blocks):
        for p, (nm, n, m) in enumerate(LLAMA2_7B_BLOCK):
            out.append(MatrixSpec(f"b{b}.{nm}", n, m, seed_base + 7 * b + p))
    return out


def rank_for(n: int, m: int, bpw: float) -> int:
    """storage.cpp:124-141 (r = llround(t*nm/(n+m) - 16), clamped) — host arithmetic."""
    r = int(np.floor(bpw * n * m / (n + m) - 16 + 0.5))
    return max(1, min(r, min(n, m)))


def cost(spec: MatrixSpec, bpw: float, iters: float = 60.0, svd_iters: float = 1000.0) -> float:
    """Relative device time: SVD init ~ r * svd_iters * n * m (HBM-bound power
    iterations) + ADMM iterations * (6nmr + 8(n+m)r^2)."""
    r = rank_for(spec.n, spec.m, bpw)
    n, m = spec.n, spec.m
    return r * svd_iters * n * m * 8 / 6.5e12 + iters * (6.0 * n * m * r + 8.0 * (n + m) * r * r) / 3e13


def lpt_assign(specs: Sequence[MatrixSpec], world: int, bpw: float) -> List[List[int]]:
    """Longest-processing-time-first assignment; deterministic (ties by index)."""
    order = sorted(range(len(specs)), key=lambda i: (-cost(specs[i], bpw), i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + cost(specs[i], bpw), r))
    for lst in out:
        lst.sort()
    return out


@dataclass
class PackedMatrix:
    """One initialised matrix as it travels to rank 0 (NQPK payload, io.cpp:139-157)."""
    index: int
    n: int
    m: int
    r: int
    u: np.ndarray          # n x ceil(r/32) uint32
    v: np.ndarray          # m x ceil(r/32) uint32
    s1: np.ndarray         # n uint16 (binary16 bits)
    s2: np.ndarray         # m uint16
    rel_error: float = 0.0
    iterations: int = 0
    converged: bool = False
    seconds: float = 0.0
    # phase statistics of the device ADMM (nqb_admm_result)
    svd_steps: int = 0
    svd_power_iters: int = 0
    seconds_svd: float = 0.0
    seconds_iter: float = 0.0

    # index n m r err iters conv secs svd_steps svd_power_iters secs_svd secs_iter
    _HDR = struct.Struct("<IIIIdIIdIQdd")

    def to_bytes(self) -> bytes:
        h = self._HDR.pack(self.index, self.n, self.m, self.r, float(self.rel_error),
                           int(self.iterations), int(self.converged), float(self.seconds),
                           int(self.svd_steps), int(self.svd_power_iters), float(self.seconds_svd),
                           float(self.seconds_iter))
        return h + np.ascontiguousarray(self.u, "<u4").tobytes() + \
            np.ascontiguousarray(self.v, "<u4").tobytes() + \
            np.ascontiguousarray(self.s1, "<u2").tobytes() + np.ascontiguousarray(self.s2, "<u2").tobytes()

    @classmethod
    def from_bytes(cls, buf: memoryview) -> Tuple["PackedMatrix", int]:
        idx, n, m, r, err, iters, conv, secs, ss, spi, tsvd, tit = cls._HDR.unpack_from(buf, 0)
        off = cls._HDR.size
        k = (r + 31) // 32
        u = np.frombuffer(buf, "<u4", n * k, off).reshape(n, k).copy()
        off += 4 * n * k
        v = np.frombuffer(buf, "<u4", m * k, off).reshape(m, k).copy()
        off += 4 * m * k
        s1 = np.frombuffer(buf, "<u2", n, off).copy()
        off += 2 * n
        s2 = np.frombuffer(buf, "<u2", m, off).copy()
        off += 2 * m
        return cls(idx, n, m, r, u, v, s1, s2, err, iters, bool(conv), secs, ss, spi, tsvd, tit), off


def pack_shard(items: Sequence[PackedMatrix]) -> np.ndarray:
    """Concatenates a rank's matrices: [count u32][len u64 per item][items...] as uint8."""
    blobs = [it.to_bytes() for it in items]
    head = struct.pack("<I", len(blobs)) + b"".join(struct.pack("<Q", len(b)) for b in blobs)
    return np.frombuffer(head + b"".join(blobs), np.uint8).copy()


def unpack_shard(buf: np.ndarray) -> List[PackedMatrix]:
    mv = memoryview(np.ascontiguousarray(buf, np.uint8))
    (count,) = struct.unpack_from("<I", mv, 0)
    lens = struct.unpack_from("<" + "Q" * count, mv, 4)
    off = 4 + 8 * count
    out = []
    for ln in lens:
        pm, _ = PackedMatrix.from_bytes(mv[off:off + ln])
        out.append(pm)
        off += ln
    return out


def synthetic_weight(spec: MatrixSpec) -> np.ndarray:
    """W_ij = fp32(0.02 * g), g from the reference Rng(spec.seed) in row-major order,
    promoted to double like NQMX (io.cpp:117-119): SURVEY §8(d) row 4, so the
    reference can regenerate exactly these inputs (nqb_synthetic_weight_host)."""
    from . import nanoquant as nq
    return nq.synthetic_weight(spec.seed, spec.n, spec.m, 0.02)


def device_factorize(spec: MatrixSpec, index: int, bpw: float, max_iters: int = 400,
                     ctx=None) -> PackedMatrix:
    """The product path: one matrix through nqb_factorize_layer on this rank's GPU."""
    import time

    from . import nanoquant as nq
    w = synthetic_weight(spec)
    r = nq.rank_for_target_bpw(spec.n, spec.m, bpw)
    t0 = time.perf_counter()
    lay, err, state = nq.factorize_layer(w, nq.AdmmConfig(rank=r, max_iters=max_iters), ctx=ctx)
    secs = time.perf_counter() - t0
    got = lay.download()
    h1 = got.s1.astype(np.float16).view(np.uint16)
    h2 = got.s2.astype(np.float16).view(np.uint16)
    st = state.stats
    return PackedMatrix(index, spec.n, spec.m, r, got.u, got.v, h1, h2, err, state.iteration,
                        state.converged, secs, int(st.get("svd_steps", 0)),
                        int(st.get("svd_power_iters", 0)), float(st.get("seconds_svd_init", 0.0)),
                        float(st.get("seconds_iterations", 0.0)))


@dataclass
class InitReport:
    matrices: Dict[int, PackedMatrix] = field(default_factory=dict)
    seconds: float = 0.0
    per_rank_seconds: List[float] = field(default_factory=list)
    assignment: List[List[int]] = field(default_factory=list)


def run_local(specs: Sequence[MatrixSpec], indices: Sequence[int], bpw: float,
              factorize: Optional[Callable[[MatrixSpec, int], PackedMatrix]] = None,
              workers: int = 1, device: int = 0) -> List[PackedMatrix]:
    """This rank's matrices.  With workers > 1 (device path), `workers`
    contexts on the same GPU, each confined to 1/workers of the SMs, factorize
    matrices concurrently (ctypes releases the GIL), so the per-iteration grid
    barriers of one matrix overlap the HBM streaming of the others."""
    if factorize is not None or workers <= 1:
        if factorize is None:  # this rank's GPU (one process per GPU)
            from . import nanoquant as nq
            ctx = nq.context(device)
            factorize = lambda s, i: device_factorize(s, i, bpw, ctx=ctx)  # noqa: E731
        return [factorize(specs[i], i) for i in indices]
    from concurrent.futures import ThreadPoolExecutor

    from . import nanoquant as nq
    ctxs = []
    for _ in range(workers):
        c = nq.Context(device)
        ctxs.append(c)
    total = ctxs[0].lib  # noqa: F841 (library loaded)
    import torch
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    for c in ctxs:
        c.set_sm_budget(max(1, sms // workers))
    queue = list(indices)
    out: Dict[int, PackedMatrix] = {}

    def worker(w):
        while True:
            try:
                i = queue.pop(0)
            except IndexError:
                return
            out[i] = device_factorize(specs[i], i, bpw, ctx=ctxs[w])

    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(worker, range(workers)))
    for c in ctxs:
        c.close()
    return [out[i] for i in indices]


def sharded_init(specs: Sequence[MatrixSpec], bpw: float,
                 factorize: Optional[Callable[[MatrixSpec, int], PackedMatrix]] = None,
                 group=None, device=None, workers: int = 1) -> Optional[InitReport]:
    """Runs on every rank of `group` (torch.distributed); returns the full
    report on rank 0 and None elsewhere.  One all-gather of shard sizes and one
    all-gather of the padded byte shards are the only collectives."""
    import time

    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    assign = lpt_assign(specs, world, bpw)
    t0 = time.perf_counter()
    dev_index = device.index if (device is not None and device.type == "cuda") else 0
    mine = run_local(specs, assign[rank], bpw, factorize, workers, dev_index or 0)
    my_secs = time.perf_counter() - t0
    blob = pack_shard(mine)
    if world == 1:
        return InitReport({p.index: p for p in mine}, my_secs, [my_secs], assign)
    dev = device if device is not None else torch.device("cpu")
    size = torch.tensor([blob.size, int(my_secs * 1e6)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    maxlen = int(max(s[0].item() for s in sizes))
    buf = torch.zeros(maxlen, dtype=torch.uint8, device=dev)
    buf[:blob.size] = torch.from_numpy(blob).to(dev)
    # all_gather rather than gather: supported by every backend (NCCL and gloo);
    # the shards are a few MB of packed factors per matrix
    gathered = [torch.zeros(maxlen, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(gathered, buf, group=group)
    if rank != 0:
        return None
    rep = InitReport(assignment=assign)
    for r, (g, s) in enumerate(zip(gathered, sizes)):
        for pm in unpack_shard(g[: int(s[0].item())].cpu().numpy()):
            rep.matrices[pm.index] = pm
        rep.per_rank_seconds.append(s[1].item() / 1e6)
    rep.seconds = max(rep.per_rank_seconds)
    return rep
