"""Host-side mirror of the NanoQuant reference API for the BLR hot path.

Same names, argument meaning and error behaviour as the reference C++ value
API (``namespace nanoquant``), every call executed on the B200 through the C ABI
of libnqb (include/nqb.h):

  packed.hpp:49-102    binarize, pack_signs, unpack_signs, make_factorized_layer,
                       reconstruct_dense, gemv_packed, gemv_packed_f32, gemm_packed
  storage.hpp:82-91    rank_for_target_bpw
  linalg.hpp:35-51     cholesky_solve, top_singular_pair, spectral_norm_estimate,
                       truncated_svd_factors
  admm.hpp:30-85       svid, admm_factor_solve, augmented_lagrangian,
                       admm_factorize, monotone_rho
  balance.hpp:38-41    balance_and_extract_scales
  errors.hpp:25-114    Error and its subclasses (raised from nqb status codes)

Matrices are numpy float64 arrays (the reference DenseMatrix is row-major fp64);
packed sign matrices are uint32 arrays of shape (rows, ceil(cols/32)) in the
reference PackedBitMatrix layout.  There is no CPU path: every function needs
libnqb.so and a B200.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L

# ---------------------------------------------------------------------------
# errors.hpp:25-114
# ---------------------------------------------------------------------------
KIND_VALIDATION = "validation"
KIND_NUMERICAL = "numerical"
KIND_RUNTIME = "runtime"


class Error(RuntimeError):
    """nanoquant::Error; `kind` is validation / numerical (CLI exit 2 / 3)."""

    kind = KIND_VALIDATION
    code = 9

    def __init__(self, what: str = "", code: Optional[int] = None):
        super().__init__(what)
        if code is not None:
            self.code = code


class DimensionMismatch(Error):
    code = 1


class NonFiniteInput(Error):
    code = 2


class NonBinaryEntry(Error):
    code = 3


class CorruptPadding(Error):
    code = 4


class RankTooLarge(Error):
    code = 5


class InvalidRank(Error):
    code = 6


class NotSymmetric(Error):
    code = 7


class TargetTooSmall(Error):
    code = 8


class ParseError(Error):
    code = 10


class IoError(Error):
    code = 11


class EmptyStats(Error):
    code = 12


class ZeroMatrix(Error):
    kind = KIND_NUMERICAL
    code = 32


class NotPositiveDefinite(Error):
    kind = KIND_NUMERICAL
    code = 33


class NonFiniteLoss(Error):  # refine.hpp:72-77; best_chain is the checkpoint written back
    kind = KIND_NUMERICAL
    code = 34


class DeviceError(Error):
    """CUDA / allocation / missing-device failures (no reference counterpart)."""

    kind = KIND_RUNTIME
    code = 64


_BY_CODE = {cls.code: cls for cls in (DimensionMismatch, NonFiniteInput, NonBinaryEntry,
                                       CorruptPadding, RankTooLarge, InvalidRank,
                                       NotSymmetric, TargetTooSmall, ParseError, IoError, EmptyStats,
                                       ZeroMatrix, NotPositiveDefinite, NonFiniteLoss)}


def _check(status: int, where: str):
    if status == 0:
        return
    msg = L.load().nqb_last_error().decode(errors="replace")
    cls = _BY_CODE.get(status)
    if cls is None:
        cls = Error if status == 9 else DeviceError
    raise cls(f"{where}: {msg}", code=status)


# ---------------------------------------------------------------------------
# Context
# ---------------------------------------------------------------------------
class Context:
    """One device, one stream, the library's workspaces (nqb_context)."""

    def __init__(self, device: int = 0):
        self.lib = L.load()
        h = C.c_void_p()
        _check(self.lib.nqb_create(device, C.byref(h)), "nqb_create")
        self.handle = h
        self.device = device
        self._stream = 0

    def register_host(self, arr) -> None:
        """nqb_host_register: page-locks (if needed) and maps a host numpy array for the
        _host entry points; keep the array alive until unregister_host."""
        _check(self.lib.nqb_host_register(self.handle, C.c_void_p(arr.ctypes.data), arr.nbytes),
               "nqb_host_register")

    def unregister_host(self, arr) -> None:
        _check(self.lib.nqb_host_unregister(self.handle, C.c_void_p(arr.ctypes.data)),
               "nqb_host_unregister")

    def close(self):
        if self.handle:
            self.lib.nqb_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        stream_ptr = stream_ptr or 0
        if stream_ptr == self._stream:
            return
        _check(self.lib.nqb_set_stream(self.handle, C.c_void_p(stream_ptr)), "nqb_set_stream")
        self._stream = stream_ptr

    def bind_torch_stream(self, device=None):
        """Run library work on torch's current stream.  torch's default stream is
        the legacy NULL stream; it is passed as cudaStreamLegacy (0x1) so the
        library never silently falls back to its own unsynchronised stream."""
        import torch
        self.set_stream(torch.cuda.current_stream(device).cuda_stream or 1)

    def set_sm_budget(self, sms: int):
        """Confine this context's persistent ADMM kernels to `sms` SMs (0: all)."""
        _check(self.lib.nqb_set_sm_budget(self.handle, int(sms)), "nqb_set_sm_budget")

    def set_pdl(self, enable: bool):
        """Programmatic Dependent Launch for decode kernels (default on)."""
        _check(self.lib.nqb_set_pdl(self.handle, 1 if enable else 0), "nqb_set_pdl")

    def capture(self):
        """Context manager capturing the context stream's work into a Graph."""
        return _Capture(self)

    def synchronize(self):
        _check(self.lib.nqb_synchronize(self.handle), "nqb_synchronize")

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.nqb_kernel_launches(self.handle))


class Graph:
    """A captured sequence of library calls, replayed with one launch (nqb_graph)."""

    def __init__(self, ctx: "Context", handle: C.c_void_p):
        self.ctx = ctx
        self.handle = handle

    def launch(self):
        _check(self.ctx.lib.nqb_graph_launch(self.ctx.handle, self.handle), "nqb_graph_launch")

    def free(self):
        if self.handle:
            self.ctx.lib.nqb_graph_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class _Capture:
    def __init__(self, ctx):
        self.ctx = ctx
        self.graph = None

    def __enter__(self):
        _check(self.ctx.lib.nqb_graph_begin(self.ctx.handle), "nqb_graph_begin")
        return self

    def __exit__(self, exc_type, exc, tb):
        h = C.c_void_p()
        st = self.ctx.lib.nqb_graph_end(self.ctx.handle, C.byref(h))
        if exc_type is None:
            _check(st, "nqb_graph_end")
            self.graph = Graph(self.ctx, h)
        return False


_CONTEXTS: dict = {}


def context(device: int = 0) -> Context:
    if device not in _CONTEXTS:
        _CONTEXTS[device] = Context(device)
    return _CONTEXTS[device]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _mat(a) -> np.ndarray:
    a = _f64(a)
    if a.ndim != 2:
        raise DimensionMismatch("expected a 2-D matrix")
    return a


def words_per_row(cols: int) -> int:
    return (cols + 31) // 32


# ---------------------------------------------------------------------------
# storage.cpp:124-141
# ---------------------------------------------------------------------------
def rank_for_target_bpw(n: int, m: int, target_bpw: float) -> int:
    out = C.c_uint32()
    _check(L.load().nqb_rank_for_target_bpw(n, m, float(target_bpw), C.byref(out)),
           "rank_for_target_bpw")
    return out.value


def synthetic_weight(seed: int, n: int, m: int, scale: float = 0.02,
                     snap_f32: bool = True) -> np.ndarray:
    """W (n x m fp64, row-major) = fp32(scale * Rng(seed).gaussian()) per entry in
    stream order (rng.hpp:25-58), generated on the host
    by libnqb with the reference's splitmix64 / Box-Muller stream."""
    out = np.empty((n, m), dtype=np.float64)
    _check(L.load().nqb_synthetic_weight_host(int(seed) & 0xFFFFFFFFFFFFFFFF, n * m, float(scale),
                                              1 if snap_f32 else 0, _ptr(out)),
           "synthetic_weight")
    return out


# ---------------------------------------------------------------------------
# packed.hpp
# ---------------------------------------------------------------------------
def binarize(latent, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or context()
    x = _f64(latent)
    out = np.empty_like(x)
    _check(ctx.lib.nqb_binarize(ctx.handle, _ptr(x), x.size, _ptr(out), 0), "binarize")
    return out


def pack_signs(signs, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or context()
    s = _mat(signs)
    rows, cols = s.shape
    words = np.zeros((rows, words_per_row(cols)), np.uint32)
    _check(ctx.lib.nqb_pack_signs(ctx.handle, _ptr(s), rows, cols, _ptr(words), 0),
           "pack_signs")
    return words


def unpack_signs(words, rows: int, cols: int, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or context()
    w = _u32(words)
    if w.size != rows * words_per_row(cols):
        raise DimensionMismatch("unpack_signs: word count mismatch")
    out = np.empty((rows, cols), np.float64)
    _check(ctx.lib.nqb_unpack_signs(ctx.handle, _ptr(w), rows, cols, _ptr(out), 0),
           "unpack_signs")
    return out


@dataclass
class FactorizedLayer:
    """FactorizedLayer (packed.hpp:57-72): packed U (n x r), V (m x r), s1, s2.

    The device copy (re-laid-out, binary16 scales) is created on first use and
    cached; `device_layer()` returns it.
    """

    n: int
    m: int
    r: int
    u: np.ndarray
    v: np.ndarray
    s1: np.ndarray
    s2: np.ndarray
    _dev: Optional["DeviceLayer"] = field(default=None, repr=False, compare=False)

    def payload_bits(self) -> int:  # packed.hpp:65-68
        return self.r * (self.n + self.m) + 16 * (self.n + self.m)

    def device_layer(self, ctx: Context | None = None) -> "DeviceLayer":
        if self._dev is None:
            self._dev = DeviceLayer.upload(self, ctx)
        return self._dev


class DeviceLayer:
    """A factorized layer resident in HBM (nqb_layer)."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.handle = handle
        n, m, r = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(ctx.lib.nqb_layer_shape(handle, C.byref(n), C.byref(m), C.byref(r)),
               "nqb_layer_shape")
        self.n, self.m, self.r = n.value, m.value, r.value

    @classmethod
    def upload(cls, layer: FactorizedLayer, ctx: Context | None = None) -> "DeviceLayer":
        ctx = ctx or context()
        h = C.c_void_p()
        u, v = _u32(layer.u), _u32(layer.v)
        s1, s2 = _f64(layer.s1), _f64(layer.s2)
        if u.size != layer.n * words_per_row(layer.r) or v.size != layer.m * words_per_row(
                layer.r) or s1.size != layer.n or s2.size != layer.m:
            raise DimensionMismatch("layer arrays do not match (n, m, r)")
        _check(ctx.lib.nqb_layer_upload(ctx.handle, layer.n, layer.m, layer.r, _ptr(u),
                                        _ptr(v), _ptr(s1), _ptr(s2), C.byref(h)),
               "nqb_layer_upload")
        return cls(ctx, h)

    @classmethod
    def upload_f16(cls, n, m, r, u, v, s1_half, s2_half, ctx: Context | None = None):
        ctx = ctx or context()
        h = C.c_void_p()
        u, v = _u32(u), _u32(v)
        s1h = np.ascontiguousarray(s1_half, dtype=np.uint16)
        s2h = np.ascontiguousarray(s2_half, dtype=np.uint16)
        _check(ctx.lib.nqb_layer_upload_f16(ctx.handle, n, m, r, _ptr(u), _ptr(v), _ptr(s1h),
                                            _ptr(s2h), C.byref(h)), "nqb_layer_upload_f16")
        return cls(ctx, h)

    def free(self):
        if self.handle:
            self.ctx.lib.nqb_layer_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        return int(self.ctx.lib.nqb_layer_device_bytes(self.handle))

    def download(self) -> FactorizedLayer:
        k = words_per_row(self.r)
        u = np.zeros((self.n, k), np.uint32)
        v = np.zeros((self.m, k), np.uint32)
        s1, s2 = np.empty(self.n), np.empty(self.m)
        _check(self.ctx.lib.nqb_layer_download(self.ctx.handle, self.handle, _ptr(u), _ptr(v),
                                               _ptr(s1), _ptr(s2)), "nqb_layer_download")
        return FactorizedLayer(self.n, self.m, self.r, u, v, s1, s2)

    # -- forward on host buffers (drop-in) --------------------------------
    def gemv_f32(self, x, out: Optional[np.ndarray] = None) -> np.ndarray:
        """gemv_packed_f32 (packed.cpp:201-204).  `out` (contiguous float32, n) is
        written in place when given, e.g. a pinned buffer."""
        # per-token path: keep the Python side thin (raw addresses, cached entry point)
        if type(x) is not np.ndarray or x.dtype != np.float32 or not x.flags.c_contiguous:
            x = np.ascontiguousarray(x, dtype=np.float32)
        if x.size != self.m:
            raise DimensionMismatch("gemv_packed: |x| != m")
        if out is None:
            y = np.empty(self.n, np.float32)
        else:
            if out.dtype != np.float32 or out.size != self.n or not out.flags.c_contiguous:
                raise DimensionMismatch("gemv_packed: out must be contiguous float32 of size n")
            y = out
        st = self.ctx.lib.nqb_gemv_f32_host(self.ctx.handle, self.handle, x.ctypes.data, y.ctypes.data)
        if st:
            _check(st, "gemv_packed_f32")
        return y

    def gemv_f64(self, x) -> np.ndarray:
        x = _f64(x)
        if x.size != self.m:
            raise DimensionMismatch("gemv_packed: |x| != m")
        y = np.empty(self.n, np.float64)
        _check(self.ctx.lib.nqb_gemv_f64_host(self.ctx.handle, self.handle, _ptr(x), _ptr(y)),
               "gemv_packed")
        return y

    def gemm_f64(self, x) -> np.ndarray:
        x = _mat(x)
        if x.shape[0] != self.m:
            raise DimensionMismatch("gemm_packed: rows(X) != m")
        y = np.empty((self.n, x.shape[1]), np.float64)
        _check(self.ctx.lib.nqb_gemm_f64_host(self.ctx.handle, self.handle, _ptr(x),
                                              x.shape[1], _ptr(y)), "gemm_packed")
        return y

    def reconstruct_dense(self) -> np.ndarray:
        w = np.empty((self.n, self.m), np.float64)
        _check(self.ctx.lib.nqb_reconstruct_dense_host(self.ctx.handle, self.handle, _ptr(w)),
               "reconstruct_dense")
        return w

    def rel_error(self, w) -> float:
        w = _mat(w)
        out = C.c_double()
        _check(self.ctx.lib.nqb_layer_rel_error(self.ctx.handle, self.handle, _ptr(w), 0,
                                                C.byref(out)), "nqb_layer_rel_error")
        return out.value

    # -- forward on device buffers (torch tensors; the hot path) -----------
    def _bind_stream(self, tensor):
        import torch
        self.ctx.bind_torch_stream(tensor.device)

    def gemv_device(self, x, y):
        """x: (m,) fp32/fp16 CUDA tensor, y: (n,) same dtype; async on torch's stream."""
        import torch
        _check_device_io(x, self.m, y, self.n, "gemv_device")
        self._bind_stream(x)
        if x.dtype == torch.float32:
            fn = self.ctx.lib.nqb_gemv_f32_device
        elif x.dtype == torch.float16:
            fn = self.ctx.lib.nqb_gemv_f16_device
        else:
            raise Error("gemv_device: dtype must be float32 or float16")
        _check(fn(self.ctx.handle, self.handle, C.c_void_p(x.data_ptr()),
                  C.c_void_p(y.data_ptr())), "gemv_device")

    def gemm_device(self, x, y):
        """x: (b, m) fp16 token-major CUDA tensor -> y: (b, n) fp16."""
        import torch
        if x.dim() != 2 or y.dim() != 2 or x.shape[0] != y.shape[0]:
            raise DimensionMismatch("gemm_packed: x must be (b, m) and y (b, n)")
        if x.dtype != torch.float16:
            raise Error("gemm_device: dtype must be float16")
        _check_device_io(x, x.shape[0] * self.m, y, y.shape[0] * self.n, "gemm_device")
        self._bind_stream(x)
        _check(self.ctx.lib.nqb_gemm_f16_device(self.ctx.handle, self.handle,
                                                C.c_void_p(x.data_ptr()), x.shape[0],
                                                C.c_void_p(y.data_ptr())), "gemm_device")


def _check_device_io(x, nx, y, ny, what):
    """Device-buffer entry points write through raw pointers: check sizes, dtypes,
    contiguity and device first (the reference throws DimensionMismatch)."""
    if x.numel() != nx or y.numel() != ny:
        raise DimensionMismatch(f"{what}: |x| = {x.numel()} (want {nx}), |y| = {y.numel()} "
                                f"(want {ny})")
    if x.dtype != y.dtype:
        raise Error(f"{what}: x and y dtypes differ ({x.dtype} vs {y.dtype})")
    if not (x.is_contiguous() and y.is_contiguous()):
        raise Error(f"{what}: x and y must be contiguous")
    if not (x.is_cuda and y.is_cuda) or x.device != y.device:
        raise Error(f"{what}: x and y must be CUDA tensors on the same device")


class DecodeGroup:
    """1..4 device layers that read the same input (q/k/v, gate/up): one fused
    decode launch computes all of them (nqb_group)."""

    def __init__(self, layers, ctx: Context | None = None):
        ctx = ctx or layers[0].ctx
        self.ctx = ctx
        self.layers = list(layers)
        arr = (C.c_void_p * len(self.layers))(*[lay.handle for lay in self.layers])
        h = C.c_void_p()
        _check(ctx.lib.nqb_group_create(ctx.handle, arr, len(self.layers), C.byref(h)),
               "nqb_group_create")
        self.handle = h
        self.m = self.layers[0].m

    @property
    def stream_bytes(self) -> int:
        return int(self.ctx.lib.nqb_group_stream_bytes(self.handle))

    def free(self):
        if self.handle:
            self.ctx.lib.nqb_group_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def gemv_device(self, x, ys):
        """x: (m,) fp16/fp32 CUDA tensor; ys: one (n_i,) tensor per layer, same dtype."""
        import torch
        if len(ys) != len(self.layers):
            raise DimensionMismatch(f"group gemv: {len(ys)} outputs for {len(self.layers)} layers")
        for lay, y in zip(self.layers, ys):
            _check_device_io(x, self.m, y, lay.n, "group gemv")
        self.ctx.bind_torch_stream(x.device)
        arr = (C.c_void_p * len(ys))(*[y.data_ptr() for y in ys])
        if x.dtype == torch.float16:
            fn = self.ctx.lib.nqb_group_gemv_f16_device
        elif x.dtype == torch.float32:
            fn = self.ctx.lib.nqb_group_gemv_f32_device
        else:
            raise Error("gemv_device: dtype must be float32 or float16")
        _check(fn(self.ctx.handle, self.handle, C.c_void_p(x.data_ptr()), arr), "group gemv")


class PassHostIO:
    """Host buffers bound to a DecodePass (nqb_pass_io_create); run() is one pass
    end to end (inputs up, the pass, outputs down, synchronous)."""

    def __init__(self, dpass, xs, ys):
        self.dpass, self.ctx = dpass, dpass.ctx
        ny = sum(len(k[2]) for k in dpass._keep)
        if len(xs) != dpass.steps or len(ys) != ny:
            raise DimensionMismatch(f"host_io: {len(xs)} inputs / {len(ys)} outputs for "
                                    f"{dpass.steps} steps / {ny} layers")
        for (unit, x, outs), hxk in zip(dpass._keep, xs):
            if hxk is not None and hxk.nbytes != x.numel() * x.element_size():
                raise DimensionMismatch("host_io: host input size differs from the step input")
        self._arrays = (list(xs), list(ys))  # keep the buffers alive while bound
        hx = (C.c_void_p * len(xs))(*[None if x is None else x.ctypes.data for x in xs])
        hy = (C.c_void_p * ny)(*[None if y is None else y.ctypes.data for y in ys])
        h = C.c_void_p()
        _check(self.ctx.lib.nqb_pass_io_create(self.ctx.handle, dpass.handle, hx, hy, C.byref(h)),
               "nqb_pass_io_create")
        self.handle = h

    def run(self):
        _check(self.ctx.lib.nqb_pass_io_run(self.ctx.handle, self.handle), "nqb_pass_io_run")

    def close(self):
        if getattr(self, "handle", None):
            self.ctx.lib.nqb_pass_io_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class DecodePass:
    """A whole decode pass as ONE launch of the persistent decode-pass kernel
    (nqb_pass).  `steps` is a list of (group_or_layer, x, ys):
    a DecodeGroup or DeviceLayer, its input tensor and one output tensor per
    layer.  All tensors are CUDA tensors of one dtype (fp16 or fp32) that stay
    allocated while the pass lives; a step whose x overlaps an earlier step's
    output waits for it inside the kernel."""

    def __init__(self, steps, ctx: Context | None = None):
        import torch
        if not steps:
            raise Error("DecodePass: no steps")
        ctx = ctx or steps[0][0].ctx
        self.ctx = ctx
        self._keep = []
        arr = (L.PassStep * len(steps))()
        for i, (unit, x, ys) in enumerate(steps):
            layers = unit.layers if isinstance(unit, DecodeGroup) else [unit]
            if len(ys) != len(layers):
                raise DimensionMismatch(f"pass step {i}: {len(ys)} outputs for {len(layers)} "
                                        "layers")
            for lay, y in zip(layers, ys):
                _check_device_io(x, layers[0].m, y, lay.n, f"pass step {i}")
            if x.dtype not in (torch.float16, torch.float32):
                raise Error("DecodePass: dtype must be float16 or float32")
            st = arr[i]
            if isinstance(unit, DecodeGroup):
                st.group = unit.handle
            else:
                st.layer = unit.handle
            st.d_x = x.data_ptr()
            for q, y in enumerate(ys):
                st.d_y[q] = y.data_ptr()
            st.f32 = 1 if x.dtype == torch.float32 else 0
            self._keep.append((unit, x, list(ys)))
        h = C.c_void_p()
        _check(ctx.lib.nqb_pass_create(ctx.handle, len(steps), arr, C.byref(h)),
               "nqb_pass_create")
        self.handle = h
        self.steps = len(steps)

    @property
    def stream_bytes(self) -> int:
        return int(self.ctx.lib.nqb_pass_stream_bytes(self.handle))

    @property
    def algorithmic_bytes(self) -> int:
        return int(self.ctx.lib.nqb_pass_algorithmic_bytes(self.handle))

    def run_host(self, xs, ys):
        """One pass end to end through nqb_pass_run_host: xs[k] (numpy, or None
        to keep step k's device input) -> device, the pass, device -> ys (numpy
        arrays, one per layer of every step in step order, or None); returns
        when the outputs are on the host.  Runs on the context's own stream."""
        hx = (C.c_void_p * self.steps)(*[None if x is None else x.ctypes.data for x in xs])
        ny = sum(len(k[2]) for k in self._keep)
        if len(ys) != ny:
            raise DimensionMismatch(f"run_host: {len(ys)} outputs for {ny} layers")
        for (unit, x, outs), hxk in zip(self._keep, xs):
            if hxk is not None and hxk.nbytes != x.numel() * x.element_size():
                raise DimensionMismatch("run_host: host input size differs from the step input")
        hy = (C.c_void_p * ny)(*[None if y is None else y.ctypes.data for y in ys])
        _check(self.ctx.lib.nqb_pass_run_host(self.ctx.handle, self.handle, hx, hy),
               "nqb_pass_run_host")

    def host_io(self, xs, ys):
        """Binds page-locked (pinned or registered) host buffers once, like
        run_host's arguments; the returned PassHostIO.run() then moves the inputs,
        runs the pass and moves the outputs with no per-call host work
        (nqb_pass_io_*)."""
        return PassHostIO(self, xs, ys)

    def launch(self):
        """Enqueues the pass on torch's current stream."""
        self.ctx.bind_torch_stream(self._keep[0][1].device)
        _check(self.ctx.lib.nqb_pass_launch(self.ctx.handle, self.handle), "nqb_pass_launch")

    def trace(self):
        """One launch with per-CTA %globaltimer stamps -> (grid, 24K+2) uint64 array:
        [CTA start, per step (stage-1 start, stage-1 end, t ready, stage-2 end,
        t barrier seen by the t loader, x staged by the x stager, stage-1 first
        chunk landed, x quantised, stage-1 MMA done, t quantised, stage-2 MMA
        done, producer issued stage 1, t loader got its slot, t copy issued, producer started / finished stage 2),
        16/17 ns warp 0 of each stage group waited for chunks, 18/19 its chunks),
        end]; stamp 6 = producer finished stage 1."""
        self.ctx.bind_torch_stream(self._keep[0][1].device)
        g = C.c_uint32()
        per = 24 * self.steps + 2
        out = np.zeros(160 * per, np.uint64)
        _check(self.ctx.lib.nqb_debug_pass_trace(self.ctx.handle, self.handle, _ptr(out),
                                                 C.byref(g)), "nqb_debug_pass_trace")
        return out[: g.value * per].reshape(g.value, per)

    def free(self):
        if getattr(self, "handle", None):
            self.ctx.lib.nqb_pass_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def make_factorized_layer(latent_u, latent_v, s1, s2, ctx: Context | None = None):
    """packed.cpp:105-124: binarize + pack both latents on the device."""
    ctx = ctx or context()
    lu, lv = _mat(latent_u), _mat(latent_v)
    if lu.shape[1] != lv.shape[1]:
        raise DimensionMismatch("make_factorized_layer: ranks differ")
    s1, s2 = _f64(s1).ravel(), _f64(s2).ravel()
    if s1.size != lu.shape[0] or s2.size != lv.shape[0]:
        raise DimensionMismatch("make_factorized_layer: scale lengths")
    r = lu.shape[1]
    u = np.zeros((lu.shape[0], words_per_row(r)), np.uint32)
    v = np.zeros((lv.shape[0], words_per_row(r)), np.uint32)
    _check(ctx.lib.nqb_pack_latent(ctx.handle, _ptr(lu), lu.shape[0], r, _ptr(u), 0),
           "make_factorized_layer")
    _check(ctx.lib.nqb_pack_latent(ctx.handle, _ptr(lv), lv.shape[0], r, _ptr(v), 0),
           "make_factorized_layer")
    return FactorizedLayer(lu.shape[0], lv.shape[0], r, u, v, s1, s2)


def reconstruct_dense(layer: FactorizedLayer, ctx: Context | None = None) -> np.ndarray:
    return layer.device_layer(ctx).reconstruct_dense()


def gemv_packed(layer: FactorizedLayer, x, ctx: Context | None = None) -> np.ndarray:
    return layer.device_layer(ctx).gemv_f64(x)


def gemv_packed_f32(layer: FactorizedLayer, x, ctx: Context | None = None) -> np.ndarray:
    return layer.device_layer(ctx).gemv_f32(x)


def gemm_packed(layer: FactorizedLayer, x, ctx: Context | None = None) -> np.ndarray:
    return layer.device_layer(ctx).gemm_f64(x)


def relative_frobenius_error(reference, approx) -> float:
    """dense.cpp:141-146 (host arithmetic on already-computed matrices)."""
    reference, approx = _mat(reference), _mat(approx)
    denom = float(np.sqrt(np.sum(reference * reference)))
    d = reference - approx
    num = float(np.sqrt(np.sum(d * d)))
    if denom == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / denom


# ---------------------------------------------------------------------------
# linalg.hpp / admm.hpp / balance.hpp
# ---------------------------------------------------------------------------
@dataclass
class SingularPair:  # linalg.hpp:27-32
    sigma: float
    left: np.ndarray
    right: np.ndarray
    converged: bool


def top_singular_pair(m, max_iters: int = 500, tol: float = 1e-12,
                      ctx: Context | None = None) -> SingularPair:
    ctx = ctx or context()
    a = _mat(m)
    rows, cols = a.shape
    sigma, conv = C.c_double(), C.c_int32()
    left, right = np.empty(rows), np.empty(cols)
    _check(ctx.lib.nqb_top_singular_pair_host(ctx.handle, _ptr(a), rows, cols, max_iters, tol,
                                              C.byref(sigma), _ptr(left), _ptr(right),
                                              C.byref(conv)), "top_singular_pair")
    return SingularPair(sigma.value, left, right, bool(conv.value))


def spectral_norm_estimate(m, iters: int = 200, ctx: Context | None = None) -> float:
    ctx = ctx or context()
    a = _mat(m)
    out = C.c_double()
    _check(ctx.lib.nqb_spectral_norm_host(ctx.handle, _ptr(a), a.shape[0], a.shape[1], iters,
                                          C.byref(out)), "spectral_norm_estimate")
    return out.value


def truncated_svd_factors(m, rank: int, ctx: Context | None = None):
    ctx = ctx or context()
    a = _mat(m)
    u = np.empty((a.shape[0], rank))
    v = np.empty((a.shape[1], rank))
    _check(ctx.lib.nqb_truncated_svd_host(ctx.handle, _ptr(a), a.shape[0], a.shape[1], rank,
                                          _ptr(u), _ptr(v)), "truncated_svd_factors")
    return u, v


def cholesky_solve(a, b, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or context()
    a, b = _mat(a), _mat(b)
    if a.shape[0] != a.shape[1]:
        raise DimensionMismatch("cholesky_solve: A is not square")
    if a.shape[0] != b.shape[0]:
        raise DimensionMismatch("cholesky_solve: rows(B) != rows(A)")
    x = np.empty_like(b)
    _check(ctx.lib.nqb_cholesky_solve_host(ctx.handle, _ptr(a), a.shape[0], _ptr(b),
                                           b.shape[1], _ptr(x)), "cholesky_solve")
    return x


def svid(p, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or context()
    a = _mat(p)
    z = np.empty_like(a)
    _check(ctx.lib.nqb_svid_host(ctx.handle, _ptr(a), a.shape[0], a.shape[1], _ptr(z)), "svid")
    return z


def admm_factor_solve(target, fixed, z, l, rho: float, ridge: float,
                      ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or context()
    target, fixed, z, l = map(_mat, (target, fixed, z, l))
    r = fixed.shape[1]
    if z.shape[1] != r or l.shape[1] != r:
        raise DimensionMismatch("admm_factor_solve: proxy rank mismatch")
    if z.shape[0] != target.shape[0] or l.shape[0] != target.shape[0]:
        raise DimensionMismatch("admm_factor_solve: proxy rows mismatch")
    if fixed.shape[0] != target.shape[1]:
        raise DimensionMismatch("admm_factor_solve: rows(fixed) != cols(target)")
    x = np.empty((target.shape[0], r))
    _check(ctx.lib.nqb_admm_factor_solve_host(ctx.handle, _ptr(target), target.shape[0],
                                              target.shape[1], _ptr(fixed), r, _ptr(z), _ptr(l),
                                              rho, ridge, _ptr(x)), "admm_factor_solve")
    return x


@dataclass
class AdmmConfig:  # admm.hpp:41-51
    rank: int = 1
    max_iters: int = 400
    rho_start: float = 0.0
    rho_end: float = 0.0
    ridge: float = 1e-4
    tol: float = 1e-4
    seed: int = 0
    record_trace: bool = True

    def c(self) -> L.AdmmConfig:
        return L.AdmmConfig(self.rank, self.max_iters, self.rho_start, self.rho_end, self.ridge,
                            self.tol, self.seed, 1 if self.record_trace else 0, 0)


@dataclass
class AdmmState:  # admm.hpp:53-62 (scalars; matrices stay on the device)
    rho: float
    iteration: int
    lagrangian_trace: list
    primal_residual: float
    converged: bool
    stats: dict


@dataclass
class AdmmResult:  # admm.hpp:69-73
    state: AdmmState
    consensus_u: np.ndarray
    consensus_v: np.ndarray


def admm_factorize(target, config: AdmmConfig, ctx: Context | None = None) -> AdmmResult:
    ctx = ctx or context()
    w = _mat(target)
    n, m = w.shape
    cfg = config.c()
    cu = np.empty((n, config.rank))
    cv = np.empty((m, config.rank))
    trace = np.empty(max(config.max_iters, 1) + 1)
    res = L.AdmmResultC()
    _check(ctx.lib.nqb_admm_factorize_host(ctx.handle, _ptr(w), n, m, C.byref(cfg), _ptr(cu),
                                           _ptr(cv), _ptr(trace), C.byref(res)),
           "admm_factorize")
    d = res.as_dict()
    state = AdmmState(res.rho, res.iteration, list(trace[: res.trace_len]),
                      res.primal_residual, bool(res.converged), d)
    return AdmmResult(state, cu, cv)


def augmented_lagrangian(u, v, z_u, z_v, l_u, l_v, rho, target, ridge,
                         ctx: Context | None = None) -> float:
    ctx = ctx or context()
    u, v, z_u, z_v, l_u, l_v, target = map(_mat, (u, v, z_u, z_v, l_u, l_v, target))
    if u.shape[0] != target.shape[0] or v.shape[0] != target.shape[1]:
        raise DimensionMismatch("augmented_lagrangian: state does not match target")
    out = C.c_double()
    _check(ctx.lib.nqb_augmented_lagrangian_host(ctx.handle, _ptr(u), _ptr(v), _ptr(z_u),
                                                 _ptr(z_v), _ptr(l_u), _ptr(l_v), u.shape[0],
                                                 v.shape[0], u.shape[1], rho, _ptr(target),
                                                 ridge, C.byref(out)), "augmented_lagrangian")
    return out.value


def monotone_rho(target, ctx: Context | None = None) -> float:
    """admm.cpp:98-100."""
    return 16.0 * max(spectral_norm_estimate(target, ctx=ctx), 1e-12)


@dataclass
class BalancedLatents:  # balance.hpp:28-34
    latent_u: np.ndarray
    latent_v: np.ndarray
    s1: np.ndarray
    s2: np.ndarray
    eta: float


def balance_and_extract_scales(consensus_u, consensus_v, diag_out=None, diag_in=None,
                               scale_floor: float = 1e-12,
                               ctx: Context | None = None) -> BalancedLatents:
    ctx = ctx or context()
    pu, pv = _mat(consensus_u), _mat(consensus_v)
    n, r = pu.shape
    m = pv.shape[0]
    if diag_out is not None and len(diag_out) not in (0, n):
        raise DimensionMismatch("balance: rows(P_U) != |diag_out|")
    if diag_in is not None and len(diag_in) not in (0, m):
        raise DimensionMismatch("balance: rows(P_V) != |diag_in|")
    if pv.shape[1] != r:
        raise DimensionMismatch("balance: factor ranks differ")
    do = _f64(diag_out) if diag_out is not None and len(diag_out) else None
    di = _f64(diag_in) if diag_in is not None and len(diag_in) else None
    lu, lv = np.empty_like(pu), np.empty_like(pv)
    s1, s2 = np.empty(n), np.empty(m)
    eta = C.c_double()
    _check(ctx.lib.nqb_balance_host(ctx.handle, _ptr(pu), _ptr(pv), n, m, r, _ptr(do),
                                    _ptr(di), scale_floor, _ptr(lu), _ptr(lv), _ptr(s1),
                                    _ptr(s2), C.byref(eta)), "balance_and_extract_scales")
    return BalancedLatents(lu, lv, s1, s2, eta.value)


def factorize_layer(w, config: AdmmConfig, scale_floor: float = 1e-12,
                    ctx: Context | None = None):
    """One matrix through pipeline.cpp:95-110 + :150-153 on the device.

    Returns (DeviceLayer, rel_fro_error, AdmmState)."""
    ctx = ctx or context()
    w = _mat(w)
    n, m = w.shape
    cfg = config.c()
    h = C.c_void_p()
    res = L.AdmmResultC()
    err = C.c_double()
    _check(ctx.lib.nqb_factorize_layer(ctx.handle, _ptr(w), n, m, C.byref(cfg), scale_floor, 0,
                                       C.byref(h), C.byref(res), C.byref(err)),
           "factorize_layer")
    d = res.as_dict()
    state = AdmmState(res.rho, res.iteration, [], res.primal_residual, bool(res.converged), d)
    return DeviceLayer(ctx, h), err.value, state


# ---------------------------------------------------------------------------
# NQPK packed-model files (io.hpp:27-54, io.cpp:139-193); SURVEY.md §8(f) row 1
# ---------------------------------------------------------------------------
def _nqpk_layers(handle) -> list:
    lib = L.load()
    out = []
    for i in range(lib.nqb_nqpk_count(handle)):
        name_len, n, m, r = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib.nqb_nqpk_layer_info(handle, i, None, 0, C.byref(name_len), C.byref(n),
                                       C.byref(m), C.byref(r)), "read_packed_model")
        buf = C.create_string_buffer(name_len.value + 1)
        _check(lib.nqb_nqpk_layer_info(handle, i, buf, name_len.value + 1, None, None, None, None),
               "read_packed_model")
        pu, pv, p1, p2 = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib.nqb_nqpk_layer_data(handle, i, C.byref(pu), C.byref(pv), C.byref(p1),
                                       C.byref(p2)), "read_packed_model")
        k = (r.value + 31) // 32

        def arr(p, count, ct, dt):
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(count,)).astype(dt)

        u = arr(pu, n.value * k, C.c_uint32, np.uint32).reshape(n.value, k)
        v = arr(pv, m.value * k, C.c_uint32, np.uint32).reshape(m.value, k)
        s1 = arr(p1, n.value, C.c_uint16, np.uint16).view(np.float16).astype(np.float64)
        s2 = arr(p2, m.value, C.c_uint16, np.uint16).view(np.float16).astype(np.float64)
        out.append((buf.value.decode("utf-8"), FactorizedLayer(n.value, m.value, r.value, u, v, s1, s2)))
    return out


def read_packed_model(path: str) -> list:
    """read_packed_model (io.cpp:191-193): [(name, FactorizedLayer)] with the file's
    binary16 scales widened exactly to float64 (host only; no device needed)."""
    lib = L.load()
    h = C.c_void_p()
    _check(lib.nqb_nqpk_open(os.fsencode(path), C.byref(h)), "read_packed_model")
    try:
        return _nqpk_layers(h)
    finally:
        lib.nqb_nqpk_free(h)


def deserialize_packed_model(data: bytes) -> list:
    """deserialize_packed_model (io.cpp:160-185)."""
    lib = L.load()
    h = C.c_void_p()
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(bytes(data) or b"\0")
    _check(lib.nqb_nqpk_parse(buf, len(data), C.byref(h)), "deserialize_packed_model")
    try:
        return _nqpk_layers(h)
    finally:
        lib.nqb_nqpk_free(h)


def load_packed_model(path: str, ctx: Context | None = None) -> list:
    """An NQPK file straight to the device layout: [(name, DeviceLayer)], uploaded
    with the file's binary16 scales unchanged."""
    ctx = ctx or context()
    lib = ctx.lib
    h = C.c_void_p()
    _check(lib.nqb_nqpk_open(os.fsencode(path), C.byref(h)), "load_packed_model")
    try:
        names = [name for name, _ in _nqpk_layers(h)]
        out = []
        for i, name in enumerate(names):
            d = C.c_void_p()
            _check(lib.nqb_nqpk_layer_upload(ctx.handle, h, i, C.byref(d)), "load_packed_model")
            out.append((name, DeviceLayer(ctx, d)))
        return out
    finally:
        lib.nqb_nqpk_free(h)


def serialize_packed_model(layers) -> bytes:
    """serialize_packed_model (io.cpp:139-158) of [(name, FactorizedLayer)]; scales
    are snapped to binary16 like double_to_half (half.hpp:83-85)."""
    lib = L.load()
    cnt = len(layers)
    names = (C.c_char_p * max(1, cnt))(*[nm.encode("utf-8") for nm, _ in layers])
    keep = []

    def arrp(arrs, ct):
        ptrs = (C.c_void_p * max(1, cnt))()
        for i, a in enumerate(arrs):
            keep.append(a)
            ptrs[i] = a.ctypes.data
        return ptrs

    lays = [lay for _, lay in layers]
    n = (C.c_uint32 * max(1, cnt))(*[l.n for l in lays])
    m = (C.c_uint32 * max(1, cnt))(*[l.m for l in lays])
    r = (C.c_uint32 * max(1, cnt))(*[l.r for l in lays])
    u = arrp([np.ascontiguousarray(l.u, np.uint32) for l in lays], C.c_uint32)
    v = arrp([np.ascontiguousarray(l.v, np.uint32) for l in lays], C.c_uint32)
    h = lambda s: np.ascontiguousarray(  # noqa: E731
        np.asarray(s, np.float64).astype(np.float32).astype(np.float16).view(np.uint16))
    s1 = arrp([h(l.s1) for l in lays], C.c_uint16)
    s2 = arrp([h(l.s2) for l in lays], C.c_uint16)
    ln = C.c_uint64()
    _check(lib.nqb_nqpk_serialize(cnt, names, n, m, r, u, v, s1, s2, None, 0, C.byref(ln)),
           "serialize_packed_model")
    buf = (C.c_uint8 * max(1, ln.value))()
    _check(lib.nqb_nqpk_serialize(cnt, names, n, m, r, u, v, s1, s2, buf, ln.value, C.byref(ln)),
           "serialize_packed_model")
    return bytes(buf)[: ln.value]


def write_packed_model(path: str, layers, ctx: Context | None = None) -> None:
    """write_packed_model (io.cpp:187-189) of [(name, DeviceLayer | FactorizedLayer)]:
    device layers are written from the device (bit-exact download)."""
    if layers and all(isinstance(l, DeviceLayer) for _, l in layers):
        ctx = ctx or layers[0][1].ctx
        cnt = len(layers)
        names = (C.c_char_p * cnt)(*[nm.encode("utf-8") for nm, _ in layers])
        hs = (C.c_void_p * cnt)(*[l.handle.value if isinstance(l.handle, C.c_void_p) else l.handle
                                  for _, l in layers])
        _check(ctx.lib.nqb_nqpk_write_layers(ctx.handle, os.fsencode(path), cnt, names, hs),
               "write_packed_model")
        return
    data = serialize_packed_model([(nm, l.download() if isinstance(l, DeviceLayer) else l)
                                   for nm, l in layers])
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from e


# ---------------------------------------------------------------------------
# Preconditioner: phase 1 of the pipeline (precondition.hpp, precondition.cpp:37-153),
# SURVEY.md §8(f) row 3.  Column statistics and the D_out W D_in scaling run on
# the device in the reference's operation order (bitwise equal results).
# ---------------------------------------------------------------------------
@dataclass
class ChannelStats:  # precondition.hpp:29-38
    sum_squares: np.ndarray
    sample_count: int = 0
    tau: float = 0.0

    @classmethod
    def zeros(cls, channel_count: int) -> "ChannelStats":
        return cls(np.zeros(channel_count, np.float64), 0, 0.0)

    def channel_count(self) -> int:
        return int(self.sum_squares.size)


@dataclass
class Preconditioner:  # precondition.hpp:50-55
    diag_in: np.ndarray
    diag_out: np.ndarray  # empty = identity
    gamma: float = 0.0
    tau_max: float = 1.0


def accumulate_stats(stats: ChannelStats, batch, percentile: float,
                     ctx: Context | None = None) -> ChannelStats:
    """accumulate_stats (precondition.cpp:37-62): batch is samples x channels (host
    array, or a CUDA torch tensor used in place).  Updates and returns `stats`."""
    ctx = ctx or context()
    ss = np.ascontiguousarray(stats.sum_squares, np.float64)
    cnt, tau = C.c_uint64(stats.sample_count), C.c_double(stats.tau)
    if hasattr(batch, "data_ptr") and getattr(batch, "is_cuda", False):
        rows, cols = batch.shape
        if cols != ss.size:
            raise DimensionMismatch("accumulate_stats: cols(batch) != channel_count")
        ctx.bind_torch_stream()
        st = ctx.lib.nqb_accumulate_stats_device(ctx.handle, batch.data_ptr(), rows, cols,
                                                 percentile, ss.ctypes.data, C.byref(cnt),
                                                 C.byref(tau))
    else:
        b = _mat(batch)
        if b.shape[1] != ss.size:
            raise DimensionMismatch("accumulate_stats: cols(batch) != channel_count")
        st = ctx.lib.nqb_accumulate_stats_host(ctx.handle, _ptr(b), b.shape[0], b.shape[1],
                                               percentile, ss.ctypes.data, C.byref(cnt),
                                               C.byref(tau))
    _check(st, "accumulate_stats")
    stats.sum_squares, stats.sample_count, stats.tau = ss, cnt.value, tau.value
    return stats


def build_preconditioner(in_stats: ChannelStats, out_stats: Optional[ChannelStats],
                         gamma: float, eps_floor: float) -> Preconditioner:
    """build_preconditioner (precondition.cpp:99-121); host arithmetic, no device."""
    lib = L.load()
    ins = np.ascontiguousarray(in_stats.sum_squares, np.float64)
    din = np.empty(ins.size, np.float64)
    tau_max = C.c_double()
    if out_stats is not None:
        outs = np.ascontiguousarray(out_stats.sum_squares, np.float64)
        dout = np.empty(outs.size, np.float64)
        st = lib.nqb_build_preconditioner(ins.size, ins.ctypes.data, in_stats.sample_count,
                                          in_stats.tau, outs.size, outs.ctypes.data,
                                          out_stats.sample_count, out_stats.tau, gamma, eps_floor,
                                          din.ctypes.data, dout.ctypes.data, C.byref(tau_max))
    else:
        dout = np.empty(0, np.float64)
        st = lib.nqb_build_preconditioner(ins.size, ins.ctypes.data, in_stats.sample_count,
                                          in_stats.tau, 0, None, 0, 0.0, gamma, eps_floor,
                                          din.ctypes.data, None, C.byref(tau_max))
    _check(st, "build_preconditioner")
    return Preconditioner(din, dout, gamma, tau_max.value)


def precondition_weight(w, p: Preconditioner, ctx: Context | None = None) -> np.ndarray:
    """precondition_weight (precondition.cpp:123-138): D_out W D_in (a copy)."""
    ctx = ctx or context()
    out = np.array(_mat(w), dtype=np.float64, copy=True)
    rows, cols = out.shape
    if p.diag_in.size and cols != p.diag_in.size:
        raise DimensionMismatch("precondition_weight: cols(W) != |diag_in|")
    if p.diag_out.size and rows != p.diag_out.size:
        raise DimensionMismatch("precondition_weight: rows(W) != |diag_out|")
    dout = _f64(p.diag_out) if p.diag_out.size else None
    din = _f64(p.diag_in) if p.diag_in.size else None
    _check(ctx.lib.nqb_precondition_weight_host(ctx.handle, out.ctypes.data, rows, cols,
                                                _ptr(dout), _ptr(din)), "precondition_weight")
    return out


def unprecondition_rows(factor, diag, ctx: Context | None = None) -> np.ndarray:
    """unprecondition_rows (precondition.cpp:143-153): rows / diag (a copy; empty diag = identity)."""
    ctx = ctx or context()
    out = np.array(_mat(factor), dtype=np.float64, copy=True)
    d = np.asarray(diag, np.float64)
    if d.size == 0:
        return out
    if out.shape[0] != d.size:
        raise DimensionMismatch("unprecondition_rows: rows(factor) != |diag|")
    _check(ctx.lib.nqb_unprecondition_rows_host(ctx.handle, out.ctypes.data, out.shape[0],
                                                out.shape[1], _ptr(_f64(d))), "unprecondition_rows")
    return out


# ---------------------------------------------------------------------------
# refine.hpp: STE refinement of one factorized latent layer on the device
#
# ---------------------------------------------------------------------------
@dataclass
class TuneConfig:  # refine.hpp:55-64
    epochs: int = 8
    learning_rate: float = 1e-4
    batch_size: int = 4
    schedule: str = "cosine"  # or "constant"
    seed: int = 0

    def c(self):
        return L.TuneConfig(self.epochs, self.batch_size, self.learning_rate,
                            1 if self.schedule == "cosine" else 0, 0, self.seed & 0xFFFFFFFFFFFFFFFF)


@dataclass
class FactorizedLatentLayer:  # refine.hpp:28-34
    latent_u: np.ndarray
    latent_v: np.ndarray
    s1: np.ndarray
    s2: np.ndarray


def ste_refine(layer: FactorizedLatentLayer, x, teacher_outputs, config: TuneConfig,
               column_weights=None, ctx: Context | None = None):
    """ste_refine (refine.cpp:420-425) on a one-layer chain, on the device: returns
    (refined FactorizedLatentLayer, best loss).  x is (m, b) and teacher_outputs
    (n, b), inputs as columns.  Raises NonFiniteLoss (with .best_chain) on
    divergence, like the reference."""
    ctx = ctx or context()
    lu, lv = _mat(layer.latent_u).copy(), _mat(layer.latent_v).copy()
    s1, s2 = _f64(layer.s1).copy(), _f64(layer.s2).copy()
    n, r = lu.shape
    m = lv.shape[0]
    X, T = _mat(x), _mat(teacher_outputs)
    if lv.shape[1] != r or s1.size != n or s2.size != m or X.shape[0] != m:
        raise DimensionMismatch("chain input dim does not match X rows")
    if T.shape != (n, X.shape[1]):
        raise DimensionMismatch("teacher outputs do not match chain output shape")
    w = None
    if column_weights is not None and len(column_weights):
        w = _f64(column_weights)
        if w.size != X.shape[1]:
            raise DimensionMismatch("column weight count does not match batch")
    best = C.c_double()
    cfg = config.c()
    st = ctx.lib.nqb_ste_refine_layer_host(ctx.handle, _ptr(lu), _ptr(lv), _ptr(s1), _ptr(s2), n, m, r,
                                           _ptr(X), _ptr(T), X.shape[1],
                                           None if w is None else _ptr(w), C.byref(cfg), C.byref(best))
    out = FactorizedLatentLayer(lu, lv, s1, s2)
    if st == NonFiniteLoss.code:
        err = NonFiniteLoss("ste_refine: " + L.load().nqb_last_error().decode(errors="replace"),
                            code=st)
        err.best_chain = out
        raise err
    _check(st, "ste_refine")
    return out, best.value
