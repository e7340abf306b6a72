"""oracle.py - TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers built by oracle/Makefile:

* ``restated()``  -> oracle/_build/libnqoracle.so, the plain-C restatement of the
  reference algorithm (oracle/nq_oracle.c);
* ``reference()`` -> oracle/_ref/libnqref.so, the unmodified NanoQuant reference
  library (/root/reference/proj/src) behind oracle/ref_harness.cpp.

Both expose the same Python surface, named after the reference functions
(packed.hpp, linalg.hpp, admm.hpp, balance.hpp, storage.hpp).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg import this module; the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(_HERE, "_build", "libnqoracle.so")
REFERENCE_SO = os.path.join(_HERE, "_ref", "libnqref.so")

_P = C.c_void_p
_U32, _I32, _U64, _D = C.c_uint32, C.c_int32, C.c_uint64, C.c_double


class AdmmConfig(C.Structure):
    """nqb_admm_config (include/nqb.h) == AdmmConfig (admm.hpp:41-51)."""

    _fields_ = [("rank", _U32), ("max_iters", _I32), ("rho_start", _D), ("rho_end", _D),
                ("ridge", _D), ("tol", _D), ("seed", _U64), ("record_trace", _I32),
                ("reserved", _I32)]

    @classmethod
    def make(cls, rank, max_iters=400, rho_start=0.0, rho_end=0.0, ridge=1e-4, tol=1e-4,
             seed=0, record_trace=1):
        return cls(rank, max_iters, rho_start, rho_end, ridge, tol, seed, record_trace, 0)


class AdmmResult(C.Structure):
    """nqb_admm_result (include/nqb.h)."""

    _fields_ = [("iteration", _U32), ("converged", _I32), ("primal_residual", _D),
                ("rho", _D), ("trace_len", _U32), ("svd_steps", _U32),
                ("svd_power_iters", _U64), ("svd_converged_steps", _U32), ("reserved", _U32),
                ("sigma_max", _D), ("seconds_svd_init", _D), ("seconds_iterations", _D)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class OracleError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: status {code}")
        self.code = code


@dataclass
class Layer:
    """FactorizedLayer (packed.hpp:57-72) in the reference layout."""

    n: int
    m: int
    r: int
    u: np.ndarray  # (n, ceil(r/32)) uint32
    v: np.ndarray  # (m, ceil(r/32)) uint32
    s1: np.ndarray  # (n,) float64
    s2: np.ndarray  # (m,) float64


def wpr(cols: int) -> int:
    return (cols + 31) // 32


def _ptr(a):
    return a.ctypes.data_as(_P) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


class Checker:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.path = path
        self.lib[prefix + "rng_create"].restype = _P
        self.lib[prefix + "rng_create"].argtypes = [_U64]
        self.lib[prefix + "rng_uniform"].argtypes = [_P, _D, _D, _U64, _P]
        for name in ("rng_u64", "rng_gaussian", "rng_sign"):
            self.lib[prefix + name].argtypes = [_P, _U64, _P]
        self.lib[prefix + "rng_index"].argtypes = [_P, _U64, _U64, _P]
        self.lib[prefix + "rng_destroy"].argtypes = [_P]

    def _fn(self, name):
        return self.lib[self.prefix + name]

    def _call(self, name, *args):
        st = self._fn(name)(*args)
        if st != 0:
            raise OracleError(st, self.prefix + name)

    # -- Rng ------------------------------------------------------------------
    def rng(self, seed: int) -> "Rng":
        return Rng(self, seed)

    # -- half ----------------------------------------------------------------
    def double_to_half(self, x):
        x = _f64(x)
        out = np.empty(x.size, np.uint16)
        f = self._fn("double_to_half")
        f.argtypes = [_P, _U64, _P]
        f(_ptr(x), x.size, _ptr(out))
        return out.reshape(x.shape)

    def half_to_double(self, h):
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(h.size, np.float64)
        f = self._fn("half_to_double")
        f.argtypes = [_P, _U64, _P]
        f(_ptr(h), h.size, _ptr(out))
        return out.reshape(h.shape)

    def snap_half(self, x):
        return self.half_to_double(self.double_to_half(x))

    # -- storage ----------------------------------------------------------------
    def rank_for_target_bpw(self, n, m, t):
        out = _U32()
        f = self._fn("rank_for_target_bpw")
        f.argtypes = [_U64, _U64, _D, C.POINTER(_U32)]
        self._call("rank_for_target_bpw", _U64(n), _U64(m), _D(t), C.byref(out))
        return out.value

    # -- packed -----------------------------------------------------------------
    def binarize(self, x):
        x = _f64(x)
        rows, cols = x.shape
        out = np.empty_like(x)
        self._call("binarize", _ptr(x), _U32(rows), _U32(cols), _ptr(out))
        return out

    def pack_signs(self, s):
        s = _f64(s)
        rows, cols = s.shape
        out = np.zeros((rows, wpr(cols)), np.uint32)
        self._call("pack_signs", _ptr(s), _U32(rows), _U32(cols), _ptr(out))
        return out

    def unpack_signs(self, words, rows, cols):
        words = _u32(words)
        out = np.empty((rows, cols), np.float64)
        self._call("unpack_signs", _ptr(words), _U32(rows), _U32(cols), _ptr(out))
        return out

    def make_factorized_layer(self, latent_u, latent_v, s1, s2) -> Layer:
        """make_factorized_layer (packed.cpp:105-124)."""
        u = self.pack_signs(self.binarize(latent_u))
        v = self.pack_signs(self.binarize(latent_v))
        return Layer(latent_u.shape[0], latent_v.shape[0], latent_u.shape[1], u, v,
                     _f64(s1), _f64(s2))

    def _layer_args(self, L: Layer):
        return [_U32(L.n), _U32(L.m), _U32(L.r), _ptr(_u32(L.u)), _ptr(_u32(L.v)),
                _ptr(_f64(L.s1)), _ptr(_f64(L.s2))]

    def reconstruct_dense(self, L: Layer):
        out = np.empty((L.n, L.m), np.float64)
        self._call("reconstruct_dense", *self._layer_args(L), _ptr(out))
        return out

    def gemv_packed(self, L: Layer, x):
        x = _f64(x)
        y = np.empty(L.n, np.float64)
        self._call("gemv_f64", *self._layer_args(L), _ptr(x), _U32(x.size), _ptr(y))
        return y

    # -- precondition.cpp (reference only; no C restatement) ------------------
    def _ref_only(self, what):
        if self.prefix != "nqref_":
            raise NotImplementedError(f"{what} is checked against the reference only")

    def accumulate_stats(self, sum_squares, count, tau, batch, percentile):
        """accumulate_stats (precondition.cpp:37-62) -> (sum_squares, count, tau)."""
        self._ref_only("accumulate_stats")
        b = _f64(batch)
        ss = np.array(sum_squares, np.float64, copy=True)
        c, t = C.c_uint64(count), C.c_double(tau)
        fn = self._fn("accumulate_stats")
        fn.argtypes = [C.c_void_p, _U32, _U32, _D, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(_D)]
        st = fn(b.ctypes.data, b.shape[0], b.shape[1], percentile, ss.ctypes.data, C.byref(c), C.byref(t))
        if st != 0:
            raise OracleError(st, "nqref_accumulate_stats")
        return ss, c.value, t.value

    def build_preconditioner(self, in_ss, in_count, in_tau, out_ss, out_count, out_tau, gamma,
                             eps_floor):
        self._ref_only("build_preconditioner")
        ins = _f64(in_ss)
        din = np.empty(ins.size, np.float64)
        outs = _f64(out_ss) if out_ss is not None else None
        dout = np.empty(outs.size, np.float64) if outs is not None else None
        tm = C.c_double()
        fn = self._fn("build_preconditioner")
        fn.argtypes = [_U32, C.c_void_p, C.c_uint64, _D, _U32, C.c_void_p, C.c_uint64, _D, _D, _D,
                       C.c_void_p, C.c_void_p, C.POINTER(_D)]
        st = fn(ins.size, ins.ctypes.data, in_count, in_tau, 0 if outs is None else outs.size,
                None if outs is None else outs.ctypes.data, out_count, out_tau, gamma, eps_floor,
                din.ctypes.data, None if dout is None else dout.ctypes.data, C.byref(tm))
        if st != 0:
            raise OracleError(st, "nqref_build_preconditioner")
        return din, dout, tm.value

    def precondition_weight(self, w, diag_out, diag_in):
        self._ref_only("precondition_weight")
        w = _f64(w)
        out = np.empty_like(w)
        do = _f64(diag_out) if diag_out is not None else None
        di = _f64(diag_in) if diag_in is not None else None
        self._call("precondition_weight", _ptr(w), _U32(w.shape[0]), _U32(w.shape[1]),
                   _ptr(do) if do is not None else None, _ptr(di) if di is not None else None,
                   _ptr(out))
        return out

    def unprecondition_rows(self, factor, diag):
        self._ref_only("unprecondition_rows")
        f = np.array(factor, np.float64, copy=True)
        d = _f64(diag) if diag is not None else None
        self._call("unprecondition_rows", _ptr(f), _U32(f.shape[0]), _U32(f.shape[1]),
                   _ptr(d) if d is not None else None)
        return f

    def serialize_nqpk(self, named_layers):
        """serialize_packed_model (io.cpp:139-158) of [(name, Layer)] -- reference only
        (nqref_serialize_nqpk in ref_harness.cpp); scales snapped by double_to_half."""
        if self.prefix != "nqref_":
            raise NotImplementedError("NQPK serialisation is checked against the reference only")
        cnt = len(named_layers)
        names = (C.c_char_p * cnt)(*[nm.encode("utf-8") for nm, _ in named_layers])
        lays = [l for _, l in named_layers]
        keep = [(_u32(l.u), _u32(l.v), _f64(l.s1), _f64(l.s2)) for l in lays]
        u32a = lambda vals: (C.c_uint32 * cnt)(*vals)  # noqa: E731
        ptrs = lambda idx: (C.c_void_p * cnt)(*[k[idx].ctypes.data for k in keep])  # noqa: E731
        cap = 64 + sum(16 + len(nm.encode()) + 4 * (l.u.size + l.v.size) + 2 * (l.n + l.m)
                       for nm, l in named_layers)
        buf = (C.c_uint8 * cap)()
        ln = C.c_uint64()
        fn = self._fn("serialize_nqpk")
        fn.argtypes = [_U32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                       C.POINTER(C.c_uint64)]
        st = fn(cnt, names, u32a([l.n for l in lays]), u32a([l.m for l in lays]),
                u32a([l.r for l in lays]), ptrs(0), ptrs(1), ptrs(2), ptrs(3), buf, cap, C.byref(ln))
        if st != 0:
            raise OracleError(st, "nqref_serialize_nqpk")
        return bytes(buf)[: ln.value]

    def gemv_packed_f32(self, L: Layer, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty(L.n, np.float32)
        self._call("gemv_f32", *self._layer_args(L), _ptr(x), _U32(x.size), _ptr(y))
        return y

    def gemm_packed(self, L: Layer, x, threads=1):
        x = _f64(x)
        b = x.shape[1]
        y = np.empty((L.n, b), np.float64)
        extra = [_U32(threads)] if self.prefix == "nqref_" else []
        self._call("gemm", *self._layer_args(L), _ptr(x), _U32(b), _ptr(y), *extra)
        return y

    # -- linalg -----------------------------------------------------------------
    def top_singular_pair(self, m, max_iters=500, tol=1e-12):
        m = _f64(m)
        rows, cols = m.shape
        sigma, conv = _D(), _I32()
        left, right = np.empty(rows), np.empty(cols)
        self._call("top_singular_pair", _ptr(m), _U32(rows), _U32(cols), _I32(max_iters),
                   _D(tol), C.byref(sigma), _ptr(left), _ptr(right), C.byref(conv))
        return sigma.value, left, right, bool(conv.value)

    def spectral_norm_estimate(self, m, iters=200):
        m = _f64(m)
        out = _D()
        self._call("spectral_norm", _ptr(m), _U32(m.shape[0]), _U32(m.shape[1]),
                   _I32(iters), C.byref(out))
        return out.value

    def truncated_svd_factors(self, m, rank):
        m = _f64(m)
        u = np.empty((m.shape[0], rank))
        v = np.empty((m.shape[1], rank))
        self._call("truncated_svd", _ptr(m), _U32(m.shape[0]), _U32(m.shape[1]), _U32(rank),
                   _ptr(u), _ptr(v))
        return u, v

    def cholesky_solve(self, a, b):
        a, b = _f64(a), _f64(b)
        x = np.empty_like(b)
        self._call("cholesky_solve", _ptr(a), _U32(a.shape[0]), _ptr(b), _U32(b.shape[1]),
                   _ptr(x))
        return x

    # -- admm -------------------------------------------------------------------
    def svid(self, p):
        p = _f64(p)
        z = np.empty_like(p)
        self._call("svid", _ptr(p), _U32(p.shape[0]), _U32(p.shape[1]), _ptr(z))
        return z

    def admm_factor_solve(self, target, fixed, z, l, rho, ridge):
        target, fixed, z, l = map(_f64, (target, fixed, z, l))
        x = np.empty((target.shape[0], fixed.shape[1]))
        self._call("factor_solve", _ptr(target), _U32(target.shape[0]), _U32(target.shape[1]),
                   _ptr(fixed), _U32(fixed.shape[1]), _ptr(z), _ptr(l), _D(rho), _D(ridge),
                   _ptr(x))
        return x

    def augmented_lagrangian(self, u, v, zu, zv, lu, lv, rho, target, ridge):
        args = list(map(_f64, (u, v, zu, zv, lu, lv)))
        target = _f64(target)
        out = _D()
        self._call("lagrangian", *[_ptr(a) for a in args], _U32(u.shape[0]),
                   _U32(v.shape[0]), _U32(u.shape[1]), _D(rho), _ptr(target), _D(ridge),
                   C.byref(out))
        return out.value

    def admm_factorize(self, w, cfg: AdmmConfig):
        w = _f64(w)
        n, m = w.shape
        cu = np.empty((n, cfg.rank))
        cv = np.empty((m, cfg.rank))
        trace = np.empty(cfg.max_iters + 1)
        res = AdmmResult()
        self._call("admm_factorize", _ptr(w), _U32(n), _U32(m), C.byref(cfg), _ptr(cu),
                   _ptr(cv), _ptr(trace), C.byref(res))
        return cu, cv, trace[: res.trace_len].copy(), res.as_dict()

    def balance_and_extract_scales(self, pu, pv, diag_out=None, diag_in=None, floor=1e-12):
        pu, pv = _f64(pu), _f64(pv)
        n, r = pu.shape
        m = pv.shape[0]
        lu, lv = np.empty_like(pu), np.empty_like(pv)
        s1, s2 = np.empty(n), np.empty(m)
        eta = _D()
        do = _f64(diag_out) if diag_out is not None else None
        di = _f64(diag_in) if diag_in is not None else None
        self._call("balance", _ptr(pu), _ptr(pv), _U32(n), _U32(m), _U32(r), _ptr(do),
                   _ptr(di), _D(floor), _ptr(lu), _ptr(lv), _ptr(s1), _ptr(s2), C.byref(eta))
        return lu, lv, s1, s2, eta.value

    def factorize_layer(self, w, cfg: AdmmConfig, floor=1e-12):
        """pipeline.cpp:95-110 + :150-153 for one matrix."""
        w = _f64(w)
        n, m = w.shape
        k = wpr(cfg.rank)
        u = np.zeros((n, k), np.uint32)
        v = np.zeros((m, k), np.uint32)
        s1, s2 = np.empty(n), np.empty(m)
        err = _D()
        trace = np.empty(cfg.max_iters + 1)
        res = AdmmResult()
        self._call("factorize_layer", _ptr(w), _U32(n), _U32(m), C.byref(cfg), _D(floor),
                   _ptr(u), _ptr(v), _ptr(s1), _ptr(s2), C.byref(err), _ptr(trace),
                   C.byref(res))
        layer = Layer(n, m, cfg.rank, u, v, s1, s2)
        return layer, err.value, trace[: res.trace_len].copy(), res.as_dict()

    def ste_refine(self, lu, lv, s1, s2, x, teacher, epochs=8, lr=1e-4, batch=4, cosine=True,
                   seed=0, column_weights=None):
        """ste_refine (refine.cpp:420-425) on a one-layer chain; returns
        (latent_u, latent_v, s1, s2, status)."""
        self._ref_only("ste_refine")
        lu, lv = _f64(lu).copy(), _f64(lv).copy()
        s1, s2 = _f64(s1).copy(), _f64(s2).copy()
        x, t = _f64(x), _f64(teacher)
        n, r = lu.shape
        m, b = x.shape
        w = None if column_weights is None else _f64(column_weights)
        fn = self.lib.nqref_ste_refine
        fn.restype = C.c_int
        st = fn(_ptr(lu), _ptr(lv), _ptr(s1), _ptr(s2), _U32(n), _U32(m), _U32(r), _ptr(x), _ptr(t),
                _U32(b), None if w is None else _ptr(w), _I32(epochs), _D(lr), _I32(batch),
                _I32(1 if cosine else 0), _U64(seed))
        return lu, lv, s1, s2, st

    def layer_rel_error(self, L: Layer, w):
        w = _f64(w)
        out = _D()
        self._call("layer_rel_error", *self._layer_args(L), _ptr(w), C.byref(out))
        return out.value


class Rng:
    """nanoquant::Rng (rng.hpp:25-58) driven through a checker library."""

    def __init__(self, checker: Checker, seed: int):
        self._c = checker
        self._h = checker._fn("rng_create")(_U64(seed))

    def __del__(self):
        try:
            self._c._fn("rng_destroy")(self._h)
        except Exception:
            pass

    def u64(self, n):
        out = np.empty(n, np.uint64)
        self._c._fn("rng_u64")(self._h, _U64(n), _ptr(out))
        return out

    def uniform(self, lo, hi, n):
        out = np.empty(n, np.float64)
        self._c._fn("rng_uniform")(self._h, _D(lo), _D(hi), _U64(n), _ptr(out))
        return out

    def gaussian(self, n):
        out = np.empty(n, np.float64)
        self._c._fn("rng_gaussian")(self._h, _U64(n), _ptr(out))
        return out

    def sign(self, n):
        out = np.empty(n, np.float64)
        self._c._fn("rng_sign")(self._h, _U64(n), _ptr(out))
        return out

    def index(self, n, count=None):
        """rng.index(n) (rng.hpp:52): an int, or an array of `count` draws."""
        k = 1 if count is None else count
        out = np.empty(k, np.uint64)
        self._c._fn("rng_index")(self._h, _U64(n), _U64(k), _ptr(out))
        return int(out[0]) if count is None else out

    def matrix(self, rows, cols):
        """random_matrix (test_support.hpp:52-56)."""
        return self.gaussian(rows * cols).reshape(rows, cols)


_CACHE: dict = {}


def restated() -> Checker:
    if "o" not in _CACHE:
        _CACHE["o"] = Checker(RESTATED_SO, "nqo_")
    return _CACHE["o"]


def reference() -> Checker:
    if "r" not in _CACHE:
        _CACHE["r"] = Checker(REFERENCE_SO, "nqref_")
    return _CACHE["r"]


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)


# ---------------------------------------------------------------------------
# Synthetic inputs shared by tests and the bench; generated
# with the reference Rng so both sides see identical bits.
# ---------------------------------------------------------------------------
def synthetic_weight(checker: Checker, seed: int, n: int, m: int) -> np.ndarray:
    """W_ij = fp32(0.02 * g), g from Rng(seed) row-major, promoted to double."""
    g = checker.rng(seed).gaussian(n * m)
    return (0.02 * g).astype(np.float32).astype(np.float64).reshape(n, m)


def synthetic_layer(checker: Checker, seed: int, n: int, m: int, r: int) -> Layer:
    """Random packed layer: bits from Rng(seed).next_u64 (pad zeroed), scales
    ~U(0.25, 2) snapped to binary16 (NQPK precision), as SURVEY §8(d) row 2."""
    rng = checker.rng(seed)
    k = wpr(r)
    tail = r % 32
    mask = np.uint32(0xFFFFFFFF if tail == 0 else (1 << tail) - 1)

    def bits(rows):
        w = (rng.u64(rows * k) & np.uint64(0xFFFFFFFF)).astype(np.uint32).reshape(rows, k)
        w[:, -1] &= mask
        return w

    u = bits(n)
    v = bits(m)
    s1 = checker.snap_half(rng.uniform(0.25, 2.0, n))
    s2 = checker.snap_half(rng.uniform(0.25, 2.0, m))
    return Layer(n, m, r, u, v, s1, s2)
