"""ctypes binding of libnqb.so (include/nqb.h).

The library is built in-tree (``paper_2602_06694_b200/libnqb.so``) by
``__graft_entry__.build()`` / ``make -C paper_2602_06694_b200/csrc``.  There is
no CPU fallback: if the library or a B200 is missing, loading or creating a
context raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnqb.so")

P = C.c_void_p
U32, I32, U64, D = C.c_uint32, C.c_int32, C.c_uint64, C.c_double
PU32 = C.POINTER(U32)
PI32 = C.POINTER(I32)
PD = C.POINTER(D)
PP = C.POINTER(P)


class AdmmConfig(C.Structure):
    """nqb_admm_config == AdmmConfig (admm.hpp:41-51) + record_trace."""

    _fields_ = [("rank", U32), ("max_iters", I32), ("rho_start", D), ("rho_end", D),
                ("ridge", D), ("tol", D), ("seed", U64), ("record_trace", I32),
                ("reserved", I32)]


class AdmmResultC(C.Structure):
    """nqb_admm_result."""

    _fields_ = [("iteration", U32), ("converged", I32), ("primal_residual", D),
                ("rho", D), ("trace_len", U32), ("svd_steps", U32),
                ("svd_power_iters", U64), ("svd_converged_steps", U32), ("reserved", U32),
                ("sigma_max", D), ("seconds_svd_init", D), ("seconds_iterations", D)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class TuneConfig(C.Structure):
    """nqb_tune_config (TuneConfig, refine.hpp:55-64)."""

    _fields_ = [("epochs", I32), ("batch_size", I32), ("learning_rate", C.c_double),
                ("schedule", I32), ("reserved", I32), ("seed", C.c_uint64)]


class PassStep(C.Structure):
    """nqb_pass_step."""

    _fields_ = [("group", P), ("layer", P), ("d_x", P), ("d_y", P * 4), ("f32", I32),
                ("reserved", I32)]


# name -> (restype, argtypes); mirrors include/nqb.h one-to-one.
PROTOTYPES = {
    "nqb_status_kind": (C.c_int, [C.c_int]),
    "nqb_last_error": (C.c_char_p, []),
    "nqb_version": (C.c_char_p, []),
    "nqb_create": (C.c_int, [C.c_int, PP]),
    "nqb_destroy": (C.c_int, [P]),
    "nqb_set_stream": (C.c_int, [P, P]),
    "nqb_host_register": (C.c_int, [P, P, C.c_size_t]),
    "nqb_host_unregister": (C.c_int, [P, P]),
    "nqb_get_stream": (P, [P]),
    "nqb_synchronize": (C.c_int, [P]),
    "nqb_kernel_launches": (U64, [P]),
    "nqb_rank_for_target_bpw": (C.c_int, [U64, U64, D, PU32]),
    "nqb_synthetic_weight_host": (C.c_int, [U64, U64, D, C.c_int, P]),
    "nqb_binarize": (C.c_int, [P, P, U64, P, C.c_int]),
    "nqb_pack_signs": (C.c_int, [P, P, U32, U32, P, C.c_int]),
    "nqb_pack_latent": (C.c_int, [P, P, U32, U32, P, C.c_int]),
    "nqb_unpack_signs": (C.c_int, [P, P, U32, U32, P, C.c_int]),
    "nqb_layer_upload": (C.c_int, [P, U32, U32, U32, P, P, P, P, PP]),
    "nqb_layer_upload_exact": (C.c_int, [P, U32, U32, U32, P, P, P, P, PP]),
    "nqb_layer_upload_f16": (C.c_int, [P, U32, U32, U32, P, P, P, P, PP]),
    "nqb_layer_free": (C.c_int, [P]),
    "nqb_layer_shape": (C.c_int, [P, PU32, PU32, PU32]),
    "nqb_layer_device_bytes": (U64, [P]),
    "nqb_layer_download": (C.c_int, [P, P, P, P, P, P]),
    "nqb_gemv_f32_host": (C.c_int, [P, P, P, P]),
    "nqb_gemv_f64_host": (C.c_int, [P, P, P, P]),
    "nqb_gemv_f32_device": (C.c_int, [P, P, P, P]),
    "nqb_gemv_f16_device": (C.c_int, [P, P, P, P]),
    "nqb_gemm_f64_host": (C.c_int, [P, P, P, U32, P]),
    "nqb_gemm_f16_device": (C.c_int, [P, P, P, U32, P]),
    "nqb_reconstruct_dense_host": (C.c_int, [P, P, P]),
    "nqb_admm_config_default": (None, [C.POINTER(AdmmConfig)]),
    "nqb_ste_refine_layer_host": (C.c_int, [P, P, P, P, P, U32, U32, U32, P, P, U32, P,
                                            C.POINTER(TuneConfig), PD]),
    "nqb_admm_factorize_host": (C.c_int, [P, P, U32, U32, C.POINTER(AdmmConfig), P, P, P,
                                          C.POINTER(AdmmResultC)]),
    "nqb_admm_factorize_state_host": (C.c_int, [P, P, U32, U32, C.POINTER(AdmmConfig), P, P,
                                                P, C.POINTER(AdmmResultC), P]),
    "nqb_admm_factorize_device": (C.c_int, [P, P, U32, U32, C.POINTER(AdmmConfig), P, P, P,
                                            C.POINTER(AdmmResultC)]),
    "nqb_balance_host": (C.c_int, [P, P, P, U32, U32, U32, P, P, D, P, P, P, P, PD]),
    "nqb_factorize_layer": (C.c_int, [P, P, U32, U32, C.POINTER(AdmmConfig), D, C.c_int, PP,
                                      C.POINTER(AdmmResultC), PD]),
    "nqb_layer_rel_error": (C.c_int, [P, P, P, C.c_int, PD]),
    "nqb_top_singular_pair_host": (C.c_int, [P, P, U32, U32, I32, D, PD, P, P, PI32]),
    "nqb_spectral_norm_host": (C.c_int, [P, P, U32, U32, I32, PD]),
    "nqb_truncated_svd_host": (C.c_int, [P, P, U32, U32, U32, P, P]),
    "nqb_cholesky_solve_host": (C.c_int, [P, P, U32, P, U32, P]),
    "nqb_svid_host": (C.c_int, [P, P, U32, U32, P]),
    "nqb_admm_factor_solve_host": (C.c_int, [P, P, U32, U32, P, U32, P, P, D, D, P]),
    "nqb_augmented_lagrangian_host": (C.c_int, [P, P, P, P, P, P, P, U32, U32, U32, D, P, D,
                                                PD]),
    "nqb_group_create": (C.c_int, [P, PP, U32, PP]),
    "nqb_group_free": (C.c_int, [P]),
    "nqb_group_stream_bytes": (U64, [P]),
    "nqb_group_gemv_f16_device": (C.c_int, [P, P, P, PP]),
    "nqb_group_gemv_f32_device": (C.c_int, [P, P, P, PP]),
    "nqb_pass_create": (C.c_int, [P, U32, P, PP]),
    "nqb_pass_launch": (C.c_int, [P, P]),
    "nqb_pass_free": (C.c_int, [P]),
    "nqb_pass_run_host": (C.c_int, [P, P, P, P]),
    "nqb_pass_io_create": (C.c_int, [P, P, P, P, P]),
    "nqb_pass_io_run": (C.c_int, [P, P]),
    "nqb_pass_io_free": (C.c_int, [P]),
    "nqb_pass_stream_bytes": (U64, [P]),
    "nqb_pass_algorithmic_bytes": (U64, [P]),
    "nqb_debug_pass_trace": (C.c_int, [P, P, P, PU32]),
    "nqb_set_pdl": (C.c_int, [P, C.c_int]),
    "nqb_set_sm_budget": (C.c_int, [P, C.c_int]),
    "nqb_debug_decode_trace": (C.c_int, [P, P, P, P, P, PU32]),
    "nqb_graph_begin": (C.c_int, [P]),
    "nqb_graph_end": (C.c_int, [P, PP]),
    "nqb_graph_launch": (C.c_int, [P, P]),
    "nqb_graph_free": (C.c_int, [P]),
    "nqb_dgemm_device": (C.c_int, [P, C.c_int, C.c_int, U32, U32, U32, D, P, U32, P, U32, D,
                                   P, U32]),
    # preconditioner (precondition.cpp:37-153)
    "nqb_accumulate_stats_host": (C.c_int, [P, P, U64, U32, D, P, C.POINTER(U64), PD]),
    "nqb_accumulate_stats_device": (C.c_int, [P, P, U64, U32, D, P, C.POINTER(U64), PD]),
    "nqb_build_preconditioner": (C.c_int, [U32, P, U64, D, U32, P, U64, D, D, D, P, P, PD]),
    "nqb_precondition_weight_host": (C.c_int, [P, P, U32, U32, P, P]),
    "nqb_precondition_weight_device": (C.c_int, [P, P, U32, U32, P, P]),
    "nqb_unprecondition_rows_host": (C.c_int, [P, P, U32, U32, P]),
    # NQPK files (io.cpp:139-193)
    "nqb_nqpk_open": (C.c_int, [C.c_char_p, PP]),
    "nqb_nqpk_parse": (C.c_int, [P, U64, PP]),
    "nqb_nqpk_count": (U32, [P]),
    "nqb_nqpk_layer_info": (C.c_int, [P, U32, C.c_char_p, U32, PU32, PU32, PU32, PU32]),
    "nqb_nqpk_layer_data": (C.c_int, [P, U32, PP, PP, PP, PP]),
    "nqb_nqpk_layer_upload": (C.c_int, [P, P, U32, PP]),
    "nqb_nqpk_free": (None, [P]),
    "nqb_nqpk_serialize": (C.c_int, [U32, P, P, P, P, P, P, P, P, P, U64, C.POINTER(U64)]),
    "nqb_nqpk_write_layers": (C.c_int, [P, C.c_char_p, U32, P, P]),
}

_LIB = None


def load() -> C.CDLL:
    """Loads libnqb.so and binds every prototype; raises if anything is missing."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` or `make -C paper_2602_06694_b200/csrc` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)  # AttributeError if the symbol is missing
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def exported_symbols():
    return sorted(PROTOTYPES)
