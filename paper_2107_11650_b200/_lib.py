"""ctypes loader for the in-tree C-ABI library ``lib/libshlr_b200.so``.

There is no fallback: if the library is missing or fails to load, importing
the product API raises.  The C-ABI is declared in ``include/shlr_cuda.h``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SHLR_LIB_PATH") or os.path.join(_HERE, "lib", "libshlr_b200.so")

SHLR_OK = 0
SHLR_EINVAL = 1
SHLR_EDIVERGE = 4
SHLR_ECUDA = 5
SHLR_EUNSUPPORTED = 6

LOG_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_char_p)


class ShlrPiArgs(C.Structure):
    _fields_ = [
        ("m", C.c_size_t), ("n", C.c_size_t), ("j", C.c_size_t),
        ("y", C.POINTER(C.c_double)),
        ("mask", C.POINTER(C.c_uint8)),
        ("mask_rows", C.c_size_t),
        ("spirit_weights", C.POINTER(C.c_double)),
        ("spirit_k", C.c_size_t),
        ("taps", C.POINTER(C.c_double)),
        ("ntaps", C.c_size_t),
        ("pencil_row", C.c_size_t), ("pencil_col", C.c_size_t),
        ("lam", C.c_double), ("lambda1", C.c_double), ("beta", C.c_double),
        ("tau", C.c_double), ("tol", C.c_double), ("cg_tol", C.c_double),
        ("max_outer", C.c_size_t), ("cg_max", C.c_size_t),
        ("enable_spirit", C.c_int), ("enable_vc", C.c_int),
        ("debug_sv_iter", C.c_int),
    ]


class ShlrParamArgs(C.Structure):
    _fields_ = [
        ("m", C.c_size_t), ("n", C.c_size_t), ("l", C.c_size_t), ("j", C.c_size_t),
        ("y", C.POINTER(C.c_double)),
        ("mask", C.POINTER(C.c_uint8)),
        ("taps", C.POINTER(C.c_double)),
        ("ntaps", C.c_size_t),
        ("pencil_pe", C.c_size_t), ("pencil_par", C.c_size_t),
        ("lam", C.c_double), ("lambda2", C.c_double), ("beta", C.c_double),
        ("tau", C.c_double), ("tol", C.c_double), ("cg_tol", C.c_double),
        ("max_outer", C.c_size_t), ("cg_max", C.c_size_t),
        ("enable_vc", C.c_int),
        ("slice_begin", C.c_size_t), ("slice_end", C.c_size_t),
        ("hybrid_input", C.c_int),
    ]


class ShlrStats(C.Structure):
    _fields_ = [("outer_iters", C.c_size_t), ("final_rel_change", C.c_double)]


# Every exported symbol and its prototype; tests check the .so exports all of
# them (the same list as include/shlr_cuda.h).
PROTOTYPES = {
    "shlr_cuda_abi_version": (C.c_int, []),
    "shlr_cuda_last_error": (C.c_char_p, []),
    "shlr_cuda_device_count": (C.c_int, []),
    "shlr_cuda_pi_reconstruct": (C.c_int, [C.POINTER(ShlrPiArgs), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(ShlrStats),
                                           LOG_FN, C.c_void_p]),
    "shlr_cuda_debug_normal_apply": (C.c_int, [C.POINTER(ShlrPiArgs), C.POINTER(C.c_double),
                                               C.POINTER(C.c_double)]),
    "shlr_cuda_pi_plan_create": (C.c_int, [C.POINTER(ShlrPiArgs), C.POINTER(C.c_void_p)]),
    "shlr_cuda_pi_plan_reset": (C.c_int, [C.c_void_p]),
    "shlr_cuda_pi_plan_run": (C.c_int, [C.c_void_p, C.c_size_t]),
    "shlr_cuda_pi_plan_sync": (C.c_int, [C.c_void_p]),
    "shlr_cuda_pi_plan_timing": (C.c_int, [C.c_void_p, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "shlr_cuda_pi_plan_download": (C.c_int, [C.c_void_p, C.POINTER(C.c_double),
                                             C.POINTER(ShlrStats), LOG_FN, C.c_void_p]),
    "shlr_cuda_pi_plan_destroy": (None, [C.c_void_p]),
    "shlr_cuda_pi_plan_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "shlr_cuda_pi_plan_set_warm_start": (C.c_int, [C.c_void_p, C.c_int]),
    "shlr_cuda_pi_plan_debug_sweeps": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.c_int]),
    "shlr_cuda_pi_plan_debug_levels": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.c_int]),
    "shlr_cuda_pi_plan_debug_phases": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]),
    "shlr_cuda_param_reconstruct": (C.c_int, [C.POINTER(ShlrParamArgs), C.POINTER(C.c_double),
                                              C.POINTER(ShlrStats), LOG_FN, C.c_void_p]),
    "shlr_cuda_param_plan_create": (C.c_int, [C.POINTER(ShlrParamArgs), C.POINTER(C.c_void_p)]),
    "shlr_cuda_param_plan_reset": (C.c_int, [C.c_void_p]),
    "shlr_cuda_param_plan_run": (C.c_int, [C.c_void_p, C.c_size_t]),
    "shlr_cuda_param_plan_sync": (C.c_int, [C.c_void_p]),
    "shlr_cuda_param_plan_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "shlr_cuda_param_plan_timing": (C.c_int, [C.c_void_p, C.POINTER(C.c_double),
                                              C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "shlr_cuda_param_plan_download": (C.c_int, [C.c_void_p, C.POINTER(C.c_double),
                                                C.POINTER(ShlrStats), LOG_FN, C.c_void_p]),
    "shlr_cuda_param_plan_destroy": (None, [C.c_void_p]),
    "shlr_cuda_fp32_peak_tflops": (C.c_int, [C.POINTER(C.c_double)]),
    "shlr_cuda_hankel_svt_batched": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.c_float, C.c_void_p, C.c_void_p, C.c_void_p]),
    "shlr_cuda_hankel_svt_batched_host": (C.c_int, [C.POINTER(C.c_double), C.c_int, C.c_int,
                                                    C.c_int, C.c_int, C.c_double,
                                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "shlr_cuda_debug_svt_sweeps": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_float, C.c_void_p, C.c_void_p]),
    "shlr_cuda_lift_index_map": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_int32)]),
    "shlr_cuda_lift_index_map_path": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                C.POINTER(C.c_int32)]),
    "shlr_cuda_fft_along_axis": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_size_t), C.c_int,
                                           C.c_int, C.c_int]),
    "shlr_cuda_ssos": (C.c_int, [C.POINTER(C.c_double), C.c_size_t, C.c_size_t, C.c_size_t,
                                 C.POINTER(C.c_double)]),
    "shlr_cuda_rlne": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t,
                                 C.POINTER(C.c_double)]),
    "shlr_cuda_mssim": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t, C.c_size_t,
                                  C.POINTER(C.c_double)]),
    "shlr_mask_gauss_cartesian": (C.c_int, [C.c_size_t, C.c_double, C.c_size_t, C.c_uint64,
                                            C.POINTER(C.c_uint8)]),
    "shlr_mask_random2d": (C.c_int, [C.c_size_t, C.c_size_t, C.c_double, C.c_size_t, C.c_uint64,
                                     C.POINTER(C.c_uint8)]),
    "shlr_acs_range": (C.c_int, [C.c_size_t, C.c_size_t, C.POINTER(C.c_size_t),
                                 C.POINTER(C.c_size_t)]),
    "shlr_pencil_for": (C.c_size_t, [C.c_size_t, C.c_size_t]),
    "shlr_pencil_for_param": (C.c_size_t, [C.c_size_t, C.c_size_t]),
    "shlr_spirit_calibrate": (C.c_int, [C.POINTER(C.c_double), C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.c_size_t, C.c_double, C.POINTER(C.c_double)]),
    "shlr_cuda_spirit_calibrate": (C.c_int, [C.POINTER(C.c_double), C.c_size_t, C.c_size_t, C.c_size_t,
                                             C.c_size_t, C.c_double, C.POINTER(C.c_double)]),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2107_11650_b200/csrc).  There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    return (lib.shlr_cuda_last_error() or b"").decode()
