"""Loader for the in-tree C-ABI library ``libbse_b200.so`` (include/bse_gpu.h).

No fallback: if the shared library is missing or no CUDA device is present, the compute
entry points raise instead of silently computing on the CPU.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbse_b200.so")

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dp = ctypes.c_void_p


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("pivot_index", ctypes.c_int64),
        ("relative_deviation", ctypes.c_double),
        ("message", ctypes.c_char * 256),
    ]


class PhaseTimes(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in (
        "product_pair", "cholesky", "triple", "reduce", "tridiag", "backtransform", "recover",
        "total", "panel_ms", "panel_launches", "panel_bytes", "gemm_ms", "gemm_launches",
        "gemm_flops", "gemm_dmma_flops")]


# (name, restype, argtypes) for every symbol include/bse_gpu.h declares.
SYMBOLS = {
    "bse_abi_version": (c_int, []),
    "bse_ctx_create": (c_int, [ctypes.POINTER(c_dp), c_int, ctypes.POINTER(Status)]),
    "bse_ctx_destroy": (c_int, [c_dp]),
    "bse_ctx_stream": (c_dp, [c_dp]),
    "bse_ctx_last_phase_times": (c_int, [c_dp, ctypes.POINTER(PhaseTimes)]),
    "bse_ctx_kernel_launches": (c_i64, [c_dp]),
    "bse_ctx_release_workspace": (c_int, [c_dp]),
    "bse_ctx_set_kernel_timing": (c_int, [c_dp, c_int]),
    "bse_solve": (c_int, [c_dp, c_int, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_dp, c_i64, c_dp,
                          c_dp, ctypes.POINTER(Status)]),
    "bse_solve_device": (c_int, [c_dp, c_int, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_dp, c_i64,
                                 c_dp, c_dp, ctypes.POINTER(Status)]),
    "bse_solve_batched": (c_int, [c_dp, c_int, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_dp,
                                  c_i64, c_dp, c_dp, c_dp, ctypes.POINTER(Status)]),
    "bse_solve_batched_device": (c_int, [c_dp, c_int, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp,
                                         c_dp, c_i64, c_dp, c_dp, c_dp, ctypes.POINTER(Status)]),
    "bse_ctx_set_batch_lanes": (c_int, [c_dp, c_int]),
    "bse_ctx_set_strict_certificates": (c_int, [c_dp, c_int]),
    "bse_set_tridiagonal_reduction": (c_int, [c_int]),
    "bse_product_pair": (c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_dp,
                                 ctypes.POINTER(Status)]),
    "bse_assemble_eigenvectors": (c_int, [c_dp, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp,
                                          c_dp, c_dp, c_i64, ctypes.POINTER(Status)]),
    "bse_assemble_from_squares": (c_int, [c_dp, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp,
                                          c_dp, c_dp, c_i64, c_dp, c_dp,
                                          ctypes.POINTER(Status)]),
    "bse_cholesky_lower": (c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_i64,
                                   ctypes.POINTER(Status)]),
    "bse_matmul": (c_int, [c_dp, c_i64, c_i64, c_dp, c_i64, c_int, c_int, c_i64, c_i64, c_dp,
                           c_i64, c_int, c_int, c_dp, c_i64, ctypes.POINTER(Status)]),
    "bse_tri_solve": (c_int, [c_dp, c_i64, c_dp, c_i64, c_i64, c_i64, c_dp, c_i64, c_int, c_int,
                              c_dp, c_i64, ctypes.POINTER(Status)]),
    "bse_hermitian_eig": (c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_dp, c_i64,
                                  ctypes.POINTER(Status)]),
    "bse_svd": (c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_dp, c_i64,
                        ctypes.POINTER(Status)]),
    "bse_hpd_sqrt": (c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_i64, ctypes.POINTER(Status)]),
    "bse_residual": (c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_i64, c_i64, c_dp, c_dp, c_i64, c_dp,
                             ctypes.POINTER(Status)]),
    "bse_residual_device": (c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_i64, c_i64, c_dp, c_dp,
                                    c_i64, c_dp, ctypes.POINTER(Status)]),
    "bse_sigma_orthogonality_error": (c_int, [c_dp, c_i64, c_i64, c_dp, c_i64,
                                              ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(Status)]),
    "bse_sigma_orthogonality_error_device": (c_int, [c_dp, c_i64, c_i64, c_dp, c_i64,
                                                     ctypes.POINTER(ctypes.c_double),
                                                     ctypes.POINTER(Status)]),
    "bse_check_form": (c_int, [c_dp, c_int, c_i64, c_dp, c_i64, ctypes.c_double,
                               ctypes.POINTER(c_int), ctypes.POINTER(Status)]),
    "bse_check_form_device": (c_int, [c_dp, c_int, c_i64, c_dp, c_i64, ctypes.c_double,
                                      ctypes.POINTER(c_int), ctypes.POINTER(Status)]),
    "bse_negative_spectrum": (c_int, [c_dp, c_i64, c_i64, c_dp, c_dp, c_i64, c_dp, c_dp, c_i64,
                                      ctypes.POINTER(Status)]),
    "bse_negative_spectrum_device": (c_int, [c_dp, c_i64, c_i64, c_dp, c_dp, c_i64, c_dp, c_dp,
                                             c_i64, ctypes.POINTER(Status)]),
    "bse_gen_dominant": (c_int, [c_i64, ctypes.c_uint64, c_int, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, c_dp, c_dp]),
    "bse_gen_gaussian_stream": (c_int, [ctypes.c_uint64, ctypes.c_uint64, c_i64, c_dp]),
    "bse_gen_normal": (c_int, [ctypes.c_uint64, ctypes.c_uint64, c_i64, c_dp]),
    "bse_gen_uniform": (c_int, [ctypes.c_uint64, ctypes.c_uint64, c_i64, c_dp]),
}

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compiles libbse_b200.so in-tree (nvcc, sm_100a) if it is absent."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-j8", "-C", _HERE])
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SYMBOLS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib
