"""CPU ORACLE — test infrastructure only.

ctypes front end of ``oracle/libbse_oracle.so``, the LAPACK restatement of the reference's
hot path (``/root/reference/proj/src/{backend,core,solvers}.cpp``; see bse_oracle.cpp).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import this package, and only as the checker or the timed CPU
baseline. The product path (``paper_2008_08825_b200``) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libbse_oracle.so")

METHOD = {"sqrt": 0, "chol": 1, "chol-svd": 2, "cholsvd": 2, "reference": 3}


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("pivot_index", ctypes.c_int64),
        ("relative_deviation", ctypes.c_double),
        ("message", ctypes.c_char * 256),
    ]


class OracleError(RuntimeError):
    def __init__(self, st: Status):
        super().__init__(st.message.decode(errors="replace"))
        self.code = st.code
        self.block = st.block
        self.pivot_index = st.pivot_index


def build() -> str:
    if not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_blas_config.restype = ctypes.c_char_p
    return _lib


def _c(x: np.ndarray) -> np.ndarray:
    """Column-major complex128 copy (the reference's Eigen::MatrixXcd layout)."""
    return np.asfortranarray(np.asarray(x, dtype=np.complex128))


def _p(x: np.ndarray):
    return x.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, st: Status):
    if rc != 0:
        raise OracleError(st)


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def blas_config() -> str:
    return lib().oracle_blas_config().decode()


def solve(method, a: np.ndarray, b: np.ndarray):
    """solvers.cpp:213-221. Returns (lambda ascending, V 2n x n, near_singular list)."""
    m = METHOD[method] if isinstance(method, str) else int(method)
    a, b = _c(a), _c(b)
    n = a.shape[0]
    lam = np.zeros(n)
    v = np.zeros((2 * n, n), dtype=np.complex128, order="F")
    ns = np.zeros(max(n, 1), dtype=np.int64)
    nn = ctypes.c_int64(0)
    st = Status()
    rc = lib().oracle_solve(ctypes.c_int(m), ctypes.c_int64(n), _p(a), _p(b), _p(lam), _p(v),
                            _p(ns), ctypes.byref(nn), ctypes.byref(st))
    _check(rc, st)
    return lam, v, [int(i) for i in ns[: nn.value]]


def cholesky_lower(m: np.ndarray) -> np.ndarray:
    m = _c(m)
    n = m.shape[0]
    out = np.zeros((n, n), dtype=np.complex128, order="F")
    st = Status()
    _check(lib().oracle_cholesky_lower(ctypes.c_int64(n), _p(m), _p(out), ctypes.byref(st)), st)
    return out


def hermitian_eig(m: np.ndarray):
    m = _c(m)
    n = m.shape[0]
    w = np.zeros(n)
    vec = np.zeros((n, n), dtype=np.complex128, order="F")
    st = Status()
    _check(lib().oracle_hermitian_eig(ctypes.c_int64(n), _p(m), _p(w), _p(vec),
                                      ctypes.byref(st)), st)
    return w, vec


def svd(m: np.ndarray):
    m = _c(m)
    n = m.shape[0]
    u = np.zeros((n, n), dtype=np.complex128, order="F")
    v = np.zeros((n, n), dtype=np.complex128, order="F")
    s = np.zeros(n)
    st = Status()
    _check(lib().oracle_svd(ctypes.c_int64(n), _p(m), _p(u), _p(s), _p(v), ctypes.byref(st)), st)
    return u, s, v


def tri_solve(l: np.ndarray, rhs: np.ndarray, side: int = 0, op: int = 0) -> np.ndarray:
    l, rhs = _c(l), _c(rhs)
    x = np.zeros(rhs.shape, dtype=np.complex128, order="F")
    st = Status()
    _check(lib().oracle_tri_solve(ctypes.c_int64(l.shape[0]), _p(l), ctypes.c_int64(rhs.shape[0]),
                                  ctypes.c_int64(rhs.shape[1]), _p(rhs), ctypes.c_int(side),
                                  ctypes.c_int(op), _p(x), ctypes.byref(st)), st)
    return x


def matmul(a, b, op_a=0, shape_a=0, op_b=0, shape_b=0) -> np.ndarray:
    a, b = _c(a), _c(b)
    rows = a.shape[0] if op_a == 0 else a.shape[1]
    cols = b.shape[1] if op_b == 0 else b.shape[0]
    c = np.zeros((rows, cols), dtype=np.complex128, order="F")
    st = Status()
    _check(lib().oracle_matmul(ctypes.c_int64(a.shape[0]), ctypes.c_int64(a.shape[1]), _p(a),
                               ctypes.c_int(op_a), ctypes.c_int(shape_a),
                               ctypes.c_int64(b.shape[0]), ctypes.c_int64(b.shape[1]), _p(b),
                               ctypes.c_int(op_b), ctypes.c_int(shape_b), _p(c),
                               ctypes.byref(st)), st)
    return c


def product_pair(a, b):
    a, b = _c(a), _c(b)
    n = a.shape[0]
    m1 = np.zeros((n, n), dtype=np.complex128, order="F")
    m2 = np.zeros((n, n), dtype=np.complex128, order="F")
    st = Status()
    _check(lib().oracle_product_pair(ctypes.c_int64(n), _p(a), _p(b), _p(m1), _p(m2),
                                     ctypes.byref(st)), st)
    return m1, m2


def assemble_eigenvectors(v1, v2, l1, l2):
    v1, v2 = _c(v1), _c(v2)
    n, k = v1.shape
    l1 = np.ascontiguousarray(l1, dtype=np.float64)
    l2 = np.ascontiguousarray(l2, dtype=np.float64)
    v = np.zeros((2 * n, k), dtype=np.complex128, order="F")
    st = Status()
    _check(lib().oracle_assemble_eigenvectors(ctypes.c_int64(n), ctypes.c_int64(k), _p(v1),
                                              _p(v2), _p(l1), _p(l2), _p(v),
                                              ctypes.byref(st)), st)
    return v


def assemble_from_squares(v1, v2, d):
    """solvers.cpp:125, 130-133: (lambda, V, near_singular) from the squared spectrum d and
    the factors V1, V2, including the breakdown rebuild (solvers.cpp:53-65)."""
    v1, v2 = _c(v1), _c(v2)
    n, k = v1.shape
    d = np.ascontiguousarray(d, dtype=np.float64)
    lam = np.zeros(k)
    v = np.zeros((2 * n, k), dtype=np.complex128, order="F")
    flags = np.zeros(k, dtype=np.int64)
    nf = ctypes.c_int64(0)
    st = Status()
    _check(lib().oracle_assemble_from_squares(ctypes.c_int64(n), ctypes.c_int64(k), _p(v1),
                                              _p(v2), _p(d), _p(lam), _p(v), _p(flags),
                                              ctypes.byref(nf), ctypes.byref(st)), st)
    return lam, v, flags[: nf.value].copy()
