"""paper_2008_08825_b200 — B200-native (sm_100a) form-I BSE eigensolver.

Python host mirror of the reference's C++ API (/root/reference/proj/include/bse/
{types,backend,solvers}.hpp) over the C-ABI library ``libbse_b200.so``
(include/bse_gpu.h). Same names, argument meaning and error classes, so the parity tests
read like the reference's doctest suites:

    h = from_blocks(a, b)                 # core.cpp:61-75 (validation + symmetrisation)
    r = solve_chol(h)                     # solvers.cpp:119-135, on the GPU
    r = solve_chol_svd(h)                 # solvers.cpp:137-161, on the GPU
    r = solve(Method.Chol, h)             # solvers.cpp:213-221

Matrices are numpy complex128 arrays (any order; copied column-major like
Eigen::MatrixXcd). Every numeric stage runs in the CUDA library; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import Status, PhaseTimes

__all__ = [
    "Method", "Side", "Op", "Shape", "Block", "BseMatrixI", "SpectralResult", "ProductPair",
    "HalfSpectralFactors", "HermitianEig", "CholeskyLower", "SvdTriple", "Error",
    "DimensionMismatch", "NotHermitian", "NotDefinite", "NotPositiveDefinite",
    "ConvergenceFailure", "SingularFactor", "NonPositiveScale", "InvalidSpec", "DeviceError",
    "from_blocks", "product_pair", "assemble_eigenvectors", "solve_chol", "solve_chol_svd",
    "solve", "negative_spectrum", "hermitian_eig", "cholesky_lower", "svd", "tri_solve", "matmul",
    "solve_sqrt", "solve_reference", "solve_batched", "solve_batched_device", "BatchError", "hpd_sqrt", "residual", "sigma_orthogonality_error",
    "check_form1", "check_form2", "check_pairing", "predicted_error", "OddDimension",
    "residual_device", "sigma_orthogonality_error_device",
    "LengthMismatch",
    "Context", "default_context", "method_name", "method_from_name", "machine_eps",
    "K_DEFAULT_HERM_TOL",
]

K_DEFAULT_HERM_TOL = 1e-12  # types.hpp:24


def machine_eps() -> float:
    return float(np.finfo(np.float64).eps)


# --------------------------------------------------------------------------- enums (types.hpp)
class Method(enum.IntEnum):
    Sqrt = 0
    Chol = 1
    CholSvd = 2
    Reference = 3


class Block(enum.IntEnum):
    M1 = 0
    M2 = 1
    Full = 2


class Side(enum.IntEnum):
    Left = 0
    Right = 1


class Op(enum.IntEnum):
    None_ = 0
    Adjoint = 1


class Shape(enum.IntEnum):
    General = 0
    Lower = 1
    Upper = 2


def method_name(m: Method) -> str:  # core.cpp:5-13
    return {Method.Sqrt: "sqrt", Method.Chol: "chol", Method.CholSvd: "chol-svd",
            Method.Reference: "reference"}.get(Method(m), "unknown")


def method_from_name(name: str) -> Method:  # core.cpp:15-21
    table = {"sqrt": Method.Sqrt, "chol": Method.Chol, "chol-svd": Method.CholSvd,
             "cholsvd": Method.CholSvd, "reference": Method.Reference}
    if name not in table:
        raise InvalidSpec("unknown method name: " + name)
    return table[name]


# --------------------------------------------------------------------------- errors (types.hpp:33-126)
class Error(RuntimeError):
    pass


class DimensionMismatch(Error):
    pass


class NotHermitian(Error):
    def __init__(self, what: str, relative_deviation: float):
        super().__init__(what)
        self.relative_deviation = relative_deviation


class NotDefinite(Error):
    def __init__(self, which: Block, what: str):
        super().__init__(what)
        self.which = Block(which)


class NotPositiveDefinite(Error):
    def __init__(self, what: str, pivot_index: int):
        super().__init__(what)
        self.pivot_index = int(pivot_index)


class ConvergenceFailure(Error):
    pass


class SingularFactor(Error):
    pass


class NonPositiveScale(Error):
    pass


class InvalidSpec(Error):
    pass


class OddDimension(Error):
    """types.hpp:99-102."""


class LengthMismatch(Error):
    """types.hpp:104-107."""


class DeviceError(Error):
    """CUDA runtime / no-device failures (no reference analogue)."""


def _raise(st: Status):
    msg = st.message.decode(errors="replace")
    c = st.code
    if c == 2:
        raise DimensionMismatch(msg)
    if c == 3:
        raise NotHermitian(msg, st.relative_deviation)
    if c == 4:
        raise NotDefinite(Block(st.block), msg)
    if c == 5:
        raise NotPositiveDefinite(msg, st.pivot_index)
    if c == 6:
        raise ConvergenceFailure(msg)
    if c == 7:
        raise SingularFactor(msg)
    if c == 8:
        raise NonPositiveScale(msg)
    if c == 9:
        raise InvalidSpec(msg)
    if c == 10:
        raise OddDimension(msg)
    if c == 11:
        raise LengthMismatch(msg)
    if c in (20, 21, 22):
        raise DeviceError(msg)
    raise Error(msg)


def _check(rc: int, st: Status):
    if rc != 0:
        _raise(st)


# --------------------------------------------------------------------------- types
@dataclass(frozen=True)
class BseMatrixI:
    """Validated pair (A, B) of Hermitian blocks (types.hpp:140-152); build via from_blocks."""
    a: np.ndarray
    b: np.ndarray

    @property
    def n(self) -> int:
        return int(self.a.shape[0])


@dataclass
class ProductPair:
    m1: np.ndarray
    m2: np.ndarray


@dataclass
class HalfSpectralFactors:
    v1: np.ndarray
    v2: np.ndarray
    lambda1: np.ndarray
    lambda2: np.ndarray


@dataclass
class SpectralResult:
    lambda_: np.ndarray  # ascending
    v: np.ndarray        # 2n x n, V^H Sigma V = I
    method: Method = Method.Reference
    near_singular: List[int] = field(default_factory=list)
    phase_ms: Optional[dict] = None


@dataclass
class HermitianEig:
    values: np.ndarray
    vectors: np.ndarray


@dataclass
class CholeskyLower:
    l: np.ndarray


@dataclass
class SvdTriple:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray


# --------------------------------------------------------------------------- context
class Context:
    """One bse_ctx (device, stream, workspace arena). Not shared across threads."""

    def __init__(self, device: int = 0):
        L = _lib.lib()
        h = ctypes.c_void_p()
        st = Status()
        _check(L.bse_ctx_create(ctypes.byref(h), int(device), ctypes.byref(st)), st)
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def phase_times(self) -> dict:
        t = PhaseTimes()
        _lib.lib().bse_ctx_last_phase_times(self._h, ctypes.byref(t))
        return {k: getattr(t, k) for k, _ in PhaseTimes._fields_}

    def set_strict_certificates(self, enable: bool = True):
        """CHOL: certify A+B by its own Cholesky on every solve, as the reference's
        product_pair does (bse_ctx_set_strict_certificates)."""
        _lib.lib().bse_ctx_set_strict_certificates(self._h, 1 if enable else 0)

    def set_kernel_timing(self, enable: bool = True):
        _lib.lib().bse_ctx_set_kernel_timing(self._h, 1 if enable else 0)

    def kernel_launches(self) -> int:
        return int(_lib.lib().bse_ctx_kernel_launches(self._h))

    def set_batch_lanes(self, lanes: int):
        """Solves in flight per batch call (1..8, default 4), see bse_ctx_set_batch_lanes."""
        if _lib.lib().bse_ctx_set_batch_lanes(self._h, int(lanes)) != 0:
            raise InvalidSpec("batch lanes must be 1..8")

    def stream(self) -> int:
        return int(_lib.lib().bse_ctx_stream(self._h) or 0)

    def release_workspace(self):
        _lib.lib().bse_ctx_release_workspace(self._h)

    def close(self):
        if self._h:
            _lib.lib().bse_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def set_tridiagonal_reduction(mode: int) -> int:
    """Process-wide tridiagonalisation inside every Hermitian eigen-decomposition: 0 one-stage
    (default), 1 two-stage (n >= 128). Returns the previous mode (bse_set_tridiagonal_reduction)."""
    return int(_lib.lib().bse_set_tridiagonal_reduction(int(mode)))


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _cm(x) -> np.ndarray:
    """Column-major complex128 copy — Eigen::MatrixXcd's layout."""
    return np.asfortranarray(np.asarray(x, dtype=np.complex128))


def _p(x: np.ndarray):
    return x.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------- core (core.cpp)
def _validated_hermitian(m: np.ndarray, tol: float, label: str) -> np.ndarray:
    """core.cpp:45-57: relative Frobenius deviation check, then (m + m^H)/2."""
    norm = float(np.linalg.norm(m))
    dev = float(np.linalg.norm(m - m.conj().T))
    if dev > tol * norm:
        rel = dev / norm if norm > 0 else dev
        raise NotHermitian(f"block {label} is not Hermitian: relative deviation {rel} exceeds "
                           f"tolerance {tol}", rel)
    return _cm(0.5 * (m + m.conj().T))


def from_blocks(a, b, tol: float = K_DEFAULT_HERM_TOL) -> BseMatrixI:
    """core.cpp:61-75."""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    if a.ndim != 2 or b.ndim != 2 or a.shape[0] != a.shape[1] or b.shape[0] != b.shape[1]:
        raise DimensionMismatch("blocks must be square")
    if a.shape[0] != b.shape[0]:
        raise DimensionMismatch(f"block dimensions differ: A is {a.shape[0]}x{a.shape[1]}, "
                                f"B is {b.shape[0]}x{b.shape[1]}")
    if a.shape[0] < 1:
        raise DimensionMismatch("blocks must be at least 1x1")
    return BseMatrixI(_validated_hermitian(a, tol, "A"), _validated_hermitian(b, tol, "B"))


def product_pair(h: BseMatrixI, ctx: Optional[Context] = None) -> ProductPair:
    """core.cpp:87-100 — (A+B, A-B), each certified by the GPU Cholesky."""
    ctx = ctx or default_context()
    n = h.n
    m1 = np.zeros((n, n), dtype=np.complex128, order="F")
    m2 = np.zeros((n, n), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_product_pair(ctx.handle, n, _p(h.a), n, _p(h.b), n, _p(m1), _p(m2),
                                       ctypes.byref(st)), st)
    return ProductPair(m1, m2)


def assemble_eigenvectors(f: HalfSpectralFactors, ctx: Optional[Context] = None) -> np.ndarray:
    """core.cpp:102-127."""
    ctx = ctx or default_context()
    v1, v2 = _cm(f.v1), _cm(f.v2)
    if v1.ndim != 2 or v2.shape != v1.shape:
        raise DimensionMismatch("factor shapes do not conform")
    n, k = v1.shape
    l1 = np.ascontiguousarray(f.lambda1, dtype=np.float64)
    l2 = np.ascontiguousarray(f.lambda2, dtype=np.float64)
    if l1.shape != (k,) or l2.shape != (k,):
        raise DimensionMismatch("factor shapes do not conform")
    v = np.zeros((2 * n, k), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_assemble_eigenvectors(ctx.handle, n, k, _p(v1), n, _p(v2), n, _p(l1),
                                                _p(l2), _p(v), 2 * n, ctypes.byref(st)), st)
    return v


def assemble_from_squares(v1: np.ndarray, v2: np.ndarray, d: np.ndarray,
                          ctx: Optional[Context] = None):
    """The recovery tail of solve_chol / solve_sqrt on the device (solvers.cpp:125, 130-133):
    lambda_from_squares(d), assemble_eigenvectors with (lambda^2, 1) and the breakdown rebuild
    of every column with d_j <= 0 (solvers.cpp:53-65). Returns (lambda, V, near_singular)."""
    ctx = ctx or default_context()
    v1, v2 = _cm(v1), _cm(v2)
    if v1.ndim != 2 or v2.shape != v1.shape:
        raise DimensionMismatch("factor shapes do not conform")
    n, k = v1.shape
    d = np.ascontiguousarray(d, dtype=np.float64)
    if d.shape != (k,):
        raise DimensionMismatch("factor shapes do not conform")
    lam = np.zeros(k)
    v = np.zeros((2 * n, k), dtype=np.complex128, order="F")
    ns = np.zeros(k, dtype=np.int64)
    nn = ctypes.c_int64(0)
    st = Status()
    _check(_lib.lib().bse_assemble_from_squares(ctx.handle, n, k, _p(v1), n, _p(v2), n, _p(d),
                                                _p(lam), _p(v), 2 * n, _p(ns), ctypes.byref(nn),
                                                ctypes.byref(st)), st)
    return lam, v, ns[: nn.value].copy()


# --------------------------------------------------------------------------- solvers (solvers.cpp)
def _solve(method: Method, h: BseMatrixI, ctx: Optional[Context]) -> SpectralResult:
    ctx = ctx or default_context()
    n = h.n
    lam = np.zeros(n)
    v = np.zeros((2 * n, n), dtype=np.complex128, order="F")
    ns = np.zeros(n, dtype=np.int64)
    nn = ctypes.c_int64(0)
    st = Status()
    rc = _lib.lib().bse_solve(ctx.handle, int(method), n, _p(h.a), n, _p(h.b), n, _p(lam), _p(v),
                              2 * n, _p(ns), ctypes.byref(nn), ctypes.byref(st))
    _check(rc, st)
    return SpectralResult(lam, v, Method(method), [int(i) for i in ns[: nn.value]],
                          ctx.phase_times())


def solve_chol(h: BseMatrixI, ctx: Optional[Context] = None) -> SpectralResult:
    """solvers.cpp:119-135 (Algorithm 2) on the GPU."""
    return _solve(Method.Chol, h, ctx)


def solve_chol_svd(h: BseMatrixI, ctx: Optional[Context] = None) -> SpectralResult:
    """solvers.cpp:137-161 (Algorithm 3) on the GPU."""
    return _solve(Method.CholSvd, h, ctx)


def solve_sqrt(h: BseMatrixI, ctx: Optional[Context] = None) -> SpectralResult:
    """solvers.cpp:94-117 (Algorithm 1, square-root form) on the GPU."""
    return _solve(Method.Sqrt, h, ctx)


def solve_reference(h: BseMatrixI, ctx: Optional[Context] = None) -> SpectralResult:
    """solvers.cpp:163-211 (Hermitian-definite pencil oracle) on the GPU (§8f row f3)."""
    return _solve(Method.Reference, h, ctx)


def solve(method: Method, h: BseMatrixI, ctx: Optional[Context] = None) -> SpectralResult:
    """solvers.cpp:213-221: dispatch over the four methods (all on the GPU)."""
    if int(method) not in (0, 1, 2, 3):
        raise InvalidSpec("unknown method")
    return _solve(Method(method), h, ctx)


class BatchError(Error):
    """A bse_solve_batched item failed: `index` is the item, `error` its typed exception
    (the payload classes above); `results` holds the items solved before it."""

    def __init__(self, index: int, error: Error, results: List[SpectralResult]):
        super().__init__(str(error))
        self.index, self.error, self.results = index, error, results


def solve_batched(method: Method, hs: List[BseMatrixI],
                  ctx: Optional[Context] = None) -> List[SpectralResult]:
    """Config-5 batch driver: the same method over independent matrices of one
    size through bse_solve_batched, which overlaps the next upload and the previous download
    with each solve (fully so for page-locked buffers; numpy arrays are pageable)."""
    ctx = ctx or default_context()
    if int(method) not in (0, 1, 2, 3):
        raise InvalidSpec("unknown method")
    if not hs:
        return []
    n = hs[0].n
    if any(h.n != n for h in hs):
        raise DimensionMismatch("batch items must share one size")
    k = len(hs)
    lams = [np.zeros(n) for _ in range(k)]
    vs = [np.zeros((2 * n, n), dtype=np.complex128, order="F") for _ in range(k)]
    ptrs = lambda arrs: (ctypes.c_void_p * k)(*[a.ctypes.data for a in arrs])  # noqa: E731
    pa, pb = ptrs([h.a for h in hs]), ptrs([h.b for h in hs])
    pl, pv = ptrs(lams), ptrs(vs)
    ns = np.zeros((k, n), dtype=np.int64)
    nn = np.zeros(k, dtype=np.int64)
    failed = ctypes.c_int64(-1)
    st = Status()
    rc = _lib.lib().bse_solve_batched(ctx.handle, int(method), n, k, pa, n, pb, n, pl, pv, 2 * n,
                                      _p(ns), _p(nn), ctypes.byref(failed), ctypes.byref(st))
    done = failed.value if rc != 0 and failed.value >= 0 else (k if rc == 0 else 0)
    out = [SpectralResult(lams[i], vs[i], Method(method), [int(j) for j in ns[i, : nn[i]]])
           for i in range(done)]
    if rc != 0:
        try:
            _check(rc, st)
        except Error as e:
            if failed.value >= 0:
                raise BatchError(failed.value, e, out) from e
            raise
    return out


def negative_spectrum(h: BseMatrixI, r: SpectralResult,
                      ctx: Optional[Context] = None) -> SpectralResult:
    """solvers.cpp:223-236: -lambda with halves swapped (bse_negative_spectrum)."""
    n = h.n
    if r.v.shape[0] != 2 * n or r.v.shape[1] != r.lambda_.shape[0]:
        raise DimensionMismatch("spectral result does not match the matrix dimension")
    ctx = ctx or default_context()
    k = r.v.shape[1]
    lam_in = np.ascontiguousarray(r.lambda_, dtype=np.float64)
    vin = _cm(r.v)
    lam = np.zeros(k)
    v = np.zeros((2 * n, k), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_negative_spectrum(ctx.handle, n, k, _p(lam_in), _p(vin), max(2 * n, 1),
                                            _p(lam), _p(v), max(2 * n, 1), ctypes.byref(st)), st)
    return SpectralResult(lam, v, r.method, list(r.near_singular))


# --------------------------------------------------------------------------- diagnostics (verify.cpp)
def residual(h: BseMatrixI, r: SpectralResult, ctx: Optional[Context] = None) -> np.ndarray:
    """verify.cpp:76-93: per-column ||H v_j - lambda_j v_j||_2 / ||H||_F (GPU, §8f row f1)."""
    ctx = ctx or default_context()
    n = h.n
    k = r.v.shape[1]
    if r.v.shape[0] != 2 * n or r.lambda_.shape[0] != k:
        raise DimensionMismatch("residual: result does not conform to the matrix")
    out = np.zeros(k)
    lam = np.ascontiguousarray(r.lambda_, dtype=np.float64)
    v = _cm(r.v)
    st = Status()
    _check(_lib.lib().bse_residual(ctx.handle, n, _p(h.a), n, _p(h.b), n, k, _p(lam), _p(v),
                                   2 * n, _p(out), ctypes.byref(st)), st)
    return out


def residual_device(n: int, a_ptr: int, b_ptr: int, k: int, lam_ptr: int, v_ptr: int,
                    out_ptr: int, ctx: Optional[Context] = None, lda: Optional[int] = None,
                    ldb: Optional[int] = None, ldv: Optional[int] = None) -> None:
    """bse_residual_device: device pointers (e.g. torch data_ptr()); out is k doubles."""
    ctx = ctx or default_context()
    st = Status()
    _check(_lib.lib().bse_residual_device(ctx.handle, n, ctypes.c_void_p(a_ptr), lda or n,
                                          ctypes.c_void_p(b_ptr), ldb or n, k,
                                          ctypes.c_void_p(lam_ptr), ctypes.c_void_p(v_ptr),
                                          ldv or 2 * n, ctypes.c_void_p(out_ptr),
                                          ctypes.byref(st)), st)


def sigma_orthogonality_error_device(rows: int, k: int, v_ptr: int,
                                     ctx: Optional[Context] = None,
                                     ldv: Optional[int] = None) -> float:
    """bse_sigma_orthogonality_error_device: V on the device, scalar result on the host."""
    ctx = ctx or default_context()
    out = ctypes.c_double(0.0)
    st = Status()
    _check(_lib.lib().bse_sigma_orthogonality_error_device(ctx.handle, rows, k,
                                                           ctypes.c_void_p(v_ptr), ldv or rows,
                                                           ctypes.byref(out), ctypes.byref(st)),
           st)
    return out.value


def sigma_orthogonality_error(v, ctx: Optional[Context] = None) -> float:
    """verify.cpp:70-74: ||V^H Sigma V - I||_F (GPU)."""
    ctx = ctx or default_context()
    v = _cm(v)
    out = ctypes.c_double(0.0)
    st = Status()
    _check(_lib.lib().bse_sigma_orthogonality_error(ctx.handle, v.shape[0], v.shape[1], _p(v),
                                                    max(v.shape[0], 1), ctypes.byref(out),
                                                    ctypes.byref(st)), st)
    return out.value


def _check_form(form: int, m, tol: float, ctx: Optional[Context]) -> bool:
    ctx = ctx or default_context()
    m = _cm(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise DimensionMismatch(f"check_form{form}: matrix must be square")
    res = ctypes.c_int(0)
    st = Status()
    _check(_lib.lib().bse_check_form(ctx.handle, form, m.shape[0], _p(m), max(m.shape[0], 1),
                                     float(tol), ctypes.byref(res), ctypes.byref(st)), st)
    return bool(res.value)


def check_form1(m, tol: float, ctx: Optional[Context] = None) -> bool:
    """verify.cpp:46-55: J m^H J = m and Sigma m^H Sigma = m within tol * ||m||_F (GPU)."""
    return _check_form(1, m, tol, ctx)


def check_form2(m, tol: float, ctx: Optional[Context] = None) -> bool:
    """verify.cpp:57-68: J m^T J = m and Sigma m^H Sigma = m within tol * ||m||_F (GPU)."""
    return _check_form(2, m, tol, ctx)


def check_pairing(pos, neg, tol: float) -> bool:
    """verify.cpp:95-106: sorted(pos) vs sorted(-neg) within tol * max|pos| (host: an
    O(n log n) sort, no device work)."""
    pos = np.asarray(pos, dtype=np.float64)
    neg = np.asarray(neg, dtype=np.float64)
    if pos.shape != neg.shape:
        raise LengthMismatch("check_pairing: spectra have different lengths")
    scale = np.abs(pos).max() if pos.size else 0.0
    return bool(np.all(np.abs(np.sort(pos) - np.sort(-neg)) <= tol * scale))


def predicted_error(norm_h: float, lam: float, s_lambda: float = 1.0, eps: float = None,
                    squared_method: bool = False) -> float:
    """verify.cpp:108-114: first-order eigenvalue error model (host scalar formula)."""
    eps = machine_eps() if eps is None else eps
    if squared_method:
        return eps * (norm_h / s_lambda) * min(norm_h / lam, 1.0 / np.sqrt(eps))
    return eps * norm_h / s_lambda


def solve_device(method: Method, n: int, a_ptr: int, b_ptr: int, lam_ptr: int, v_ptr: int,
                 ctx: Optional[Context] = None, lda: Optional[int] = None,
                 ldb: Optional[int] = None, ldv: Optional[int] = None) -> List[int]:
    """bse_solve_device: device pointers (e.g. torch tensors' data_ptr()) in and out."""
    ctx = ctx or default_context()
    ns = np.zeros(max(n, 1), dtype=np.int64)
    nn = ctypes.c_int64(0)
    st = Status()
    rc = _lib.lib().bse_solve_device(ctx.handle, int(method), n, ctypes.c_void_p(a_ptr),
                                     lda or n, ctypes.c_void_p(b_ptr), ldb or n,
                                     ctypes.c_void_p(lam_ptr), ctypes.c_void_p(v_ptr),
                                     ldv or 2 * n, _p(ns), ctypes.byref(nn), ctypes.byref(st))
    _check(rc, st)
    return [int(i) for i in ns[: nn.value]]


def solve_batched_device(method: Method, n: int, a_ptrs: List[int], b_ptrs: List[int],
                         lam_ptrs: List[int], v_ptrs: List[int],
                         ctx: Optional[Context] = None) -> List[List[int]]:
    """bse_solve_batched_device: a batch resident in device memory (column-major a, b with
    ld n; lambda n; v 2n x n with ld 2n). Returns each item's near-singular indices."""
    ctx = ctx or default_context()
    k = len(a_ptrs)
    if not (len(b_ptrs) == len(lam_ptrs) == len(v_ptrs) == k):
        raise LengthMismatch("solve_batched_device: pointer lists differ in length")
    arr = lambda xs: (ctypes.c_void_p * max(k, 1))(*xs)  # noqa: E731
    ns = np.zeros((max(k, 1), max(n, 1)), dtype=np.int64)
    nn = np.zeros(max(k, 1), dtype=np.int64)
    failed = ctypes.c_int64(-1)
    st = Status()
    rc = _lib.lib().bse_solve_batched_device(ctx.handle, int(method), n, k, arr(a_ptrs), n,
                                             arr(b_ptrs), n, arr(lam_ptrs), arr(v_ptrs), 2 * n,
                                             _p(ns), _p(nn), ctypes.byref(failed),
                                             ctypes.byref(st))
    _check(rc, st)
    return [[int(j) for j in ns[i, : nn[i]]] for i in range(k)]


# --------------------------------------------------------------------------- backend (backend.cpp)
def hermitian_eig(m, ctx: Optional[Context] = None) -> HermitianEig:
    """backend.cpp:28-45 (zheevd 'V','L': reads the lower triangle only)."""
    ctx = ctx or default_context()
    m = _cm(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise DimensionMismatch(f"hermitian_eig: matrix is {m.shape[0]}x{m.shape[1]}, expected square")
    n = m.shape[0]
    w = np.zeros(n)
    vec = np.zeros((n, n), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_hermitian_eig(ctx.handle, n, _p(m), n, _p(w), _p(vec), n,
                                        ctypes.byref(st)), st)
    return HermitianEig(w, vec)


def hpd_sqrt(m, ctx: Optional[Context] = None) -> np.ndarray:
    """backend.cpp:88-107: Hermitian square root of an HPD matrix (GPU, §8f row f2)."""
    ctx = ctx or default_context()
    m = _cm(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise DimensionMismatch(f"hpd_sqrt: matrix is {m.shape[0]}x{m.shape[1]}, expected square")
    n = m.shape[0]
    out = np.zeros((n, n), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_hpd_sqrt(ctx.handle, n, _p(m), n, _p(out), n, ctypes.byref(st)), st)
    return out


def cholesky_lower(m, ctx: Optional[Context] = None) -> CholeskyLower:
    """backend.cpp:47-62."""
    ctx = ctx or default_context()
    m = _cm(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise DimensionMismatch(f"cholesky_lower: matrix is {m.shape[0]}x{m.shape[1]}, expected square")
    n = m.shape[0]
    out = np.zeros((n, n), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_cholesky_lower(ctx.handle, n, _p(m), n, _p(out), n, ctypes.byref(st)),
           st)
    return CholeskyLower(out)


def svd(m, ctx: Optional[Context] = None) -> SvdTriple:
    """backend.cpp:64-86 (s descending, v not v^H)."""
    ctx = ctx or default_context()
    m = _cm(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise DimensionMismatch(f"svd: matrix is {m.shape[0]}x{m.shape[1]}, expected square")
    n = m.shape[0]
    u = np.zeros((n, n), dtype=np.complex128, order="F")
    v = np.zeros((n, n), dtype=np.complex128, order="F")
    s = np.zeros(n)
    st = Status()
    _check(_lib.lib().bse_svd(ctx.handle, n, _p(m), n, _p(u), n, _p(s), _p(v), n,
                              ctypes.byref(st)), st)
    return SvdTriple(u, s, v)


def tri_solve(l: CholeskyLower, rhs, side: Side = Side.Left, op: Op = Op.None_,
              ctx: Optional[Context] = None) -> np.ndarray:
    """backend.cpp:109-129."""
    ctx = ctx or default_context()
    L = _cm(l.l)
    if L.shape[0] != L.shape[1]:
        raise DimensionMismatch("tri_solve: matrix is not square")
    x0 = _cm(rhs)
    rows, cols = x0.shape
    x = np.zeros((rows, cols), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_tri_solve(ctx.handle, L.shape[0], _p(L), L.shape[0], rows, cols, _p(x0),
                                    max(rows, 1), int(side), int(op), _p(x), max(rows, 1),
                                    ctypes.byref(st)), st)
    return x


def matmul(a, b, op_a: Op = Op.None_, shape_a: Shape = Shape.General, op_b: Op = Op.None_,
           shape_b: Shape = Shape.General, ctx: Optional[Context] = None) -> np.ndarray:
    """backend.cpp:131-175 (MatmulOpts as keyword arguments)."""
    ctx = ctx or default_context()
    a, b = _cm(a), _cm(b)
    am = a.shape[0] if op_a == Op.None_ else a.shape[1]
    bn = b.shape[1] if op_b == Op.None_ else b.shape[0]
    c = np.zeros((am, bn), dtype=np.complex128, order="F")
    st = Status()
    _check(_lib.lib().bse_matmul(ctx.handle, a.shape[0], a.shape[1], _p(a), max(a.shape[0], 1),
                                 int(op_a), int(shape_a), b.shape[0], b.shape[1], _p(b),
                                 max(b.shape[0], 1), int(op_b), int(shape_b), _p(c),
                                 max(am, 1), ctypes.byref(st)), st)
    return c
