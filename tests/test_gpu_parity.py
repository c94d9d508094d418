"""GPU parity: the CUDA path through the C-ABI against the CPU oracle (oracle/), the
reference's known-answer tests and the committed golden fixtures.

Tolerances (BASELINE.json north_star):
  * eigenvalues: relative error <= 1e-10 vs the oracle for the same method;
  * residual ||Hx - lambda x|| / (||H||_F ||x||) <= 100 n eps;
  * eigenvectors equal up to a unit phase within c eps ||H|| / gap (c = 1e3) for
    well-separated eigenvalues (the reference accepts any basis of a cluster);
  * backend factors: reconstruction <= 100 eps n ||M|| (test_backend.cpp:13-14).
"""
import ctypes
import glob
import os

import numpy as np
import pytest

import oracle
import paper_2008_08825_b200 as bse
from paper_2008_08825_b200 import configs
from tests.helpers import (EPS, check_pairing, norm_h, residual, residual_ref,
                           sigma_orthogonality_error, vector_phase_errors)

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SQ3 = np.sqrt(3.0)
RNG = np.random.default_rng(1234)
SIZES = [1, 2, 3, 7, 16, 33, 64, 65, 100, 127, 128, 129, 255, 256, 257, 300]


def crand(*shape):
    return RNG.standard_normal(shape) + 1j * RNG.standard_normal(shape)


def herm(n):
    x = crand(n, n)
    return 0.5 * (x + x.conj().T)


def hpd(n):
    m = herm(n)
    return m + (np.abs(m).sum(axis=0).max() + 1.0) * np.eye(n)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def assert_solution(a, b, r, ref_lam=None, ref_v=None, lam_tol=1e-10):
    n = a.shape[0]
    assert r.lambda_.shape == (n,) and r.v.shape == (2 * n, n)
    assert np.all(np.isfinite(r.lambda_)) and np.all(np.isfinite(r.v))
    assert np.all(np.diff(r.lambda_) >= 0) and r.lambda_[0] > 0
    keep = np.setdiff1d(np.arange(n), r.near_singular)
    res = residual(a, b, r.lambda_[keep], r.v[:, keep])
    assert res.max() <= 100 * n * EPS, res.max()
    if ref_lam is not None:
        err = np.max(np.abs(r.lambda_ - ref_lam) / np.abs(ref_lam))
        assert err <= lam_tol, err
    if ref_v is not None:
        errs, bounds, sep = vector_phase_errors(r.v, ref_v, r.lambda_, norm_h(a, b))
        sep &= np.isin(np.arange(n), keep)
        assert np.all(errs[sep] <= np.maximum(bounds[sep], 1e-10)), (errs[sep] / bounds[sep]).max()


# ------------------------------------------------------------------ dense backend
@pytest.mark.parametrize("n", SIZES)
def test_cholesky_lower(n):
    m = hpd(n)
    l = bse.cholesky_lower(m).l
    assert rel(l, oracle.cholesky_lower(m)) < 1e-13
    assert np.linalg.norm(l @ l.conj().T - m) <= 100 * EPS * n * np.linalg.norm(m)
    assert np.all(np.triu(l, 1) == 0) and np.all(np.diag(l).real > 0)
    assert np.all(np.diag(l).imag == 0)


@pytest.mark.parametrize("n", [2, 5, 64, 65, 130, 200])
def test_cholesky_pivot_index(n):
    """test_backend.cpp:78-85, 237-254: the first failing pivot matches LAPACK's info."""
    m = hpd(n)
    k = n // 2
    m[k, k] = -abs(m[k, k])
    with pytest.raises(bse.NotPositiveDefinite) as e:
        bse.cholesky_lower(m)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.cholesky_lower(m)
    assert e.value.pivot_index == eo.value.pivot_index


def test_backend_kats_gpu():
    e = bse.hermitian_eig(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(e.values, [1.0, 3.0], rtol=1e-14)
    d = bse.hermitian_eig(np.diag([3.0, 1.0]))
    assert np.allclose(d.values, [1.0, 3.0]) and abs(abs(d.vectors[1, 0]) - 1) < 1e-14
    l = bse.cholesky_lower(np.array([[4.0, 2.0], [2.0, 5.0]])).l
    assert np.array_equal(l, np.array([[2.0, 0.0], [1.0, 2.0]]))
    assert np.array_equal(bse.cholesky_lower(np.eye(5)).l, np.eye(5))
    with pytest.raises(bse.NotPositiveDefinite) as ex:
        bse.cholesky_lower(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert ex.value.pivot_index == 1
    t = bse.svd(np.diag([2.0, 1.0]))
    assert np.allclose(t.s, [2.0, 1.0])
    t = bse.svd(np.array([[SQ3]]))
    assert abs(t.s[0] - SQ3) < 1e-15 and abs(abs(t.u[0, 0]) - 1) < 1e-15
    assert np.allclose(bse.svd(np.array([[0.0, 1.0], [-1.0, 0.0]])).s, [1.0, 1.0])
    L = bse.CholeskyLower(np.array([[2.0, 0.0], [1.0, 2.0]], dtype=complex))
    assert np.allclose(bse.tri_solve(L, np.array([[4.0], [4.0]])).real.ravel(), [2.0, 1.0])
    assert np.allclose(bse.tri_solve(L, np.array([[2.0], [2.0]]), bse.Side.Left,
                                     bse.Op.Adjoint).real.ravel(), [0.5, 1.0])
    with pytest.raises(bse.SingularFactor):
        bse.tri_solve(bse.CholeskyLower(np.array([[1.0, 0.0], [1.0, 0.0]])), np.eye(2))
    p = bse.matmul(L.l, L.l, op_a=bse.Op.Adjoint)
    assert np.allclose(p.real, [[5.0, 2.0], [2.0, 4.0]])
    with pytest.raises(bse.DimensionMismatch):
        bse.matmul(np.eye(2), np.eye(3))
    assert bse.matmul(np.zeros((2, 3)), np.zeros((2, 3)), op_a=bse.Op.Adjoint).shape == (3, 3)


@pytest.mark.parametrize("n", [1, 7, 64, 129, 257])
@pytest.mark.parametrize("opa,opb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_matmul_general(n, opa, opb):
    a = crand(n + 3, n) if opa else crand(n, n + 3)
    b = crand(n - 1 if n > 1 else 1, n + 3) if opb else crand(n + 3, max(n - 1, 1))
    c = bse.matmul(a, b, op_a=bse.Op(opa), op_b=bse.Op(opb))
    ref = oracle.matmul(a, b, opa, 0, opb, 0)
    assert rel(c, ref) < 1e-14


@pytest.mark.parametrize("n", [1, 13, 64, 100, 257])
@pytest.mark.parametrize("shape", [1, 2])
@pytest.mark.parametrize("op", [0, 1])
def test_matmul_triangular_hints(n, shape, op):
    """test_backend.cpp:215-229 + ztrmm semantics: only the hinted triangle is read."""
    t = crand(n, n)
    x = crand(n, n + 2)
    ref = oracle.matmul(t, x, op, shape, 0, 0)
    assert rel(bse.matmul(t, x, op_a=bse.Op(op), shape_a=bse.Shape(shape)), ref) < 1e-14
    y = crand(n + 2, n)
    ref = oracle.matmul(y, t, 0, 0, op, shape)
    assert rel(bse.matmul(y, t, op_b=bse.Op(op), shape_b=bse.Shape(shape)), ref) < 1e-14


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("side,op", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_tri_solve(n, side, op):
    l = oracle.cholesky_lower(hpd(n))
    rhs = crand(n, n + 5) if side == 0 else crand(n + 5, n)
    x = bse.tri_solve(bse.CholeskyLower(l), rhs, bse.Side(side), bse.Op(op))
    assert rel(x, oracle.tri_solve(l, rhs, side, op)) < 1e-12


@pytest.mark.parametrize("n", SIZES)
def test_hermitian_eig(n):
    m = herm(n)
    e = bse.hermitian_eig(m)
    w, vref = oracle.hermitian_eig(m)
    assert np.max(np.abs(e.values - w)) <= 100 * EPS * n * np.abs(w).max()
    bound = 100 * EPS * n
    assert np.linalg.norm(m @ e.vectors - e.vectors * e.values[None, :]) <= bound * np.linalg.norm(m)
    assert np.linalg.norm(e.vectors.conj().T @ e.vectors - np.eye(n)) <= bound
    errs, bounds, sep = vector_phase_errors(e.vectors, vref, w, np.linalg.norm(m, 2))
    assert np.all(errs[sep] <= np.maximum(bounds[sep], 1e-10))


def test_hermitian_eig_reads_lower_only():
    """zheevd 'L' semantics (backend.cpp:34): garbage in the strict upper triangle is ignored."""
    m = herm(50)
    g = m.copy()
    g[np.triu_indices(50, 1)] = 1e3 + 7j
    assert np.allclose(bse.hermitian_eig(g).values, oracle.hermitian_eig(m)[0], rtol=1e-13,
                       atol=1e-13)


@pytest.mark.parametrize("n", SIZES)
def test_svd(n):
    m = crand(n, n)
    t = bse.svd(m)
    _, s, _ = oracle.svd(m)
    assert np.max(np.abs(t.s - s)) <= 100 * EPS * n * s[0]
    bound = 100 * EPS * n
    assert np.linalg.norm(m - (t.u * t.s[None, :]) @ t.v.conj().T) <= bound * np.linalg.norm(m)
    assert np.linalg.norm(t.u.conj().T @ t.u - np.eye(n)) <= bound
    assert np.linalg.norm(t.v.conj().T @ t.v - np.eye(n)) <= bound
    assert np.all(np.diff(t.s) <= 0)


# ------------------------------------------------------------------ core glue
def test_product_pair_and_errors():
    a, b = configs.generate_random_definite(20, 4)
    h = bse.from_blocks(a, b)
    pp = bse.product_pair(h)
    m1, m2 = oracle.product_pair(h.a, h.b)
    assert np.array_equal(pp.m1, m1) and np.array_equal(pp.m2, m2)
    with pytest.raises(bse.NotDefinite) as e:
        bse.product_pair(bse.from_blocks(np.array([[1.0]]), np.array([[2.0]])))
    assert e.value.which == bse.Block.M2
    with pytest.raises(bse.NotDefinite) as e:
        bse.product_pair(bse.from_blocks(np.array([[1.0]]), np.array([[-2.0]])))
    assert e.value.which == bse.Block.M1


def test_assemble_eigenvectors_gpu():
    v = bse.assemble_eigenvectors(bse.HalfSpectralFactors(np.array([[3 ** 0.25]]),
                                                          np.array([[3 ** -0.25]]),
                                                          np.array([1.0]), np.array([1.0])))
    assert abs(v[0, 0] - 1.0379549) < 1e-7 and abs(v[1, 0] + 0.2781192) < 1e-7
    v1, v2 = crand(9, 4), crand(9, 4)
    l1, l2 = RNG.uniform(0.5, 3, 4), RNG.uniform(0.5, 3, 4)
    got = bse.assemble_eigenvectors(bse.HalfSpectralFactors(v1, v2, l1, l2))
    assert rel(got, oracle.assemble_eigenvectors(v1, v2, l1, l2)) < 1e-15
    with pytest.raises(bse.NonPositiveScale):
        bse.assemble_eigenvectors(bse.HalfSpectralFactors(v1, v2, -l1, l2))
    with pytest.raises(bse.NonPositiveScale):
        bse.assemble_eigenvectors(bse.HalfSpectralFactors(v1, v2, l1 * np.inf, l2))


# ------------------------------------------------------------------ solver KATs (test_solvers.cpp)
@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_canonical_1x1_gpu(method):
    r = bse.solve(method, bse.from_blocks(np.array([[2.0]]), np.array([[1.0]])))
    assert abs(r.lambda_[0] - SQ3) <= 1e-13 * SQ3
    ph = r.v[0, 0] / abs(r.v[0, 0])
    assert abs(r.v[0, 0] / ph - 0.5 * (3 ** 0.25 + 3 ** -0.25)) < 1e-12
    assert abs(r.v[1, 0] / ph - 0.5 * (3 ** -0.25 - 3 ** 0.25)) < 1e-12
    assert r.method == method and r.near_singular == []


@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_decoupled_gpu(method):
    a = np.diag([3.0, 1.0, 2.0])
    r = bse.solve(method, bse.from_blocks(a, np.zeros((3, 3))))
    assert np.allclose(r.lambda_, [1, 2, 3], rtol=1e-13)
    assert np.linalg.norm(r.v[3:]) < 1e-12
    assert np.allclose(np.linalg.norm(r.v, axis=0), 1.0, atol=1e-12)


@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_indefinite_gpu(method):
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve(method, bse.from_blocks(np.array([[1.0]]), np.array([[2.0]])))
    assert e.value.which == bse.Block.M2
    a, b = configs.generate_random_definite(30, 2)
    b = b + 5 * np.abs(a).max() * np.eye(30)  # A-B indefinite, A+B definite
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve(method, bse.from_blocks(a, b))
    assert e.value.which == bse.Block.M2
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve(method, bse.from_blocks(a, -b))  # A+B indefinite: M1 checked first
    assert e.value.which == bse.Block.M1


def test_conditioned_kappa10_gpu():
    a, b = configs.generate_conditioned(50, 10.0, 3)
    for m in (bse.Method.Chol, bse.Method.CholSvd):
        r = bse.solve(m, bse.from_blocks(a, b))
        assert abs(r.lambda_[0] - SQ3 / 2) / (SQ3 / 2) < 1e-12 and r.near_singular == []


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_oracle_equivalence_gpu(seed):
    """test_solvers.cpp:90-105 on the GPU path."""
    a, b = configs.generate_random_definite(16, seed)
    h = bse.from_blocks(a, b)
    lr, _, _ = oracle.solve("reference", h.a, h.b)
    for m in (bse.Method.Chol, bse.Method.CholSvd):
        r = bse.solve(m, h)
        assert np.max(np.abs(r.lambda_ - lr) / np.abs(lr)) < 1e-10
        assert residual_ref(h.a, h.b, r.lambda_, r.v).max() < 1e-12
        assert sigma_orthogonality_error(r.v) < 1e-11


def test_ordering_pairing_negative_gpu():
    a, b = configs.generate_random_definite(24, 5)
    h = bse.from_blocks(a, b)
    for m in (bse.Method.Chol, bse.Method.CholSvd):
        r = bse.solve(m, h)
        assert r.lambda_.shape == (24,) and r.lambda_[0] > 0 and np.all(np.diff(r.lambda_) >= 0)
        neg = bse.negative_spectrum(h, r)
        assert check_pairing(r.lambda_, neg.lambda_, 1e-14)
        assert np.array_equal(neg.v[:24], r.v[24:])


def test_sigma_orthonormality_kappa1e3_gpu():
    a, b = configs.generate_conditioned(40, 1000.0, 13)
    for m in (bse.Method.Chol, bse.Method.CholSvd):
        assert sigma_orthogonality_error(bse.solve(m, bse.from_blocks(a, b)).v) <= 1e-10 * 40


@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_clamp_and_flag_gpu(method):
    a = np.diag([1e-40, 1.0])
    r = bse.solve(method, bse.from_blocks(a, np.zeros((2, 2))))
    lo, vo, nso = oracle.solve(int(method), a, np.zeros((2, 2)))
    assert r.near_singular == [0] == nso
    assert abs(r.lambda_[0] - EPS) <= 1e-6 * EPS
    assert np.all(np.isfinite(r.lambda_)) and np.all(np.isfinite(r.v))
    assert abs(r.lambda_[1] - 1.0) < 1e-12
    assert np.allclose(np.abs(r.v), np.abs(vo), rtol=1e-10, atol=1e-6)


def test_breakdown_regime_gpu():
    a, b = configs.generate_conditioned(200, 1e10, 1)
    r = bse.solve_chol_svd(bse.from_blocks(a, b))
    assert sigma_orthogonality_error(r.v) < 1e-8
    # CHOL far beyond the squaring barrier: finite, clamp contract respected (whether the
    # garbage smallest squares come out <= eps*d_max depends on rounding)
    rc = bse.solve_chol(bse.from_blocks(a, b))
    assert np.all(np.isfinite(rc.lambda_)) and np.all(np.isfinite(rc.v))
    assert np.all(rc.lambda_ >= EPS * rc.lambda_[-1] * (1 - 1e-12))


def test_all_methods_dispatch():
    """solvers.cpp:213-221: every method runs (SQRT / REFERENCE composed on the GPU, §8f)."""
    h = bse.from_blocks(np.array([[2.0]]), np.array([[1.0]]))
    for m in (bse.Method.Sqrt, bse.Method.Chol, bse.Method.CholSvd, bse.Method.Reference):
        r = bse.solve(m, h)
        assert abs(r.lambda_[0] - np.sqrt(3.0)) <= 1e-14 and r.method == m
    with pytest.raises(bse.InvalidSpec):
        bse.solve(7, h)


def test_from_blocks_contract():
    with pytest.raises(bse.NotHermitian):
        bse.from_blocks(np.array([[0.0, 1.0], [0.0, 0.0]]), np.zeros((2, 2)))
    with pytest.raises(bse.DimensionMismatch):
        bse.from_blocks(np.eye(2), np.eye(3))


# ------------------------------------------------------------------ golden fixtures
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden(path):
    g = np.load(path)
    m = bse.method_from_name(str(g["method"]))
    r = bse.solve(m, bse.from_blocks(g["a"], g["b"]))
    assert r.near_singular == list(g["near_singular"])
    assert_solution(g["a"], g["b"], r, g["lam"], g["v"])


# ------------------------------------------------------------------ configs vs oracle
def _oracle_threads():
    oracle.set_threads(os.cpu_count() or 1)


@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 64, 97, 256, 512])
def test_config1_real(n):
    """Config 1 (real fp64 n=512 through the complex path) and its small versions."""
    _oracle_threads()
    a, b = configs.config1(0, n=n)
    lo, vo, _ = oracle.solve("chol", a, b)
    assert_solution(a, b, bse.solve_chol(bse.from_blocks(a, b)), lo, vo)


@pytest.mark.parametrize("n", [40, 200, 513, 2048])
def test_config2_chol(n):
    _oracle_threads()
    a, b = configs.config2(1, n=n)
    lo, vo, _ = oracle.solve("chol", a, b)
    assert_solution(a, b, bse.solve_chol(bse.from_blocks(a, b)), lo, vo)


@pytest.mark.parametrize("n", [40, 256, 512])
def test_config2_chol_svd(n):
    _oracle_threads()
    a, b = configs.config2(2, n=n)
    lo, vo, _ = oracle.solve("chol-svd", a, b)
    assert_solution(a, b, bse.solve_chol_svd(bse.from_blocks(a, b)), lo, vo)


@pytest.mark.parametrize("n", [64, 300, 600])
def test_config3_ill_conditioned(n):
    """Config 3 generator (lambda_min(H) ~ 1e-3): CHOL+SVD gated at 1e-10 against the oracle;
    CHOL's error against CHOL+SVD within 10x the CPU CHOL error (squaring penalty,
    PAPER.md:566-571)."""
    _oracle_threads()
    a, b = configs.config3(0, n=n)
    ls, vs, _ = oracle.solve("chol-svd", a, b)
    r = bse.solve_chol_svd(bse.from_blocks(a, b))
    assert_solution(a, b, r, ls, vs)
    lc, _, _ = oracle.solve("chol", a, b)
    rc = bse.solve_chol(bse.from_blocks(a, b))
    cpu_err = np.abs(lc - ls) / ls
    gpu_err = np.abs(rc.lambda_ - r.lambda_) / r.lambda_
    # squared-eigenvalue error model: eps (||H|| / lambda)^2 per eigenvalue
    model = 100 * EPS * (r.lambda_[-1] / r.lambda_) ** 2
    assert np.all(gpu_err <= np.maximum(10 * cpu_err, model)), (gpu_err / np.maximum(10 * cpu_err, model)).max()


# ------------------------------------------------------------------ C-ABI specifics
def test_leading_dimensions_and_determinism():
    """bse_solve with lda, ldb > n and ldv > 2n; bitwise determinism across calls."""
    n, pad = 37, 5
    a, b = configs.config2(3, n=n)
    ap = np.zeros((n + pad, n), dtype=complex, order="F")
    bp = np.zeros((n + pad, n), dtype=complex, order="F")
    ap[:n], bp[:n] = a, b
    L = bse._lib.lib()
    ctx = bse.default_context()
    outs = []
    for _ in range(2):
        lam = np.zeros(n)
        v = np.zeros((2 * n + 3, n), dtype=complex, order="F")
        ns = np.zeros(n, dtype=np.int64)
        nn = ctypes.c_int64(0)
        st = bse.Status()
        rc = L.bse_solve(ctx.handle, 1, n, ap.ctypes.data_as(ctypes.c_void_p), n + pad,
                         bp.ctypes.data_as(ctypes.c_void_p), n + pad,
                         lam.ctypes.data_as(ctypes.c_void_p), v.ctypes.data_as(ctypes.c_void_p),
                         2 * n + 3, ns.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nn),
                         ctypes.byref(st))
        assert rc == 0, st.message
        outs.append((lam, v[: 2 * n]))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    lo, vo, _ = oracle.solve("chol", a, b)
    assert np.max(np.abs(outs[0][0] - lo) / lo) < 1e-12


def test_kernel_launch_counter_moves(ctx):
    before = ctx.kernel_launches()
    a, b = configs.config2(0, n=64)
    bse.solve_chol(bse.from_blocks(a, b), ctx=ctx)
    assert ctx.kernel_launches() > before + 10


def test_cpp_dropin_binary(tmp_path):
    """The reference-style C++ test (tests/cpp/test_dropin.cpp) against include/bse/*.hpp."""
    import subprocess
    root = os.path.dirname(HERE)
    libdir = os.path.join(root, "paper_2008_08825_b200")
    exe = tmp_path / "test_dropin"
    subprocess.check_call(["g++", "-std=c++20", f"-I{root}/include",
                           os.path.join(HERE, "cpp", "test_dropin.cpp"), f"-L{libdir}",
                           "-lbse_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


# ------------------------------------------------------------------ degenerate / clustered spectra
@pytest.mark.parametrize("n", [3, 64, 100, 300])
@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_fully_degenerate_spectrum(n, method):
    """kappa = 3 in the conditioned family: every eigenvalue equals sqrt(3)/2 (the D&C
    deflates everything); any orthonormal basis is acceptable."""
    a, b = configs.generate_conditioned(n, 3.0, 5)
    r = bse.solve(method, bse.from_blocks(a, b))
    assert np.allclose(r.lambda_, SQ3 / 2, rtol=1e-12)
    assert residual(a, b, r.lambda_, r.v).max() <= 100 * n * EPS
    assert sigma_orthogonality_error(r.v) <= 1e-10 * n


@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_identity_and_repeated_diagonal(method):
    for a in (np.eye(150), np.diag(np.repeat([1.0, 2.0, 3.0], 70))):
        n = a.shape[0]
        r = bse.solve(method, bse.from_blocks(a, np.zeros((n, n))))
        assert np.allclose(r.lambda_, np.sort(np.diag(a)), rtol=1e-13)
        assert residual(a, np.zeros((n, n)), r.lambda_, r.v).max() <= 100 * n * EPS
        assert sigma_orthogonality_error(r.v) <= 1e-10 * n


@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_clustered_spectrum(method):
    """Tight clusters (gaps ~1e-9 relative) mixed with isolated eigenvalues."""
    n = 240
    q = configs.random_unitary(n, 17)
    d = np.concatenate([1.0 + 1e-9 * np.arange(80), 2.0 + 1e-12 * np.arange(80),
                        np.linspace(3.0, 9.0, 80)])
    a = (q.conj().T * d[None, :]) @ q
    a = 0.5 * (a + a.conj().T)
    b = 0.25 * a
    h = bse.from_blocks(a, b)
    r = bse.solve(method, h)
    lo, _, _ = oracle.solve(int(method), h.a, h.b)
    assert np.max(np.abs(r.lambda_ - lo) / lo) <= 1e-10
    assert residual(h.a, h.b, r.lambda_, r.v).max() <= 100 * n * EPS
    assert sigma_orthogonality_error(r.v) <= 1e-10 * n


@pytest.mark.parametrize("n", [2, 33, 200])
def test_hermitian_eig_degenerate(n):
    """Backend eig on a diagonal / identity / rank-1-perturbed identity."""
    for m in (np.eye(n), np.diag(np.arange(n) % 3 + 1.0),
              np.eye(n) + 1e-3 * np.outer(np.ones(n), np.ones(n))):
        e = bse.hermitian_eig(m)
        w = np.linalg.eigvalsh(m)
        assert np.max(np.abs(e.values - w)) <= 100 * EPS * n * np.abs(w).max()
        assert np.linalg.norm(m @ e.vectors - e.vectors * e.values[None, :]) <= 100 * EPS * n * max(np.linalg.norm(m), 1)
        assert np.linalg.norm(e.vectors.conj().T @ e.vectors - np.eye(n)) <= 100 * EPS * n
