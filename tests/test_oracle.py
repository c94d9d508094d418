"""Pins the CPU oracle (oracle/, LAPACK restatement) against the reference's own known-answer
tests (proj/tests/test_solvers.cpp, test_backend.cpp, test_core.cpp; SPEC.md examples), an
independent scipy restatement, and the committed golden fixtures. CPU only."""
import glob
import os

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from tests.helpers import EPS, check_pairing, residual_ref, sigma_orthogonality_error

SQ3 = np.sqrt(3.0)
HERE = os.path.dirname(os.path.abspath(__file__))


def _gen():
    from paper_2008_08825_b200 import configs
    return configs


# ------------------------------------------------------------------ solver KATs (test_solvers.cpp)
@pytest.mark.parametrize("method", ["sqrt", "chol", "chol-svd", "reference"])
def test_canonical_1x1(method):
    """test_solvers.cpp:33-42 — A=[2], B=[1]: lambda=sqrt(3), v~[1.0379549; -0.2781192]."""
    lam, v, ns = oracle.solve(method, np.array([[2.0]]), np.array([[1.0]]))
    assert abs(lam[0] - SQ3) <= 1e-13 * SQ3
    top = 0.5 * (3 ** 0.25 + 3 ** -0.25)
    bottom = 0.5 * (3 ** -0.25 - 3 ** 0.25)
    ph = v[0, 0] / abs(v[0, 0])
    assert abs(v[0, 0] / ph - top) < 1e-12 and abs(v[1, 0] / ph - bottom) < 1e-12
    assert abs(top - 1.0379549) < 1e-7 and abs(bottom + 0.2781192) < 1e-7
    assert ns == []


@pytest.mark.parametrize("method", ["sqrt", "chol", "chol-svd", "reference"])
def test_decoupled(method):
    """test_solvers.cpp:24-31,44-53 — B=0, A=diag(3,1,2) -> lambda=(1,2,3), bottom half 0."""
    a = np.diag([3.0, 1.0, 2.0]).astype(complex)
    lam, v, _ = oracle.solve(method, a, np.zeros((3, 3)))
    assert np.allclose(lam, [1, 2, 3], rtol=1e-13)
    assert np.linalg.norm(v[3:]) < 1e-12
    assert np.allclose(np.linalg.norm(v, axis=0), 1.0, atol=1e-12)


@pytest.mark.parametrize("method", ["sqrt", "chol", "chol-svd", "reference"])
def test_indefinite(method):
    """test_solvers.cpp:73-79 — A=[1], B=[2] -> NotDefinite{M2}."""
    with pytest.raises(oracle.OracleError) as e:
        oracle.solve(method, np.array([[1.0]]), np.array([[2.0]]))
    assert e.value.code == 4 and e.value.block == 1


def test_conditioned_kappa10():
    """test_solvers.cpp:81-88 — conditioned n=50 kappa=10 seed 3: lambda_min = sqrt(3)/2."""
    a, b = _gen().generate_conditioned(50, 10.0, 3)
    for m in ["sqrt", "chol", "chol-svd", "reference"]:
        lam, _, ns = oracle.solve(m, a, b)
        assert abs(lam[0] - SQ3 / 2) / (SQ3 / 2) < 1e-12
        assert ns == []


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_oracle_equivalence(seed):
    """test_solvers.cpp:90-105 — random definite n=16 vs the pencil oracle."""
    a, b = _gen().generate_random_definite(16, seed)
    lr, vr, _ = oracle.solve("reference", a, b)
    for m in ["sqrt", "chol", "chol-svd"]:
        lam, v, _ = oracle.solve(m, a, b)
        assert np.max(np.abs(lam - lr) / np.abs(lr)) < 1e-10
        assert residual_ref(a, b, lam, v).max() < 1e-12
        assert sigma_orthogonality_error(v) < 1e-11
    assert residual_ref(a, b, lr, vr).max() < 1e-12


def test_ordering_and_pairing():
    """test_solvers.cpp:107-115, 160-166 — ascending, positive, pairing symmetric."""
    a, b = _gen().generate_random_definite(24, 5)
    for m in ["sqrt", "chol", "chol-svd", "reference"]:
        lam, v, _ = oracle.solve(m, a, b)
        assert lam.shape == (24,) and lam[0] > 0 and np.all(np.diff(lam) >= 0)
        assert check_pairing(lam, -lam, 1e-14)


def test_sigma_orthonormality_kappa1e3():
    """test_solvers.cpp:160-166 — n=40 kappa=1e3 seed 13: ||V^H Sigma V - I|| <= 1e-10 n."""
    a, b = _gen().generate_conditioned(40, 1000.0, 13)
    for m in ["sqrt", "chol", "chol-svd", "reference"]:
        _, v, _ = oracle.solve(m, a, b)
        assert sigma_orthogonality_error(v) <= 1e-10 * 40


@pytest.mark.parametrize("method", ["chol", "chol-svd"])
def test_clamp_and_flag(method):
    """test_solvers.cpp:168-186 — A=diag(1e-40,1), B=0: near_singular=[0], lambda0=eps."""
    a = np.diag([1e-40, 1.0]).astype(complex)
    lam, v, ns = oracle.solve(method, a, np.zeros((2, 2)))
    assert ns == [0]
    assert abs(lam[0] - EPS) <= 1e-6 * EPS
    assert np.all(np.isfinite(lam)) and np.all(np.isfinite(v))
    assert abs(lam[1] - 1.0) < 1e-12


def test_breakdown_regime():
    """test_solvers.cpp:188-199 — kappa=1e10: chol-svd stays Sigma-orthonormal."""
    a, b = _gen().generate_conditioned(200, 1e10, 1)
    lam, v, ns = oracle.solve("sqrt", a, b)
    assert np.all(np.isfinite(lam)) and np.all(np.isfinite(v)) and ns
    assert sigma_orthogonality_error(v) > 1e-4
    _, vg, _ = oracle.solve("chol-svd", a, b)
    assert sigma_orthogonality_error(vg) < 1e-8


# ------------------------------------------------------------------ backend KATs (test_backend.cpp)
def test_backend_kats():
    w, _ = oracle.hermitian_eig(np.array([[2.0, 1.0], [1.0, 2.0]]))  # :47-52
    assert np.allclose(w, [1.0, 3.0], rtol=1e-14)
    l = oracle.cholesky_lower(np.array([[4.0, 2.0], [2.0, 5.0]]))   # :65-71
    assert np.array_equal(l, np.array([[2.0, 0.0], [1.0, 2.0]]))
    with pytest.raises(oracle.OracleError) as e:                     # :78-85
        oracle.cholesky_lower(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.code == 5 and e.value.pivot_index == 1
    u, s, v = oracle.svd(np.diag([2.0, 1.0]))                        # :100-118
    assert np.allclose(s, [2.0, 1.0])
    _, s, _ = oracle.svd(np.array([[0.0, 1.0], [-1.0, 0.0]]))
    assert np.allclose(s, [1.0, 1.0])
    lt = np.array([[2.0, 0.0], [1.0, 2.0]])                          # :175-191
    assert np.allclose(oracle.tri_solve(lt, np.array([[4.0], [4.0]]), 0, 0).real.ravel(), [2.0, 1.0])
    assert np.allclose(oracle.tri_solve(lt, np.array([[2.0], [2.0]]), 0, 1).real.ravel(), [0.5, 1.0])
    with pytest.raises(oracle.OracleError) as e:                     # :193-196
        oracle.tri_solve(np.array([[1.0, 0.0], [1.0, 0.0]]), np.eye(2), 0, 0)
    assert e.value.code == 7
    p = oracle.matmul(lt, lt, 1, 0, 0, 0)                            # :198-213
    assert np.allclose(p.real, [[5.0, 2.0], [2.0, 4.0]])


def test_backend_random_reconstruction():
    """test_backend.cpp:54-63, 87-98, 120-131 with c = 100."""
    cf = _gen()
    for n in (3, 17, 64):
        m = cf.random_hermitian(n, 100 + n)
        w, vec = oracle.hermitian_eig(m)
        bound = 100 * EPS * n
        assert np.linalg.norm(m @ vec - vec * w[None, :]) <= bound * np.linalg.norm(m)
        assert np.linalg.norm(vec.conj().T @ vec - np.eye(n)) <= bound
    m = cf.random_hermitian(32, 7)
    m = m + (np.abs(m).sum(axis=0).max() + 1.0) * np.eye(32)
    l = oracle.cholesky_lower(m)
    assert np.linalg.norm(l @ l.conj().T - m) <= 100 * EPS * 32 * np.linalg.norm(m)
    assert np.all(np.diag(l).imag == 0) and np.all(np.diag(l).real > 0)


def test_assemble_kats():
    """SPEC.md assemble_eigenvectors examples; test_core.cpp:100-138."""
    v = oracle.assemble_eigenvectors(np.array([[3 ** 0.25]]), np.array([[3 ** -0.25]]),
                                     np.array([1.0]), np.array([1.0]))
    assert abs(v[0, 0] - 1.0379549) < 1e-7 and abs(v[1, 0] + 0.2781192) < 1e-7
    e1 = np.eye(3)[:, :1]
    v = oracle.assemble_eigenvectors(e1, e1, np.array([1.0]), np.array([1.0]))
    assert np.allclose(v[:3], e1) and np.allclose(v[3:], 0)
    with pytest.raises(oracle.OracleError) as e:
        oracle.assemble_eigenvectors(e1, e1, np.array([0.0]), np.array([1.0]))
    assert e.value.code == 8


def test_product_pair_errors():
    """test_core.cpp:86-93 — NotDefinite names the failing block."""
    with pytest.raises(oracle.OracleError) as e:
        oracle.product_pair(np.array([[1.0]]), np.array([[2.0]]))
    assert e.value.code == 4 and e.value.block == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.product_pair(np.array([[1.0]]), np.array([[-2.0]]))
    assert e.value.code == 4 and e.value.block == 0


# ------------------------------------------------------------------ independent restatement
def test_oracle_vs_scipy_restatement():
    """The oracle's CHOL/CHOL+SVD against an independent scipy.linalg restatement of
    solvers.cpp:119-161 (different wrapper, same LAPACK algorithms)."""
    a, b = _gen().generate_random_definite(20, 3)
    m1, m2 = a + b, a - b
    l = sla.cholesky(m2, lower=True)
    m = l.conj().T @ m1 @ l
    d, vm = sla.eigh(m, driver="evd")
    lam = np.sqrt(d)
    lam_o, v_o, _ = oracle.solve("chol", a, b)
    assert np.max(np.abs(lam - lam_o) / lam) < 1e-13
    l1 = sla.cholesky(m1, lower=True)
    s = sla.svd(l1.conj().T @ l, compute_uv=False)[::-1]
    lam_s, _, _ = oracle.solve("chol-svd", a, b)
    assert np.max(np.abs(s - lam_s) / s) < 1e-13


# ------------------------------------------------------------------ golden fixtures
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_matches_golden(path):
    g = np.load(path)
    lam, v, ns = oracle.solve(str(g["method"]), g["a"], g["b"])
    assert np.max(np.abs(lam - g["lam"]) / np.abs(g["lam"])) < 1e-12
    assert list(ns) == list(g["near_singular"])
    keep = np.setdiff1d(np.arange(len(lam)), ns)  # clamped columns carry no accuracy guarantee
    assert residual_ref(g["a"], g["b"], lam[keep], v[:, keep]).max() < 1e-10


def test_golden_present():
    assert len(GOLDEN) >= 8
