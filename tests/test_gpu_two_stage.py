"""GPU parity of the two-stage tridiagonal reduction (hetrd2.cu: he2hb panel QR + DMMA her2k,
bulge chase, Q2/Q1 back-transform), selected with bse.set_tridiagonal_reduction(1).

Same tolerances as test_gpu_parity.py: eigen-decompositions against the oracle's zheevd,
solves against the oracle's CHOL / SQRT restatements (eigenvalues <= 1e-10 relative,
residual <= 100 n eps, eigenvectors up to a phase for separated eigenvalues).
"""
import numpy as np
import pytest

import oracle
import paper_2008_08825_b200 as bse
from paper_2008_08825_b200 import configs
from tests.helpers import EPS, residual, sigma_orthogonality_error, vector_phase_errors

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng(4321)


@pytest.fixture(autouse=True)
def two_stage():
    prev = bse.set_tridiagonal_reduction(1)
    yield
    bse.set_tridiagonal_reduction(prev)


def herm(n):
    x = RNG.standard_normal((n, n)) + 1j * RNG.standard_normal((n, n))
    return 0.5 * (x + x.conj().T)


# 128 is the smallest two-stage size; 129 / 161 / 300 leave partial bands and short sweeps
@pytest.mark.parametrize("n", [128, 129, 161, 192, 255, 300, 513, 1024])
def test_hermitian_eig_two_stage(n):
    m = herm(n)
    e = bse.hermitian_eig(m)
    w, vref = oracle.hermitian_eig(m)
    assert np.max(np.abs(e.values - w)) <= 100 * EPS * n * np.abs(w).max()
    bound = 100 * EPS * n
    assert np.linalg.norm(m @ e.vectors - e.vectors * e.values[None, :]) <= bound * np.linalg.norm(m)
    assert np.linalg.norm(e.vectors.conj().T @ e.vectors - np.eye(n)) <= bound
    errs, bounds, sep = vector_phase_errors(e.vectors, vref, w, np.linalg.norm(m, 2))
    assert np.all(errs[sep] <= np.maximum(bounds[sep], 1e-10))


def test_two_stage_reads_lower_only():
    m = herm(200)
    g = m.copy()
    g[np.triu_indices(200, 1)] = 1e3 + 7j
    assert np.allclose(bse.hermitian_eig(g).values, oracle.hermitian_eig(m)[0], rtol=1e-13,
                       atol=1e-13)


def test_two_stage_real_and_clustered_spectra():
    n = 256
    q, _ = np.linalg.qr(RNG.standard_normal((n, n)) + 1j * RNG.standard_normal((n, n)))
    d = np.repeat(np.arange(1.0, 9.0), n // 8)  # 8 clusters of 32 equal eigenvalues
    m = (q * d) @ q.conj().T
    e = bse.hermitian_eig(m)
    assert np.max(np.abs(e.values - np.sort(d))) <= 100 * EPS * n * 8
    assert np.linalg.norm(e.vectors.conj().T @ e.vectors - np.eye(n)) <= 100 * EPS * n
    r = np.diag(np.linspace(-3.0, 5.0, n))  # already diagonal, real
    e2 = bse.hermitian_eig(r)
    assert np.allclose(e2.values, np.linspace(-3.0, 5.0, n), rtol=0, atol=1e-13)


@pytest.mark.parametrize("n,seed", [(300, 3), (520, 5)])
def test_chol_two_stage_vs_oracle(n, seed):
    a, b = configs.config2(seed, n=n)
    h = bse.from_blocks(a, b)
    r = bse.solve_chol(h)
    lo, _, _ = oracle.solve("chol", h.a, h.b)
    assert np.max(np.abs(r.lambda_ - lo) / lo) <= 1e-10
    assert residual(h.a, h.b, r.lambda_, r.v).max() <= 100 * n * EPS
    assert sigma_orthogonality_error(r.v) <= 1e-10


def test_sqrt_two_stage_vs_oracle():
    n = 260
    a, b = configs.config2(11, n=n)
    h = bse.from_blocks(a, b)
    r = bse.solve_sqrt(h)
    lo, _, _ = oracle.solve("sqrt", h.a, h.b)
    assert np.max(np.abs(r.lambda_ - lo) / lo) <= 1e-10
    assert residual(h.a, h.b, r.lambda_, r.v).max() <= 100 * n * EPS


def test_batched_two_stage_lanes():
    """Batch lanes run the two-stage chase and panel QR with the per-lane SM cap."""
    n = 300
    hs = [bse.from_blocks(*configs.config2(s, n=n)) for s in range(3)]
    ctx = bse.Context(0)
    ctx.set_batch_lanes(2)
    res = bse.solve_batched(bse.Method.Chol, hs, ctx=ctx)
    for h, r in zip(hs, res):
        lo, _, _ = oracle.solve("chol", h.a, h.b)
        assert np.max(np.abs(r.lambda_ - lo) / lo) <= 1e-10
    ctx.close()
