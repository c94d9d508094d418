"""Deterministic parity of the CHOL recovery tail:
lambda_from_squares (solvers.cpp:25-45) -> assemble_eigenvectors with (lambda^2, 1)
(core.cpp:102-127) -> rebuild_nonpositive_columns (solvers.cpp:53-65).

Crafted inputs: random factors V1, V2 and a squared spectrum d holding every case of the
clamp/rebuild contract at once - negative d (rebuilt with the pi/4 quarter root), d = 0
(rebuilt at the floor), positive d whose root falls below eps*sqrt(d_max) (clamped and flagged,
not rebuilt) and ordinary positive d.

CPU (not gpu): the oracle's restatement against a numpy transcription of the three reference
functions. GPU: bse_assemble_from_squares (the same launches the CHOL solve runs after its
eigensolve) against the oracle, column by column.
"""
import numpy as np
import pytest

import oracle

EPS = float(np.finfo(float).eps)


def crafted(n=48, seed=11):
    rng = np.random.default_rng(seed)
    d = np.array([-3.0e-2, -1.0e-20, 0.0, 1.0e-40, 2.5e-33, 1.0e-6, 0.37, 1.0, 2.0, 4.0])
    k = d.size
    v1 = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    v2 = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    return np.asfortranarray(v1), np.asfortranarray(v2), d


def numpy_restatement(v1, v2, d):
    """solvers.cpp:25-45 + core.cpp:102-127 (factors (lambda^2, 1)) + solvers.cpp:53-65."""
    n, k = v1.shape
    floor = EPS * np.sqrt(d[-1])
    lam = np.where(d > 0, np.sqrt(np.maximum(d, 0.0)), 0.0)
    flagged = [j for j in range(k) if lam[j] < floor]
    nonpos = [j for j in flagged if not d[j] > 0]
    lam = np.where(lam < floor, floor, lam)
    l1 = lam * lam
    s1, s2 = (l1 / 1.0) ** 0.25, (1.0 / l1) ** 0.25
    x, y = v1 * s1[None, :], v2 * s2[None, :]
    v = np.vstack([0.5 * (x + y), 0.5 * (y - x)])
    for j in nonpos:
        mag = max(np.sqrt(abs(d[j])), floor)
        q = np.sqrt(mag) * complex(np.sqrt(2.0) / 2.0, np.sqrt(2.0) / 2.0)
        xj, yj = v1[:, j] * q, v2[:, j] / q
        v[:n, j] = 0.5 * (xj + yj)
        v[n:, j] = 0.5 * (yj - xj)
    return lam, v, np.array(flagged, dtype=np.int64), nonpos


def test_oracle_recovery_tail_matches_reference_formulas():
    v1, v2, d = crafted()
    lam, v, flags = oracle.assemble_from_squares(v1, v2, d)
    lr, vr, fr, nonpos = numpy_restatement(v1, v2, d)
    assert nonpos == [0, 1, 2]          # d < 0 twice and d == 0 are rebuilt
    assert list(flags) == [0, 1, 2, 3, 4]  # + two tiny positive d clamped, not rebuilt
    assert np.array_equal(lam, lr)
    assert np.allclose(v, vr, rtol=0, atol=4 * EPS * np.abs(vr).max())
    # Sigma-norm |top|^2 - |bottom|^2 = Re(x^H y): Re(v1^H v2) for assembled columns, but
    # Im(v1^H v2) for rebuilt ones - the pi/4 phase rotates x against y, which is the
    # "honest breakdown" signature the reference keeps (solvers.cpp:47-52)
    n = v1.shape[0]
    sig = np.sum(np.abs(v[:n]) ** 2 - np.abs(v[n:]) ** 2, axis=0)
    ip = np.sum(v1.conj() * v2, axis=0)
    expect = np.where(np.isin(np.arange(d.size), nonpos), ip.imag, ip.real)
    assert np.all(np.isfinite(v))
    # (tolerance relative to the column's norm^2: clamped columns carry 1/sqrt(floor) scales)
    assert np.all(np.abs(sig - expect) <= 1e-12 * np.sum(np.abs(v) ** 2, axis=0))


def test_oracle_recovery_tail_no_positive_entry():
    v1, v2, _ = crafted()
    d = np.linspace(-1.0, 0.0, v1.shape[1])
    with pytest.raises(oracle.OracleError) as e:
        oracle.assemble_from_squares(v1, v2, d)
    assert e.value.code == 6  # ConvergenceFailure (solvers.cpp:28-30)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 48, 333])
def test_recovery_tail_gpu_matches_oracle(n):
    import paper_2008_08825_b200 as bse
    v1, v2, d = crafted(n=n, seed=n)
    lam_o, v_o, f_o = oracle.assemble_from_squares(v1, v2, d)
    lam, v, flags = bse.assemble_from_squares(v1, v2, d)
    assert list(flags) == list(f_o)
    assert np.array_equal(lam, lam_o)  # sqrt / clamp are exact operations
    # column by column: the rebuilt columns (0..2) and the assembled ones, a few ulps
    scale = np.abs(v_o).max(axis=0)
    err = np.abs(v - v_o).max(axis=0) / scale
    assert np.all(err <= 8 * EPS), err


@pytest.mark.gpu
def test_recovery_tail_gpu_no_positive_entry():
    import paper_2008_08825_b200 as bse
    v1, v2, _ = crafted()
    with pytest.raises(bse.ConvergenceFailure):
        bse.assemble_from_squares(v1, v2, np.linspace(-1.0, 0.0, v1.shape[1]))
