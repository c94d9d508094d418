"""Parity metrics (restating proj/src/verify.cpp) used by the tests. Test-only code."""
from __future__ import annotations

import numpy as np

EPS = float(np.finfo(np.float64).eps)


def residual(a, b, lam, v):
    """verify.cpp:72-90 per column, additionally divided by ||x||:
    ||H x - lambda x|| / (||H||_F ||x||) with H = [A B; -B -A]."""
    n = a.shape[0]
    top, bot = v[:n], v[n:]
    ht = a @ top + b @ bot
    hb = -(b @ top) - a @ bot
    nh = np.sqrt(2 * np.linalg.norm(a) ** 2 + 2 * np.linalg.norm(b) ** 2)
    r = np.sqrt(np.linalg.norm(ht - top * lam[None, :], axis=0) ** 2 +
                np.linalg.norm(hb - bot * lam[None, :], axis=0) ** 2)
    return r / (nh * np.linalg.norm(v, axis=0))


def residual_ref(a, b, lam, v):
    """verify.cpp:72-90 exactly (no ||x|| normalisation)."""
    n = a.shape[0]
    top, bot = v[:n], v[n:]
    ht = a @ top + b @ bot
    hb = -(b @ top) - a @ bot
    nh = np.sqrt(2 * np.linalg.norm(a) ** 2 + 2 * np.linalg.norm(b) ** 2)
    return np.sqrt(np.linalg.norm(ht - top * lam[None, :], axis=0) ** 2 +
                   np.linalg.norm(hb - bot * lam[None, :], axis=0) ** 2) / nh


def sigma_orthogonality_error(v):
    """verify.cpp:66-70: ||V^H Sigma V - I||_F."""
    n = v.shape[0] // 2
    sv = np.vstack([v[:n], -v[n:]])
    return float(np.linalg.norm(v.conj().T @ sv - np.eye(v.shape[1])))


def check_pairing(pos, neg, tol):
    """verify.cpp:92-102."""
    p = np.sort(pos)
    m = np.sort(-neg)
    scale = np.abs(pos).max() if len(pos) else 0.0
    return bool(np.all(np.abs(p - m) <= tol * scale))


def vector_phase_errors(v, vref, lam, norm_h, c=1e3):
    """Eigenvectors equal up to phase: theta = arg(vref^H v),
    ||v - e^{i theta} vref|| / ||vref||, compared against c * eps * ||H|| / gap_j. Returns
    (errors, bounds, mask_of_well_separated_columns)."""
    k = v.shape[1]
    lam = np.asarray(lam)
    gaps = np.full(k, np.inf)
    if k > 1:
        d = np.diff(lam)
        gaps[:-1] = np.minimum(gaps[:-1], d)
        gaps[1:] = np.minimum(gaps[1:], d)
    errs = np.zeros(k)
    for j in range(k):
        ip = np.vdot(vref[:, j], v[:, j])
        ph = ip / abs(ip) if abs(ip) > 0 else 1.0
        errs[j] = np.linalg.norm(v[:, j] - ph * vref[:, j]) / np.linalg.norm(vref[:, j])
    bounds = c * EPS * norm_h / np.maximum(gaps, 1e-300)
    separated = gaps > 1e3 * EPS * norm_h
    return errs, bounds, separated


def norm_h(a, b):
    return float(np.sqrt(2 * np.linalg.norm(a) ** 2 + 2 * np.linalg.norm(b) ** 2))
