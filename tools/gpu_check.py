"""Quick GPU-vs-oracle smoke across the building blocks (dev tool; tests/ hold the gates)."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

rng = np.random.default_rng(0)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def herm(n):
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return 0.5 * (x + x.conj().T)


def step(name, fn):
    t = time.time()
    try:
        out = fn()
        print(f"[ok ] {name:40s} {out}  ({time.time()-t:.2f}s)", flush=True)
    except Exception as e:  # noqa
        print(f"[ERR] {name:40s} {type(e).__name__}: {e}", flush=True)
        traceback.print_exc()


def t_gemm(n, opa, opb):
    a = rng.standard_normal((n, n + 3)) + 1j * rng.standard_normal((n, n + 3))
    b = rng.standard_normal((n + 3, n - 1)) + 1j * rng.standard_normal((n + 3, n - 1))
    if opa:
        a = a.conj().T.copy()
    if opb:
        b = b.conj().T.copy()
    c = bse.matmul(a, b, op_a=bse.Op(opa), op_b=bse.Op(opb))
    ref = (a.conj().T if opa else a) @ (b.conj().T if opb else b)
    return rel(c, ref)


def t_trmm(n):
    m = herm(n) + 2 * n * np.eye(n)
    l = np.linalg.cholesky(m)
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    out = []
    for opa in (0, 1):
        c = bse.matmul(l, x, op_a=bse.Op(opa), shape_a=bse.Shape.Lower)
        out.append(rel(c, (l.conj().T if opa else l) @ x))
        c = bse.matmul(x, l, op_b=bse.Op(opa), shape_b=bse.Shape.Lower)
        out.append(rel(c, x @ (l.conj().T if opa else l)))
    return max(out)


def t_potrf(n):
    m = herm(n) + 2 * n * np.eye(n)
    l = bse.cholesky_lower(m).l
    lo = oracle.cholesky_lower(m)
    return rel(l, lo), rel(l @ l.conj().T, m)


def t_trsm(n):
    m = herm(n) + 2 * n * np.eye(n)
    l = np.linalg.cholesky(m)
    x = rng.standard_normal((n, n + 5)) + 1j * rng.standard_normal((n, n + 5))
    out = []
    for op in (0, 1):
        sol = bse.tri_solve(bse.CholeskyLower(l), x, bse.Side.Left, bse.Op(op))
        out.append(rel(sol, oracle.tri_solve(l, x, 0, op)))
    xr = x.T.copy()
    for op in (0, 1):
        sol = bse.tri_solve(bse.CholeskyLower(l), xr, bse.Side.Right, bse.Op(op))
        out.append(rel(sol, oracle.tri_solve(l, xr, 1, op)))
    return max(out)


def t_heev(n):
    m = herm(n)
    e = bse.hermitian_eig(m)
    w, _ = oracle.hermitian_eig(m)
    res = np.linalg.norm(m @ e.vectors - e.vectors * e.values[None, :]) / np.linalg.norm(m)
    orth = np.linalg.norm(e.vectors.conj().T @ e.vectors - np.eye(n))
    return float(np.max(np.abs(e.values - w)) / np.max(np.abs(w))), float(res), float(orth)


def t_svd(n):
    m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    t = bse.svd(m)
    _, s, _ = oracle.svd(m)
    rec = np.linalg.norm(m - (t.u * t.s[None, :]) @ t.v.conj().T) / np.linalg.norm(m)
    ou = np.linalg.norm(t.u.conj().T @ t.u - np.eye(n))
    ov = np.linalg.norm(t.v.conj().T @ t.v - np.eye(n))
    return float(np.max(np.abs(t.s - s)) / s[0]), float(rec), float(ou), float(ov)


def t_solve(method, a, b):
    h = bse.from_blocks(a, b)
    t0 = time.time()
    r = bse.solve(method, h)
    dt = time.time() - t0
    lo, vo, nso = oracle.solve(int(method), a, b)
    n = a.shape[0]
    top, bot = r.v[:n], r.v[n:]
    hv_top = h.a @ top + h.b @ bot
    hv_bot = -(h.b @ top) - h.a @ bot
    nh = np.sqrt(2 * np.linalg.norm(h.a) ** 2 + 2 * np.linalg.norm(h.b) ** 2)
    res = np.sqrt(np.linalg.norm(hv_top - top * r.lambda_[None, :], axis=0) ** 2 +
                  np.linalg.norm(hv_bot - bot * r.lambda_[None, :], axis=0) ** 2)
    res /= nh * np.linalg.norm(r.v, axis=0)
    sig = r.v.conj().T @ np.vstack([top, -bot])
    sdev = np.linalg.norm(sig - np.eye(n))
    lrel = np.max(np.abs(r.lambda_ - lo) / np.abs(lo))
    return dict(lam_rel=float(lrel), res=float(res.max()), sigma=float(sdev), t=round(dt, 3),
                flags=(r.near_singular, nso), phases={k: round(v, 2) for k, v in (r.phase_ms or {}).items()})


if __name__ == "__main__":
    sizes = [int(x) for x in (sys.argv[1:] or ["1", "2", "7", "64", "100", "257"])]
    step("1x1 chol", lambda: t_solve(bse.Method.Chol, np.array([[2.0]]), np.array([[1.0]])))
    for n in sizes:
        step(f"gemm NN n={n}", lambda: t_gemm(n, 0, 0))
        step(f"gemm CN n={n}", lambda: t_gemm(n, 1, 0))
        step(f"gemm NC n={n}", lambda: t_gemm(n, 0, 1))
        step(f"gemm CC n={n}", lambda: t_gemm(n, 1, 1))
        step(f"trmm n={n}", lambda: t_trmm(n))
        step(f"potrf n={n}", lambda: t_potrf(n))
        step(f"trsm n={n}", lambda: t_trsm(n))
        step(f"heev n={n}", lambda: t_heev(n))
        step(f"svd n={n}", lambda: t_svd(n))
        a, b = configs.generate_random_definite(n, 21)
        step(f"solve chol n={n}", lambda: t_solve(bse.Method.Chol, a, b))
        step(f"solve chol-svd n={n}", lambda: t_solve(bse.Method.CholSvd, a, b))
