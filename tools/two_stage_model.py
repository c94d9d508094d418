"""Numpy model of the two-stage Hermitian tridiagonalisation used by hetrd2.cu.

Validates the index bookkeeping of the GPU kernels on small sizes (CPU only):
  stage 1  he2hb : dense lower Hermitian -> lower band of width b (panel QR + her2k)
  stage 2  hb2st : band -> real symmetric tridiagonal by bulge chasing, task (s, j) =
                   {right-apply G(s,j-1) to Bk_j, reflector from Bk_j's first column,
                    left-apply to the rest of Bk_j, two-sided on the diagonal block D_j}
                   with the schedule rule "(s, j) after (s-1, j+1)" (random valid order)
  back-transform : Z <- Q1 Q2 Z, Q2 applied in groups (S desc, j asc, s desc in group).
Run: python tools/two_stage_model.py
"""
import numpy as np


def larfg(alpha, x):
    """LAPACK zlarfg: H^H [alpha; x] = [beta; 0], H = I - tau v v^H, v[0] = 1, beta real."""
    xn2 = float(np.vdot(x, x).real)
    if xn2 == 0.0 and alpha.imag == 0.0:
        return alpha.real, 0.0 + 0.0j, np.zeros_like(x)
    nrm = np.sqrt(abs(alpha) ** 2 + xn2)
    beta = -nrm if alpha.real >= 0 else nrm
    tau = complex((beta - alpha.real) / beta, -alpha.imag / beta)
    return beta, tau, x / (alpha - beta)


def he2hb(A, b):
    n = A.shape[0]
    A = np.tril(A).astype(complex)
    A = A + np.tril(A, -1).conj().T  # full Hermitian working copy (model only)
    refl = []  # (c0, r0, V (m x k), T (k x k))
    for c0 in range(0, n - b - 1, b):
        r0 = c0 + b
        m = n - r0
        P = A[r0:, c0:c0 + b].copy()
        k = min(m, b)
        V = np.zeros((m, k), complex)
        taus = np.zeros(k, complex)
        for j in range(k):
            beta, tau, v = larfg(P[j, j], P[j + 1:, j])
            vv = np.zeros(m, complex)
            vv[j] = 1.0
            vv[j + 1:] = v
            V[:, j] = vv
            taus[j] = tau
            # H^H applied to the rest of the panel
            w = vv.conj() @ P[:, j + 1:]
            P[:, j + 1:] -= np.conj(tau) * np.outer(vv, w)
            P[j, j] = beta
            P[j + 1:, j] = 0
        # T (zlarft forward columnwise)
        T = np.zeros((k, k), complex)
        for j in range(k):
            T[j, j] = taus[j]
            if j:
                g = V[:, :j].conj().T @ V[:, j]
                T[:j, j] = -taus[j] * (T[:j, :j] @ g)
        Q = np.eye(m) - V @ T @ V.conj().T
        assert np.allclose(Q.conj().T @ A[r0:, c0:c0 + b], P, atol=1e-10)
        A[r0:, c0:c0 + b] = P
        A[c0:c0 + b, r0:] = P.conj().T
        A22 = A[r0:, r0:]
        X = A22 @ (V @ T)
        M = T.conj().T @ (V.conj().T @ X)
        Wm = X - 0.5 * V @ M
        A[r0:, r0:] = A22 - V @ Wm.conj().T - Wm @ V.conj().T
        refl.append((c0, r0, V, T))
    return A, refl


def chase(Afull, b, rng=None):
    """Bulge chasing on the full Hermitian band matrix; returns d, e, reflectors[(s, j)]."""
    A = Afull.copy()
    n = A.shape[0]
    nt = [-(-(n - 1 - s) // b) for s in range(n - 1)]  # tasks of sweep s
    done = [0] * (n - 1)
    prev = {}
    refl = {}

    def rng_of(s, j):
        lo = s + 1 + j * b
        return lo, min(s + (j + 1) * b, n - 1)

    def task(s, j):
        lo, hi = rng_of(s, j)
        I = np.arange(lo, hi + 1)
        if j == 0:
            col = s
        else:
            plo, phi = rng_of(s, j - 1)
            P = np.arange(plo, phi + 1)
            v, tau = prev[s]
            # right-apply the previous reflector to Bk_j = A[I, P] (and, Hermitian, A[P, I])
            Bk = A[np.ix_(I, P)]
            Bk = Bk - tau * np.outer(Bk @ v, v.conj())
            A[np.ix_(I, P)] = Bk
            A[np.ix_(P, I)] = Bk.conj().T
            col = plo
        x = A[I, col]
        beta, tau, vt = larfg(x[0], x[1:])
        v = np.concatenate([[1.0], vt]).astype(complex)
        # left-apply H^H to rows I over the columns < lo (Bk_j; for j == 0 column s only)
        cols = np.arange(col, lo)
        blk = A[np.ix_(I, cols)]
        blk = blk - np.conj(tau) * np.outer(v, v.conj() @ blk)
        A[np.ix_(I, cols)] = blk
        A[np.ix_(cols, I)] = blk.conj().T
        # two-sided on D_j
        D = A[np.ix_(I, I)]
        x2 = tau * (D @ v)
        alpha = -0.5 * tau * np.vdot(x2, v)
        w = x2 + alpha * v
        D = D - np.outer(v, w.conj()) - np.outer(w, v.conj())
        A[np.ix_(I, I)] = D
        prev[s] = (v, tau)
        refl[(s, j)] = (lo, v, tau)

    # random valid schedule: (s, j) runnable when done[s] == j and sweep s-1 has finished
    # task j+1 (or all of its tasks)
    rng = rng or np.random.default_rng(0)
    total = sum(nt)
    while total:
        ready = [s for s in range(n - 1) if done[s] < nt[s] and
                 (s == 0 or done[s - 1] >= min(done[s] + 2, nt[s - 1]))]
        s = ready[rng.integers(len(ready))]
        task(s, done[s])
        done[s] += 1
        total -= 1
    d = np.real(np.diag(A)).copy()
    e = np.real(np.diag(A, -1)).copy()
    off = A - np.diag(np.diag(A)) - np.diag(np.diag(A, -1), -1) - np.diag(np.diag(A, 1), 1)
    assert np.abs(off).max() < 1e-10 * np.abs(Afull).max(), np.abs(off).max()
    assert np.abs(np.imag(np.diag(A, -1))).max() < 1e-12 * np.abs(Afull).max()
    return d, e, refl


def apply_q2(Z, refl, n, b, nb):
    """Z <- Q2 Z, groups (S desc, j asc), s desc inside a group."""
    Z = Z.astype(complex).copy()
    nS = -(-(n - 1) // nb)
    for S in range(nS - 1, -1, -1):
        s0 = S * nb
        jmax = max(j for (s, j) in refl if s0 <= s < s0 + nb)
        for j in range(jmax + 1):
            for s in range(min(s0 + nb, n - 1) - 1, s0 - 1, -1):
                if (s, j) not in refl:
                    continue
                lo, v, tau = refl[(s, j)]
                rows = slice(lo, lo + len(v))
                Z[rows] -= tau * np.outer(v, v.conj() @ Z[rows])
    return Z


def apply_q2_seq(Z, refl):
    Z = Z.astype(complex).copy()
    for (s, j) in sorted(refl, reverse=True):  # last (s, j) first
        lo, v, tau = refl[(s, j)]
        rows = slice(lo, lo + len(v))
        Z[rows] -= tau * np.outer(v, v.conj() @ Z[rows])
    return Z


def main():
    rng = np.random.default_rng(1)
    for n, b, nb in ((40, 4, 4), (53, 5, 5), (70, 8, 8), (37, 8, 8), (9, 4, 4)):
        X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        H = X + X.conj().T
        Ab, refl1 = he2hb(H, b)
        # band structure
        mask = np.abs(np.subtract.outer(np.arange(n), np.arange(n))) > b
        assert np.abs(Ab[mask]).max(initial=0) < 1e-10
        assert np.allclose(np.linalg.eigvalsh(Ab), np.linalg.eigvalsh(H))
        d, e, refl2 = chase(Ab, b, rng)
        T = np.diag(d) + np.diag(e, -1) + np.diag(e, 1)
        w, Zt = np.linalg.eigh(T)
        assert np.allclose(w, np.linalg.eigvalsh(H))
        Z = apply_q2(Zt, refl2, n, b, nb)
        assert np.allclose(Z, apply_q2_seq(Zt, refl2))
        for (c0, r0, V, Tm) in reversed(refl1):
            Z[r0:] -= V @ (Tm @ (V.conj().T @ Z[r0:]))
        res = np.abs(H @ Z - Z * w).max()
        assert res < 1e-10 * np.abs(H).max(), res
        print(f"n={n} b={b}: eigenvalues ok, residual {res:.2e}")


if __name__ == "__main__":
    main()
