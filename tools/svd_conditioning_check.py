"""SVD orthogonality on ill-conditioned and rank-deficient inputs (dev tool): the TGK route
with tgk_reorthogonalize checked with numpy: U^H U, V^H V and the reconstruction."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse
rng = np.random.default_rng(11)
def orth(q): return np.linalg.norm(q.conj().T @ q - np.eye(q.shape[1]))
n = 1100
bd = np.diag(rng.standard_normal(n)).astype(complex) + np.diag(rng.standard_normal(n - 1), 1)
H = np.zeros((2 * n, 2 * n), complex); H[:n, n:] = bd; H[n:, :n] = bd.conj().T
he = bse.hermitian_eig(np.asfortranarray(H))
print("eig of [[0,B],[B^H,0]] (random bidiagonal B): orth %.1e  recon %.1e" % (orth(he.vectors),
      np.linalg.norm(H - (he.vectors * he.values) @ he.vectors.conj().T) / np.linalg.norm(H)))
g = np.diag(rng.uniform(1, 2, n)).astype(complex) + np.diag(rng.uniform(1, 2, n - 1), 1)
sv = bse.svd(np.asfortranarray(g))
print("svd bidiagonal entries in [1,2]: orthU %.1e orthV %.1e" % (orth(sv.u), orth(sv.v)), "smin/smax %.1e" % (sv.s.min() / sv.s.max()))
x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
u0, s0, vh0 = np.linalg.svd(x); s0[-2:] = 0.0
g = np.asfortranarray((u0 * s0) @ vh0)
sv = bse.svd(g)
print("svd rank n-2: orthU %.1e orthV %.1e recon %.1e" % (orth(sv.u), orth(sv.v), np.linalg.norm(g - (sv.u * sv.s) @ sv.v.conj().T) / np.linalg.norm(g)))
s0 = np.logspace(0, -18, n)
g = np.asfortranarray((u0 * s0) @ vh0)
sv = bse.svd(g)
print("svd sigma 1..1e-18 log-spaced: orthU %.1e orthV %.1e recon %.1e" % (orth(sv.u), orth(sv.v), np.linalg.norm(g - (sv.u * sv.s) @ sv.v.conj().T) / np.linalg.norm(g)))
