"""GPU parity of the cooperative panel kernels under other CTA counts (SURVEY §8a rows a8.1,
a9.1: zhetrd / zgebrd inside zheevd / zgesvd, backend.cpp:34, 74).

The hetrd and gebrd panels split the trailing tile triangle / square into one contiguous run
of tiles per CTA (hetrd: folded column order with column segments; gebrd: column order), so
the segment boundaries, the diagonal tiles and the runs shorter than the 3-slot TMA ring all
move with the CTA count. A batch lane runs its panels on 148/lanes CTAs and a single solve on
every SM; here each CTA count of interest (1 CTA: every tile on one run; small odd counts:
runs shorter than the ring and runs that end inside a tile column) runs in its own process
through the developer switch BSE_SOLO_PANEL_CTAS (read once per process), and the spectra and
reconstructions are checked against numpy on the same matrix.

Tolerances: eigenvalues / singular values 1e-11 relative to the largest; reconstruction
||A - Q diag Q^H|| (resp. ||A - U S V^H||) <= 100 n eps ||A||.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2008_08825_b200 as bse
n = {n}
rng = np.random.default_rng(n)
x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
h = np.asfortranarray(x + x.conj().T)
he = bse.hermitian_eig(h.copy())
w, q = he.values, he.vectors
eps = np.finfo(float).eps
ref = np.linalg.eigvalsh(h)
e1 = np.max(np.abs(np.sort(w) - ref)) / np.max(np.abs(ref))
r1 = np.linalg.norm(h - (q * w) @ q.conj().T) / np.linalg.norm(h)
g = np.asfortranarray(x)
sv = bse.svd(g.copy())
u, s, vh = sv.u, sv.s, sv.v.conj().T
refs = np.linalg.svd(g, compute_uv=False)
e2 = np.max(np.abs(np.sort(s)[::-1] - refs)) / refs[0]
r2 = np.linalg.norm(g - (u * s) @ vh) / np.linalg.norm(g)
print(e1, r1, e2, r2, 100 * n * eps)
"""


@pytest.mark.parametrize("ctas", [1, 3, 7, 37, 61])
@pytest.mark.parametrize("n", [250, 700])
def test_panels_under_cta_counts(ctas, n):
    env = dict(os.environ, BSE_SOLO_PANEL_CTAS=str(ctas))
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, n=n)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    e1, r1, e2, r2, tol = map(float, out.stdout.split()[-5:])
    assert e1 <= 1e-11, e1
    assert e2 <= 1e-11, e2
    assert r1 <= tol, r1
    assert r2 <= tol, r2


SPECIAL = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2008_08825_b200 as bse
n, kind = {n}, {kind!r}
rng = np.random.default_rng(7)
q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
if kind == "repeated":      # three eigenvalues with multiplicities n/2, n/4, n/4
    lam = np.repeat([1.0, -2.0, 5.0], [n // 2, n // 4, n - n // 2 - n // 4])
    h = (q * lam) @ q.conj().T
elif kind == "diagonal":    # every reflector is the identity (tau = 0)
    h = np.diag(rng.standard_normal(n)).astype(complex)
elif kind == "tridiagonal":  # already reduced: x = 0 below the subdiagonal in every column
    h = np.diag(rng.standard_normal(n)).astype(complex)
    off = rng.standard_normal(n - 1) + 1j * rng.standard_normal(n - 1)
    h += np.diag(off, -1) + np.diag(off.conj(), 1)
elif kind == "graded":      # entries from 1 down to 1e-12 across the matrix
    s = np.logspace(0, -6, n)
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (s[:, None] * (x + x.conj().T)) * s[None, :]
h = np.asfortranarray((h + h.conj().T) / 2)
he = bse.hermitian_eig(h.copy())
w, v = he.values, he.vectors
ref = np.linalg.eigvalsh(h)
e = np.max(np.abs(np.sort(w) - ref)) / np.max(np.abs(ref))
r = np.linalg.norm(h - (v * w) @ v.conj().T) / np.linalg.norm(h)
o = np.linalg.norm(v.conj().T @ v - np.eye(n))
print(e, r, o, 100 * n * np.finfo(float).eps)
"""


@pytest.mark.parametrize("kind", ["repeated", "diagonal", "tridiagonal", "graded"])
@pytest.mark.parametrize("ctas", [0, 37])
@pytest.mark.parametrize("n", [300, 1100])
def test_hermitian_eig_special_structure(kind, ctas, n):
    """Degenerate spectra (D&C deflation), reflectors with tau = 0 (diagonal input), input
    already tridiagonal, and graded entries, through the restructured hetrd sweep at every SM
    and at a lane's 37 CTAs, against numpy: eigenvalues 1e-12 of the largest, reconstruction
    and orthogonality <= 100 n eps."""
    env = dict(os.environ)
    if ctas:
        env["BSE_SOLO_PANEL_CTAS"] = str(ctas)
    out = subprocess.run([sys.executable, "-c", SPECIAL.format(root=ROOT, n=n, kind=kind)],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    e, r, o, tol = map(float, out.stdout.split()[-4:])
    assert e <= 1e-12, e
    assert r <= tol, r
    assert o <= tol, o


SPECIAL_SVD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2008_08825_b200 as bse
n, kind = {n}, {kind!r}
rng = np.random.default_rng(11)
x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
if kind == "diagonal":
    g = np.diag(rng.standard_normal(n) + 1j * rng.standard_normal(n))
elif kind == "bidiagonal":
    g = np.diag(rng.standard_normal(n)).astype(complex) + np.diag(rng.standard_normal(n - 1), 1)
elif kind == "rank_deficient":   # rank n/2: half of the singular values are zero
    g = x[:, : n // 2] @ (rng.standard_normal((n // 2, n)) + 0j)
elif kind == "graded":
    s = np.logspace(0, -6, n)
    g = s[:, None] * x
g = np.asfortranarray(g)
sv = bse.svd(g.copy())
u, s, vh = sv.u, sv.s, sv.v.conj().T
ref = np.linalg.svd(g, compute_uv=False)
e = np.max(np.abs(np.sort(s)[::-1] - ref)) / ref[0]
r = np.linalg.norm(g - (u * s) @ vh) / np.linalg.norm(g)
ou = np.linalg.norm(u.conj().T @ u - np.eye(n))
ov = np.linalg.norm(vh @ vh.conj().T - np.eye(n))
print(e, r, ou, ov, 100 * n * np.finfo(float).eps)
"""


@pytest.mark.parametrize("kind", ["diagonal", "bidiagonal", "rank_deficient", "graded"])
@pytest.mark.parametrize("ctas", [0, 37])
@pytest.mark.parametrize("n", [300, 1100])
def test_svd_special_structure(kind, ctas, n):
    """The restructured gebrd sweeps (column segments) on diagonal, already-bidiagonal,
    rank-deficient and graded inputs at every SM and at a lane's 37 CTAs, against numpy:
    singular values 1e-12 of the largest, reconstruction and orthogonality <= 100 n eps."""
    env = dict(os.environ)
    if ctas:
        env["BSE_SOLO_PANEL_CTAS"] = str(ctas)
    out = subprocess.run([sys.executable, "-c", SPECIAL_SVD.format(root=ROOT, n=n, kind=kind)],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    e, r, ou, ov, tol = map(float, out.stdout.split()[-5:])
    assert e <= 1e-12, e
    assert r <= tol, r
    assert ou <= tol and ov <= tol, (ou, ov)


@pytest.mark.parametrize("n", [1, 2, 3, 63, 64, 65, 127, 129, 193, 517, 1031])
def test_sizes_eig_svd_against_numpy(n):
    """Tile-edge and odd sizes through the restructured panels (in-process, every SM):
    eigenvalues / singular values 1e-12 of the largest, reconstructions and orthogonality
    within 10 n eps (tools/size_fuzz.py: worst 2.4 n eps over 36 sizes up to 2100)."""
    import paper_2008_08825_b200 as bse

    rng = np.random.default_rng(n)
    eps = np.finfo(float).eps
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = np.asfortranarray(x + x.conj().T)
    he = bse.hermitian_eig(h.copy())
    ref = np.linalg.eigvalsh(h)
    assert np.max(np.abs(np.sort(he.values) - ref)) <= 1e-12 * np.max(np.abs(ref))
    q = he.vectors
    assert np.linalg.norm(h - (q * he.values) @ q.conj().T) <= 10 * n * eps * np.linalg.norm(h)
    assert np.linalg.norm(q.conj().T @ q - np.eye(n)) <= 10 * n * eps
    sv = bse.svd(np.asfortranarray(x))
    refs = np.linalg.svd(x, compute_uv=False)
    assert np.max(np.abs(np.sort(sv.s)[::-1] - refs)) <= 1e-12 * refs[0]
    assert np.linalg.norm(x - (sv.u * sv.s) @ sv.v.conj().T) <= 10 * n * eps * np.linalg.norm(x)
    assert np.linalg.norm(sv.u.conj().T @ sv.u - np.eye(n)) <= 10 * n * eps
    assert np.linalg.norm(sv.v.conj().T @ sv.v - np.eye(n)) <= 10 * n * eps
