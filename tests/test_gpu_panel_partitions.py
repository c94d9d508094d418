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
