"""Backend components at size n against numpy reconstructions (dev tool).
Usage: python tools/component_check.py [n]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
a, b = configs.config2(0, n=n)
m1, m2 = a + b, a - b


def rel(x, y):
    return np.linalg.norm(x - y) / np.linalg.norm(y)


for name, m in (("M1", m1), ("M2", m2)):
    t = time.time()
    lo = bse.cholesky_lower(m).l
    print(f"cholesky {name}: |LL^H - M|/|M| = {rel(lo @ lo.conj().T, m):.2e} "
          f"upper zero {np.abs(np.triu(lo, 1)).max():.1e} ({time.time() - t:.1f}s)", flush=True)
l1 = bse.cholesky_lower(m1).l
l2 = bse.cholesky_lower(m2).l
c = l1.conj().T @ l2
t = time.time()
s = bse.svd(c)
print(f"svd: |U S V^H - C|/|C| = {rel((s.u * s.s) @ s.v.conj().T, c):.2e} "
      f"|U^H U - I| = {np.linalg.norm(s.u.conj().T @ s.u - np.eye(n)):.2e} "
      f"|V^H V - I| = {np.linalg.norm(s.v.conj().T @ s.v - np.eye(n)):.2e} "
      f"sv err {np.max(np.abs(np.sort(s.s) - np.sort(np.linalg.svd(c, compute_uv=False)))) / s.s.max():.2e}"
      f" ({time.time() - t:.1f}s)", flush=True)
h = c + c.conj().T
e = bse.hermitian_eig(h)
print(f"heevd: |Q L Q^H - H|/|H| = {rel((e.vectors * e.values) @ e.vectors.conj().T, h):.2e}",
      flush=True)
pp = bse.matmul(l1, l2, op_a=bse.Op.Adjoint)
print(f"matmul L1^H L2: {rel(pp, c):.2e}", flush=True)
