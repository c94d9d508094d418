"""GPU check of the two-stage tridiagonal reduction (hetrd2.cu) against numpy / the oracle.

BSE_TWO_STAGE=1 python tools/two_stage_check.py [n ...]
For each n: bse.hermitian_eig on a random Hermitian matrix (eigenvalues vs numpy, residual,
orthogonality), then one CHOL solve of the config-2 generator vs the oracle. Also times the
reduction against the one-stage path when BSE_TWO_STAGE is unset in a second process.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [128, 130, 200, 257, 300, 513, 1000]
    rng = np.random.default_rng(7)
    eps = np.finfo(float).eps
    for n in sizes:
        x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        m = (x + x.conj().T) / 2
        t0 = time.time()
        e = bse.hermitian_eig(m)
        t1 = time.time()
        w = np.linalg.eigvalsh(m)
        nm = np.linalg.norm(m, 2)
        lam_err = np.abs(e.values - w).max() / nm
        res = np.linalg.norm(m @ e.vectors - e.vectors * e.values) / (nm * np.sqrt(n))
        orth = np.abs(e.vectors.conj().T @ e.vectors - np.eye(n)).max()
        ok = lam_err < 50 * n * eps and res < 50 * n * eps and orth < 50 * n * eps
        print(f"heevd n={n}: lam_err={lam_err:.2e} res={res:.2e} orth={orth:.2e} "
              f"{'OK' if ok else 'FAIL'} ({(t1 - t0) * 1e3:.1f} ms)", flush=True)
    for n in [s for s in sizes if s >= 256][:3]:
        import oracle
        a, b = configs.config2(3, n=n)
        h = bse.from_blocks(a, b)
        r = bse.solve_chol(h)
        lo, _, _ = oracle.solve("chol", h.a, h.b)
        err = float(np.max(np.abs(r.lambda_ - lo) / lo))
        print(f"chol n={n}: lambda_rel_err={err:.2e} {'OK' if err < 1e-10 else 'FAIL'}",
              flush=True)


if __name__ == "__main__":
    main()
