"""Run one backend op at size n (for ncu captures). Usage: python tools/run_once.py svd|eig|chol|chol-svd n"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

what = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
rng = np.random.default_rng(0)
if what in ("svd", "eig"):
    m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    if what == "eig":
        m = m + m.conj().T
    m = np.asfortranarray(m)
    (bse.svd if what == "svd" else bse.hermitian_eig)(m)
else:
    a, b = configs.config2(0, n=n)
    bse.solve(bse.Method.Chol if what == "chol" else bse.Method.CholSvd, bse.from_blocks(a, b))
print("done")
