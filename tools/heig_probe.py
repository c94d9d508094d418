"""One Hermitian eigen-decomposition (hetrd + D&C + back-transform) at size n (dev tool, for
ncu captures of the panel kernels): python tools/heig_probe.py [n] [reps]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(0)
x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
m = np.asfortranarray(x + x.conj().T)
for _ in range(reps):
    t0 = time.perf_counter()
    bse.hermitian_eig(m)
    print(f"heig n={n} {1e3 * (time.perf_counter() - t0):.1f} ms (incl. copies)", flush=True)
