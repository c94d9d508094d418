"""Phase breakdown of the hetrd panel kernel from BSE_HETRD_TRACE timestamps (dev tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
path = "/tmp/hetrd_trace.csv"
os.environ["BSE_HETRD_TRACE"] = path
rng = np.random.default_rng(0)
x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
m = np.asfortranarray(x + x.conj().T)
bse.hermitian_eig(m)
t = np.loadtxt(path, delimiter=",")
t = t[t[:, 2] > 0]
names = ["A:reflector", "A:tiles", "gridsync1", "B:update", "gridsync2"]
for who in (0, 1):
    cols = t[t[:, 1] == who]
    d = np.diff(cols[:, 2:8], axis=1) / 1e3  # us: A-pre, tiles, syncA, phaseB, syncB
    print("CTA 0" if who == 0 else "owner of the last slab")
    for lo, hi in ((0, n // 4), (n // 4, n // 2), (n // 2, 3 * n // 4), (3 * n // 4, n)):
        sel = (cols[:, 0] >= lo) & (cols[:, 0] < hi)
        mean = d[sel].mean(axis=0)
        print(f"  cols {lo:5d}-{hi:5d}: " + "  ".join(f"{k}={v:6.2f}us" for k, v in zip(names, mean)),
              f" total={mean.sum():6.2f}us")
