"""Phase breakdown of the gebrd panel kernel from BSE_GEBRD_TRACE timestamps (dev tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
path = "/tmp/gebrd_trace.csv"
os.environ["BSE_GEBRD_TRACE"] = path
rng = np.random.default_rng(0)
m = np.asfortranarray(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
bse.svd(m)
t = np.loadtxt(path, delimiter=",")
t = t[t[:, 2] > 0]
names = ["P1 rows", "sync1", "P2 colrefl+tiles", "sync2", "P3 cols", "sync3", "P4 rowrefl+tiles"]
for who in (0, 1):
    cols = t[t[:, 1] == who]
    d = np.diff(cols[:, 2:10], axis=1) / 1e3
    print("CTA 0" if who == 0 else "owner of the last slab")
    for lo, hi in ((0, n // 4), (n // 4, n // 2), (n // 2, 3 * n // 4), (3 * n // 4, n)):
        sel = (cols[:, 0] >= lo) & (cols[:, 0] < hi)
        mean = d[sel].mean(axis=0)
        print(f"  cols {lo:5d}-{hi:5d}: " + " ".join(f"{k}={v:5.1f}" for k, v in zip(names, mean)),
              f" sum={mean.sum():6.1f}us")
