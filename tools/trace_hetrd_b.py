"""Phase-B sub-steps of the hetrd panel (dev tool): stamps 3 (B start), 6 (loads done), 7
(scalars done), 4 (B end) of the slab owner, from BSE_HETRD_TRACE."""
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
bse.hermitian_eig(np.asfortranarray(x + x.conj().T))
t = np.loadtxt(path, delimiter=",")
t = t[(t[:, 1] == 1) & (t[:, 2 + 6] > 0)]
s3, s6, s7, s4 = t[:, 2 + 3], t[:, 2 + 6], t[:, 2 + 7], t[:, 2 + 4]
for lo, hi in ((0, n // 4), (n // 4, n // 2), (n // 2, 3 * n // 4), (3 * n // 4, n)):
    sel = (t[:, 0] >= lo) & (t[:, 0] < hi)
    print(f"cols {lo:5d}-{hi:5d}: loads={np.mean(s6[sel]-s3[sel])/1e3:6.2f}us "
          f"scalars={np.mean(s7[sel]-s6[sel])/1e3:6.2f}us rest={np.mean(s4[sel]-s7[sel])/1e3:6.2f}us")
