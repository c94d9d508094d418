"""Batch of 4 host-pointer CHOL solves (n = 4096, 2 lanes) into page-locked V outputs: the
first item of each lane downloads through the L2-streaming copy kernel (dev tool, for ncu)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 4
ctx = bse.Context(0)
ctx.set_batch_lanes(2)
hs = [bse.from_blocks(*configs.config2(s, n=n)) for s in range(k)]
ha = [torch.from_numpy(h.a.T.copy()).pin_memory() for h in hs]
hb = [torch.from_numpy(h.b.T.copy()).pin_memory() for h in hs]
hv = [torch.empty((n, 2 * n), dtype=torch.complex128).pin_memory() for _ in range(k)]
hl = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(k)]
arr = lambda ts: (ctypes.c_void_p * k)(*[t.data_ptr() for t in ts])  # noqa: E731
failed = ctypes.c_int64(-1)
st = bse.Status()
t0 = time.time()
rc = bse._lib.lib().bse_solve_batched(ctx.handle, int(bse.Method.Chol), n, k, arr(ha), n, arr(hb), n,
                                      arr(hl), arr(hv), 2 * n, None, None, ctypes.byref(failed),
                                      ctypes.byref(st))
print("rc", rc, "wall", round(time.time() - t0, 3), "s")
