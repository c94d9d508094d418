"""Wall time of bse_solve (host pointers) with page-locked vs pageable buffers.
Usage: python tools/e2e_probe.py [n] [method...]"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
methods = sys.argv[2:] or ["chol", "chol-svd"]
a, b = configs.config2(0, n=n)
ctx = bse.default_context()
lib = bse._lib.lib()
for mname in methods:
    meth = bse.method_from_name(mname)
    for pinned in (True, False, True):
        ha = torch.from_numpy(np.asfortranarray(a).T.copy())
        hb = torch.from_numpy(np.asfortranarray(b).T.copy())
        hv = torch.empty((n, 2 * n), dtype=torch.complex128)
        hl = torch.empty(n, dtype=torch.float64)
        if pinned:
            ha, hb, hv, hl = ha.pin_memory(), hb.pin_memory(), hv.pin_memory(), hl.pin_memory()
        st = bse.Status()
        ns = np.zeros(n, dtype=np.int64)
        nn = ctypes.c_int64(0)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            rc = lib.bse_solve(ctx.handle, int(meth), n, ctypes.c_void_p(ha.data_ptr()), n,
                               ctypes.c_void_p(hb.data_ptr()), n, ctypes.c_void_p(hl.data_ptr()),
                               ctypes.c_void_p(hv.data_ptr()), 2 * n,
                               ns.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nn),
                               ctypes.byref(st))
            ts.append((time.perf_counter() - t0) * 1e3)
            assert rc == 0, st.message
        pt = bse.PhaseTimes()
        lib.bse_ctx_last_phase_times(ctx.handle, ctypes.byref(pt))
        print(f"{mname:9s} pinned={pinned!s:5s} wall ms {[round(t, 1) for t in ts]} "
              f"device total {pt.total:.1f} recover {pt.recover:.1f}", flush=True)
