"""Full-size check (BASELINE config 4, n=16384, or any n): solve on the GPU through
bse_solve_device, then verify with the library's own device diagnostics:
per-column residual ||H v - lambda v|| / ||H||_F and ||V^H Sigma V - I||_F.
Usage: python tools/big_check.py [n] [chol|chol-svd|sqrt|reference|all]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
which = sys.argv[2] if len(sys.argv) > 2 else "both"
dev = torch.device("cuda", 0)
t0 = time.time()
a, b = configs.config4(0, n=n) if n == 16384 else configs.config2(0, n=n)
print(f"generated n={n} in {time.time() - t0:.1f}s", flush=True)
da = torch.from_numpy(a.T).to(dev)  # column-major bytes
db = torch.from_numpy(b.T).to(dev)
del a, b
ctx = bse.Context(0)
ctx.set_kernel_timing(True)
eps = np.finfo(float).eps
methods = {"chol": bse.Method.Chol, "chol-svd": bse.Method.CholSvd, "sqrt": bse.Method.Sqrt,
           "reference": bse.Method.Reference}
for name, m in methods.items():
    if which not in ("all", name) and not (which == "both" and name in ("chol", "chol-svd")):
        continue
    lam = torch.empty(n, dtype=torch.float64, device=dev)
    v = torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)
    torch.cuda.synchronize()
    t0 = time.time()
    flags = bse.solve_device(m, n, da.data_ptr(), db.data_ptr(), lam.data_ptr(), v.data_ptr(),
                             ctx=ctx)
    torch.cuda.synchronize()
    dt = time.time() - t0
    ph = ctx.phase_times()
    res = torch.empty(n, dtype=torch.float64, device=dev)
    t1 = time.time()
    bse.residual_device(n, da.data_ptr(), db.data_ptr(), n, lam.data_ptr(), v.data_ptr(),
                        res.data_ptr(), ctx=ctx)
    sdev = bse.sigma_orthogonality_error_device(2 * n, n, v.data_ptr(), ctx=ctx)
    tv = time.time() - t1
    keep = torch.ones(n, dtype=torch.bool, device=dev)
    if flags:
        keep[torch.tensor(flags, device=dev)] = False
    rmax = res[keep].max().item()
    lc = lam.cpu().numpy()
    ok = bool(np.all(np.diff(lc) >= 0) and lc[0] > 0 and rmax <= 100 * n * eps)
    print(f"{name}: n={n} wall {dt:.2f}s solve {ph['total']:.0f} ms phases "
          f"{ {k: round(x, 1) for k, x in ph.items() if k in ('product_pair', 'triple', 'reduce', 'tridiag', 'backtransform', 'recover')} } "
          f"lambda [{lc[0]:.6g}, {lc[-1]:.6g}] residual {rmax:.2e} (bound {100 * n * eps:.2e}) "
          f"sigma_dev {sdev:.2e} flags {len(flags)} verify {tv:.2f}s {'OK' if ok else 'FAIL'}",
          flush=True)
    del v
    torch.cuda.empty_cache()
