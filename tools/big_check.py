"""Full-size check (BASELINE config 4, n=16384, or any n): solve on the GPU through
bse_solve_device, then verify residual / Sigma-orthogonality with torch on the GPU (checker
only). Usage: python tools/big_check.py [n] [chol|chol-svd|both]"""
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
A = da.T  # logical n x n (column-major storage)
B = db.T
normh = torch.sqrt(2 * torch.linalg.norm(A) ** 2 + 2 * torch.linalg.norm(B) ** 2).item()
ctx = bse.Context(0)
ctx.set_kernel_timing(True)
eps = np.finfo(float).eps
for name, m in (("chol", bse.Method.Chol), ("chol-svd", bse.Method.CholSvd)):
    if which not in ("both", name):
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
    V = v.T  # 2n x n
    top, bot = V[:n], V[n:]
    res = 0.0
    sdev = 0.0
    for j0 in range(0, n, 2048):
        sl = slice(j0, min(n, j0 + 2048))
        ht = A @ top[:, sl] + B @ bot[:, sl]
        hb = -(B @ top[:, sl]) - A @ bot[:, sl]
        r = torch.sqrt(torch.linalg.norm(ht - top[:, sl] * lam[sl], dim=0) ** 2 +
                       torch.linalg.norm(hb - bot[:, sl] * lam[sl], dim=0) ** 2)
        r = r / (normh * torch.linalg.norm(V[:, sl], dim=0))
        res = max(res, r.max().item())
        g = V.conj().T[sl] @ torch.cat([top, -bot])  # rows sl of V^H Sigma V
        g[:, sl] -= torch.eye(sl.stop - sl.start, dtype=g.dtype, device=dev)
        sdev += (torch.linalg.norm(g) ** 2).item()
    lc = lam.cpu().numpy()
    ok = bool(np.all(np.diff(lc) >= 0) and lc[0] > 0 and res <= 100 * n * eps)
    print(f"{name}: n={n} wall {dt:.2f}s solve {ph['total']:.0f} ms phases "
          f"{ {k: round(v, 1) for k, v in ph.items() if k in ('product_pair', 'triple', 'reduce', 'tridiag', 'backtransform', 'recover')} } "
          f"lambda [{lc[0]:.6g}, {lc[-1]:.6g}] residual {res:.2e} (bound {100 * n * eps:.2e}) "
          f"sigma_dev {np.sqrt(sdev):.2e} flags {len(flags)} {'OK' if ok else 'FAIL'}", flush=True)
    del v, V, top, bot
    torch.cuda.empty_cache()
