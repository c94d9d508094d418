"""Config 5 end to end: the 64 seeds (n = 4096, config-2 generator) through the batch driver
(bse_solve_batched_device, default 4 lanes) on one GPU, every result checked by the device
diagnostics (residual / (||H||_F ||x||) <= 100 n eps, ||V^H Sigma V - I||_F, ascending
positive eigenvalues), and eight of them against a single-lane solve of the same matrix.
Usage: python tools/batch64_check.py [n] [method]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
meth = bse.Method.Chol if (sys.argv[2] if len(sys.argv) > 2 else "chol") == "chol" else bse.Method.CholSvd
dev = torch.device("cuda", 0)
eps = np.finfo(float).eps
ctx = bse.Context(0)
ctx.set_batch_lanes(4)
worst_res, worst_sig, worst_ref = 0.0, 0.0, 0.0
t_solve = 0.0
for chunk in range(8):  # 8 chunks of 8 matrices (8 x 512 MiB of inputs + 8 x 512 MiB of V)
    seeds = list(range(chunk * 8, chunk * 8 + 8))
    mats = [configs.config5(s, n=n) for s in seeds]
    da = [torch.from_numpy(a.T).to(dev) for a, _ in mats]
    db = [torch.from_numpy(b.T).to(dev) for _, b in mats]
    lam = [torch.empty(n, dtype=torch.float64, device=dev) for _ in seeds]
    v = [torch.empty((n, 2 * n), dtype=torch.complex128, device=dev) for _ in seeds]
    torch.cuda.synchronize()
    t0 = time.time()
    flags = bse.solve_batched_device(meth, n, [x.data_ptr() for x in da], [x.data_ptr() for x in db],
                                     [x.data_ptr() for x in lam], [x.data_ptr() for x in v], ctx=ctx)
    torch.cuda.synchronize()
    t_solve += time.time() - t0
    res = torch.empty(n, dtype=torch.float64, device=dev)
    for k, s in enumerate(seeds):
        bse.residual_device(n, da[k].data_ptr(), db[k].data_ptr(), n, lam[k].data_ptr(),
                            v[k].data_ptr(), res.data_ptr(), ctx=ctx)
        r = (res / torch.linalg.vector_norm(v[k], dim=1)).max().item()
        sg = bse.sigma_orthogonality_error_device(2 * n, n, v[k].data_ptr(), ctx=ctx)
        lc = lam[k].cpu().numpy()
        assert np.all(np.diff(lc) >= 0) and lc[0] > 0, s
        worst_res, worst_sig = max(worst_res, r), max(worst_sig, sg)
    # the first matrix of the chunk again as a single solve owning the GPU
    l1 = torch.empty(n, dtype=torch.float64, device=dev)
    v1 = torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)
    bse.solve_device(meth, n, da[0].data_ptr(), db[0].data_ptr(), l1.data_ptr(), v1.data_ptr(),
                     ctx=ctx)
    worst_ref = max(worst_ref, ((l1 - lam[0]).abs() / l1).max().item())
    print(f"chunk {chunk}: seeds {seeds[0]}..{seeds[-1]} ok (worst residual {worst_res:.2e}, "
          f"sigma dev {worst_sig:.2e}, batch vs single lambda {worst_ref:.2e})", flush=True)
    del da, db, lam, v, v1
    torch.cuda.empty_cache()
ok = worst_res <= 100 * n * eps and worst_sig <= 1e-8 and worst_ref <= 1e-12
print(f"config 5: 64 matrices n={n} {meth.name}: batch solve time {t_solve:.2f} s (8 calls of 8), "
      f"max residual {worst_res:.2e} (bound {100 * n * eps:.2e}), max sigma dev {worst_sig:.2e}, "
      f"max batch-vs-single eigenvalue deviation {worst_ref:.2e} -> {'OK' if ok else 'FAIL'}")
sys.exit(0 if ok else 1)
