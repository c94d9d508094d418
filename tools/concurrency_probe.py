"""Throughput of 1 vs 2 vs 3 concurrent solves (separate contexts / host threads) on one GPU."""
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
method = bse.Method.Chol if (len(sys.argv) < 3 or sys.argv[2] == "chol") else bse.Method.CholSvd
dev = torch.device("cuda", 0)
mats = []
for sd in range(6):
    a, b = configs.config5(sd, n=n)
    mats.append((torch.from_numpy(a.T).to(dev), torch.from_numpy(b.T).to(dev)))
ctxs = [bse.Context(0) for _ in range(3)]
outs = [(torch.empty(n, dtype=torch.float64, device=dev),
         torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)) for _ in range(3)]


def work(k, idx):
    for i in idx:
        a, b = mats[i]
        bse.solve_device(method, n, a.data_ptr(), b.data_ptr(), outs[k][0].data_ptr(),
                         outs[k][1].data_ptr(), ctx=ctxs[k])


for nt in (1, 2, 3):
    # warm up every context once
    for k in range(nt):
        work(k, [k])
    torch.cuda.synchronize()
    per = 6 // nt
    t0 = time.time()
    th = [threading.Thread(target=work, args=(k, list(range(k * per, (k + 1) * per))))
          for k in range(nt)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    dt = time.time() - t0
    print(f"{nt} concurrent solve(s): {6 / dt:.2f} solves/s ({1000 * dt / 6:.1f} ms per solve)",
          flush=True)
