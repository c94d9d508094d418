"""Two independent solves at once (two contexts, two host threads) vs one after the other
(throughput experiment, dev tool). Usage: python tools/concurrency2.py [n] [method] [pairs]"""
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
meth = bse.method_from_name(sys.argv[2] if len(sys.argv) > 2 else "chol")
pairs = int(sys.argv[3]) if len(sys.argv) > 3 else 3
K = int(sys.argv[4]) if len(sys.argv) > 4 else 2  # solves in flight
dev = torch.device("cuda", 0)
mats = []
for s in range(K):
    a, b = configs.config2(s, n=n)
    mats.append((torch.from_numpy(a.T.copy()).to(dev), torch.from_numpy(b.T.copy()).to(dev)))
outs = [(torch.empty(n, dtype=torch.float64, device=dev),
         torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)) for _ in range(K)]
ctxs = [bse.Context(0) for _ in range(K)]


def work(k, reps):
    da, db = mats[k]
    lam, v = outs[k]
    for _ in range(reps):
        bse.solve_device(meth, n, da.data_ptr(), db.data_ptr(), lam.data_ptr(), v.data_ptr(),
                         ctx=ctxs[k])


for k in range(K):
    work(k, 1)  # warm-up every context
torch.cuda.synchronize()
t0 = time.time()
for k in range(K):
    work(k, pairs)
torch.cuda.synchronize()
seq = (time.time() - t0) / (K * pairs)
t0 = time.time()
th = [threading.Thread(target=work, args=(k, pairs)) for k in range(K)]
for t in th:
    t.start()
for t in th:
    t.join()
torch.cuda.synchronize()
con = (time.time() - t0) / (K * pairs)
print(f"n={n} {sys.argv[2] if len(sys.argv) > 2 else 'chol'}: sequential {seq * 1e3:.1f} ms/solve, "
      f"{K} at once {con * 1e3:.1f} ms/solve ({seq / con:.2f}x)", flush=True)
