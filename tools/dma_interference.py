"""Does concurrent PCIe traffic slow the 4-lane device batch? (dev tool; e2e gap study)
Times bse_solve_batched_device over 16 config-5 items alone and with a background stream
copying pinned host buffers H2D and D2H at the rate of the e2e path's copies."""
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

n, items = 4096, 16
dev = torch.device("cuda", 0)
ctx = bse.Context(0)
mats = []
for s in range(4):
    a, b = configs.config2(s, n=n)
    mats.append((torch.from_numpy(a).to(dev).t().contiguous().t(), torch.from_numpy(b).to(dev).t().contiguous().t()))
lams = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(items)]
vs = [torch.empty((n, 2 * n), dtype=torch.complex128, device=dev) for _ in range(4)]


def run():
    bse.solve_batched_device(bse.Method.Chol, n, [mats[i % 4][0].data_ptr() for i in range(items)],
                             [mats[i % 4][1].data_ptr() for i in range(items)],
                             [lams[i].data_ptr() for i in range(items)],
                             [vs[i % 4].data_ptr() for i in range(items)], ctx=ctx)
    torch.cuda.synchronize()


run()
stop = threading.Event()
moved = [0]


def pump(rate_gbs, h2d=True, d2h=True, mb=512):
    hs = torch.empty(mb * 2**20, dtype=torch.uint8).pin_memory()
    hd = torch.empty(mb * 2**20, dtype=torch.uint8).pin_memory()
    ds = torch.empty(mb * 2**20, dtype=torch.uint8, device=dev)
    dd = torch.empty(mb * 2**20, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t0 = time.perf_counter()
    while not stop.is_set():
        if h2d:
            with torch.cuda.stream(s1):
                ds.copy_(hs, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                hd.copy_(dd, non_blocking=True)
        s1.synchronize()
        s2.synchronize()
        moved[0] += (int(h2d) + int(d2h)) * mb * 2**20
        # throttle to the target average rate
        while moved[0] / 1e9 / max(time.perf_counter() - t0, 1e-9) > rate_gbs and not stop.is_set():
            time.sleep(0.002)


for label, rate, hh, dh, mb in (("alone", 0, 1, 1, 512), ("d2h 11.5 512MB", 11.5, 0, 1, 512),
                               ("d2h 11.5 16MB", 11.5, 0, 1, 16), ("d2h full 16MB", 1e9, 0, 1, 16),
                               ("d2h full 512MB", 1e9, 0, 1, 512), ("alone", 0, 1, 1, 512)):
    th = None
    moved[0] = 0
    if rate:
        stop.clear()
        th = threading.Thread(target=pump, args=(rate, bool(hh), bool(dh), mb), daemon=True)
        th.start()
        time.sleep(0.5)
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    if th:
        stop.set()
        th.join()
    print(f"{label:16s} {dt * 1e3 / items:7.2f} ms per matrix, copied {moved[0] / 1e9 / dt:5.1f} GB/s", flush=True)
