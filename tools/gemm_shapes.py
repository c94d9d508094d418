"""Throughput of the DMMA zgemm for the skinny shapes used by the solver (dev tool)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402

rng = np.random.default_rng(0)
ctx = bse.default_context()
ctx.set_kernel_timing(True)
for m, n, k, opa, opb in [(4096, 4096, 4096, 0, 0), (4096, 4096, 64, 0, 1), (4096, 4096, 128, 0, 1),
                          (4096, 4096, 256, 0, 1), (128, 4096, 4096, 1, 0), (4096, 4096, 128, 0, 0),
                          (2048, 2048, 64, 0, 1), (16384, 64, 64, 0, 1)]:
    a = rng.standard_normal((k, m) if opa else (m, k)) + 0j
    b = rng.standard_normal((n, k) if opb else (k, n)) + 0j
    best = 0
    for _ in range(3):
        bse.matmul(a, b, op_a=bse.Op(opa), op_b=bse.Op(opb))
        pt = ctx.phase_times()
        best = max(best, pt['gemm_flops'] / pt['gemm_ms'] / 1e9)
    print(f"m={m:6d} n={n:6d} k={k:6d} op=({opa},{opb}): {best:6.2f} TFLOP/s", flush=True)
