"""k = 128 complex GEMM (the back-transform update shape) through bse_matmul, for ncu (dev tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402

m, k, n = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 128, 4096
rng = np.random.default_rng(0)
a = np.asfortranarray(rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)))
b = np.asfortranarray(rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)))
ctx = bse.default_context()
ctx.set_kernel_timing(True)
for _ in range(3):
    bse.matmul(a, b)
pt = ctx.phase_times()
print(f"k={k}: gemm {pt['gemm_ms']:.3f} ms {pt['gemm_flops'] / pt['gemm_ms'] / 1e9:.2f} TFLOP/s (complex-equivalent)")
