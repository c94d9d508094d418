"""Large complex GEMM through bse_matmul for ncu / timing (dev tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(0)
a = np.asfortranarray(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
b = np.asfortranarray(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
ctx = bse.default_context()
ctx.set_kernel_timing(True)
for opa, opb in ((0, 0), (1, 0), (0, 1)):
    bse.matmul(a, b, op_a=bse.Op(opa), op_b=bse.Op(opb))
    t0 = time.time()
    c = bse.matmul(a, b, op_a=bse.Op(opa), op_b=bse.Op(opb))
    pt = ctx.phase_times()
    print(f"op=({opa},{opb}) wall {time.time() - t0:.3f}s gemm {pt['gemm_ms']:.3f} ms "
          f"{pt['gemm_flops'] / pt['gemm_ms'] / 1e9:.2f} TFLOP/s", flush=True)
