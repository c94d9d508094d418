"""Full-size golden fixtures for BASELINE.json configs 2 and 3, from the CPU oracle (oracle/,
the LAPACK restatement of proj/src/{backend,core,solvers}.cpp; zgesvd('A','A') makes the
CHOL+SVD oracle take ~40 min at n = 4096 on 8 cores, which is why these are precomputed).
Only the inputs' generator arguments, the eigenvalues and three eigenvector columns (smallest,
median, largest eigenvalue) are stored; the GPU tests regenerate the inputs from the seeds.

    python tests/golden/make_big_golden.py [config3|config2svd|all|config4]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "full")


def big_case(name, gen, seed, n, methods, note):
    a, b = getattr(configs, gen)(seed, n=n)
    out = {"gen": gen, "seed": seed, "n": n, "note": note}
    for m in methods:
        t0 = time.time()
        lam, v, ns = oracle.solve(m, a, b)
        cols = np.array([0, n // 2, n - 1])
        key = m.replace("-", "_")
        out[f"lam_{key}"] = lam
        out[f"vcols_{key}"] = v[:, cols]
        out[f"cols_{key}"] = cols
        out[f"near_singular_{key}"] = np.asarray(ns, dtype=np.int64)
        out[f"seconds_{key}"] = time.time() - t0
        print(name, m, n, f"{time.time() - t0:.1f} s", lam[:2], lam[-1], flush=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)


if __name__ == "__main__":
    oracle.set_threads(os.cpu_count() or 1)
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("config2svd", "all"):
        big_case("config2_n2048_full", "config2", 2, 2048, ("chol-svd",),
                 "BASELINE config 2 at full size, CHOL+SVD")
    if which == "config4":  # separate target: ~1 h and ~40 GB of host memory
        big_case("config4_n16384_full", "config4", 0, 16384, ("chol",),
                 "BASELINE config 4 at full size, CHOL")
    if which in ("config3", "all"):
        big_case("config3_n4096_full", "config3", 0, 4096, ("chol", "chol-svd"),
                 "BASELINE config 3 at full size (ill-conditioned, lambda_min ~ 1e-3)")
