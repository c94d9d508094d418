"""Generates the committed golden fixtures from the CPU oracle (oracle/, LAPACK
restatement of proj/src/{backend,core,solvers}.cpp). Inputs follow the reference's own test
families (proj/tests/test_solvers.cpp) and BASELINE.json's configs at reduced size.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def case(name, a, b, method, note):
    lam, v, ns = oracle.solve(method, a, b)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), a=np.asarray(a, complex),
                        b=np.asarray(b, complex), method=method, lam=lam, v=v,
                        near_singular=np.asarray(ns, dtype=np.int64), note=note)
    print(name, method, a.shape[0], lam[:3])


if __name__ == "__main__":
    one = (np.array([[2.0 + 0j]]), np.array([[1.0 + 0j]]))
    for m in ("chol", "chol-svd"):
        case(f"canonical_1x1_{m}", *one, m, "test_solvers.cpp:33-42")
    case("decoupled_chol", np.diag([3.0, 1.0, 2.0]).astype(complex), np.zeros((3, 3), complex),
         "chol", "test_solvers.cpp:24-31")
    for s in (21, 22, 23):
        a, b = configs.generate_random_definite(16, s)
        for m in ("chol", "chol-svd"):
            case(f"random_definite16_s{s}_{m}", a, b, m, "test_solvers.cpp:90-105")
    a, b = configs.generate_conditioned(50, 10.0, 3)
    for m in ("chol", "chol-svd"):
        case(f"conditioned50_k10_s3_{m}", a, b, m, "test_solvers.cpp:81-88")
    a, b = configs.generate_conditioned(40, 1000.0, 13)
    case("conditioned40_k1e3_s13_chol-svd", a, b, "chol-svd", "test_solvers.cpp:160-166")
    a = np.diag([1e-40, 1.0]).astype(complex)
    for m in ("chol", "chol-svd"):
        case(f"clamp_flag_{m}", a, np.zeros((2, 2), complex), m, "test_solvers.cpp:168-186")
    a, b = configs.config1(0, n=48)
    case("config1_n48_chol", a, b, "chol", "BASELINE config 1 generator at n=48 (real)")
    a, b = configs.config2(0, n=40)
    case("config2_n40_chol", a, b, "chol", "BASELINE config 2 generator at n=40")
    a, b = configs.config3(0, n=32)
    case("config3_n32_chol-svd", a, b, "chol-svd", "BASELINE config 3 generator at n=32")
