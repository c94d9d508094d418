"""Stage-by-stage CHOL pipeline through the building-block API vs the oracle (dev tool)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


for n in [int(x) for x in sys.argv[1:]]:
    a, b = configs.generate_random_definite(n, 21)
    h = bse.from_blocks(a, b)
    m1, m2 = h.a + h.b, h.a - h.b
    L = bse.cholesky_lower(m2).l
    M = bse.matmul(bse.matmul(L, m1, op_a=bse.Op.Adjoint, shape_a=bse.Shape.Lower), L,
                   shape_b=bse.Shape.Lower)
    e = bse.hermitian_eig(M)
    res = np.linalg.norm(M @ e.vectors - e.vectors * e.values[None, :]) / np.linalg.norm(M)
    orth = np.linalg.norm(e.vectors.conj().T @ e.vectors - np.eye(n))
    v1 = bse.tri_solve(bse.CholeskyLower(L), e.vectors, bse.Side.Left, bse.Op.Adjoint)
    v2 = bse.matmul(L, e.vectors, shape_a=bse.Shape.Lower)
    lam = np.sqrt(e.values)
    V = bse.assemble_eigenvectors(bse.HalfSpectralFactors(v1, v2, lam * lam, np.ones(n)))
    top, bot = V[:n], V[n:]
    r = np.linalg.norm(h.a @ top + h.b @ bot - top * lam[None, :])
    r2 = bse.solve_chol(h)
    top2, bot2 = r2.v[:n], r2.v[n:]
    rr = np.linalg.norm(h.a @ top2 + h.b @ bot2 - top2 * r2.lambda_[None, :])
    print(n, "heev res", res, "orth", orth, "blocks res", r, "solve res", rr,
          "V diff", rel(np.abs(r2.v), np.abs(V)), flush=True)
    # direct heev on the same M, twice (determinism)
    e2 = bse.hermitian_eig(M)
    print("   heev repeat diff", rel(e2.vectors, e.vectors), flush=True)
