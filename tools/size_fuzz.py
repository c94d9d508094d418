"""Size fuzz of hermitian_eig / svd / both BSE methods against numpy (dev tool): random n in
[1, 2100], seeded; prints the worst errors."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
sizes = sorted(set([1, 2, 3, 63, 64, 65, 127, 128, 129, 191, 192, 193] +
                   list(rng.integers(1, 2100, 24))))
eps = np.finfo(float).eps
worst = {}
for n in sizes:
    n = int(n)
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = np.asfortranarray(x + x.conj().T)
    he = bse.hermitian_eig(h.copy())
    ref = np.linalg.eigvalsh(h)
    e1 = np.max(np.abs(np.sort(he.values) - ref)) / max(np.max(np.abs(ref)), 1e-300)
    r1 = np.linalg.norm(h - (he.vectors * he.values) @ he.vectors.conj().T) / np.linalg.norm(h) / (n * eps)
    sv = bse.svd(np.asfortranarray(x))
    refs = np.linalg.svd(x, compute_uv=False)
    e2 = np.max(np.abs(np.sort(sv.s)[::-1] - refs)) / refs[0]
    r2 = np.linalg.norm(x - (sv.u * sv.s) @ sv.v.conj().T) / np.linalg.norm(x) / (n * eps)
    o2 = max(np.linalg.norm(sv.u.conj().T @ sv.u - np.eye(n)), np.linalg.norm(sv.v.conj().T @ sv.v - np.eye(n))) / (n * eps)
    a, b = configs.config2(int(n) % 97, n=n)
    res = []
    for m in (bse.Method.Chol, bse.Method.CholSvd):
        r = bse.solve(m, bse.from_blocks(a, b))
        top, bot = r.v[:n], r.v[n:]
        nh = np.sqrt(2 * np.linalg.norm(a) ** 2 + 2 * np.linalg.norm(b) ** 2)
        rr = np.sqrt(np.linalg.norm(a @ top + b @ bot - top * r.lambda_, axis=0) ** 2 +
                     np.linalg.norm(-(b @ top) - a @ bot - bot * r.lambda_, axis=0) ** 2)
        res.append(float((rr / (nh * np.linalg.norm(r.v, axis=0))).max() / (n * eps)))
    row = dict(eig_err=e1, eig_rec=r1, svd_err=e2, svd_rec=r2, svd_orth=o2, chol_res=res[0], svd_res=res[1])
    for k, v in row.items():
        if v > worst.get(k, (0, 0))[0]:
            worst[k] = (v, n)
    print(n, " ".join(f"{k}={v:.1e}" for k, v in row.items()), flush=True)
print("worst:", {k: f"{v:.2e} @ n={m}" for k, (v, m) in worst.items()})
