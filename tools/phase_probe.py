"""Phase times of single solves (CUDA events inside the library). Usage:
python tools/phase_probe.py [chol|chol-svd] [n] [reps]"""
import sys

sys.path.insert(0, ".")
import paper_2008_08825_b200 as bse  # noqa: E402
from paper_2008_08825_b200 import configs  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "chol"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a, b = configs.config2(0, n=n)
h = bse.from_blocks(a, b)
ctx = bse.Context(0)
m = bse.Method.Chol if what == "chol" else bse.Method.CholSvd
for i in range(reps):
    bse.solve(m, h, ctx=ctx)
    ph = ctx.phase_times()
    print(what, n, {k: round(v, 2) for k, v in ph.items() if isinstance(v, float)}, flush=True)
