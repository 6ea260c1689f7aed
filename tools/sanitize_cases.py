"""Small device solves of every family and kernel plan, run under
compute-sanitizer (memcheck / racecheck / synccheck) by tools/sanitize.sh:
dense CTA / TA / min-norm, sparse CSR (thread-per-row and sliced-ELL plans),
TA-LP, the Gram pair, a column-sharded and a row-sharded emulated world of
2 ranks.  Prints one line per case; any sanitizer error fails the run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W
from paper_2304_12168_b200.shard import LocalWorld


def forced(a, plan):
    os.environ["TS_CSR_SHORT"] = plan
    try:
        return ts.DeviceMatrix(a)
    finally:
        del os.environ["TS_CSR_SHORT"]


w = W.dense_gaussian(300, 260, seed=1)
bn = float(np.linalg.norm(w.b))
dm = ts.DeviceMatrix(w.a)
print("dense cta", ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-8, max_iters=30)).iterations)
print("dense ta", ts.solve_adaptive(dm, w.b, eps=1e-8 * bn, max_iters=40).iterations)
print("dense ta gram", ts.solve_adaptive(ts.GramProduct(dm), dm.rmatvec(w.b), eps=1e-6 * bn, max_iters=20).iterations)
print("dense min-norm", ts.min_norm_solve(dm, w.b, eps=1e-4 * bn, x_eps=np.zeros(w.a.shape[1]), inner_cap=200, max_iters=2000).status)
c4 = W.convdiff_upwind(40, seed=2)
for plan in ("thread", "sell"):
    s = forced(c4.a, plan)
    print("csr cta", plan, ts.centering_solve(s, c4.b, ts.CenteringOptions(epsilon=1e-8, max_iters=30)).iterations)
lp = W.lp_columns(60, 3000, 10, seed=5)
lb = float(np.linalg.norm(lp.b))
for plan in ("thread", "sell"):
    s = forced(lp.a, plan)
    print("lp", plan, ts.nonnegative_feasibility(s, lp.b, eps=1e-6 * lb).status)
big = W.lp_columns(200, 20000, 10, seed=3)  # long rows: k_rows_wrow
print("lp long rows", ts.nonnegative_feasibility(big.a, big.b, eps=1e-6 * np.linalg.norm(big.b)).status)
lw = LocalWorld(2)
cols = lw.columns(lp.a)
print("world2 columns lp", [r.status for r in lw.run(ts.nonnegative_feasibility, cols, lp.b, eps=1e-6 * lb)])
rows = lw.rows(c4.a)
print("world2 rows cta", [r.iterations for r in lw.run(ts.centering_solve, rows, c4.b,
                                                        ts.CenteringOptions(epsilon=1e-8, max_iters=20))])
tall = lw.tall(w.a)
print("world2 tall cta", [r.iterations for r in lw.run(ts.centering_solve, tall, w.b,
                                                        ts.CenteringOptions(epsilon=1e-8, max_iters=20))])
del cols, rows, tall
lw.close()
print("sanitize cases done")
