"""Maintenance-step probe (not the bench contract): a C3 CTA solve of 1200
iterations (4 residual rechecks) and a C1 TA solve of 1500 iterations (2
revalidations).  With TS_DEBUG_MAINT=1 the library prints every HOST-driven
maintenance step: none in graph mode, all of them with TS_NO_GRAPH=1; the
printed results must be identical."""
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W
w = W.make("c3")
dm = ts.DeviceMatrix(w.a)
r = ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-8, max_iters=1200))
print("c3 cta", r.status, r.iterations, r.residual_norm)
w = W.make("c1")
dm = ts.DeviceMatrix(w.a)
bn = float(np.linalg.norm(w.b))
r = ts.solve_adaptive(dm, w.b, eps=1e-8 * bn, max_iters=1500)
print("c1 ta", r.status, r.iterations, r.residual_norm)
