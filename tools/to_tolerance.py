"""Full solves to the reference's stopping rule on C3 and C4 (not the bench
contract; their bench lines use fixed iteration budgets).  Prints status,
iterations, device time and final residuals as JSON lines."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

for name, cap in [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]:
    w = W.make(name)
    dm = ts.DeviceMatrix(w.a)
    bn = float(np.linalg.norm(w.b))
    t0 = time.perf_counter()
    r = ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-8, max_iters=cap))
    wall = time.perf_counter() - t0
    atb = float(np.linalg.norm(ts.matvec_transpose(dm, w.b)))
    print(json.dumps({"config": name, "status": r.status, "detail": r.detail, "iterations": r.iterations,
                      "device_s": r.device_ms / 1e3, "wall_s": wall,
                      "us_per_iteration": r.device_ms * 1e3 / max(r.iterations, 1),
                      "rel_residual": r.residual_norm / bn,
                      "normal_residual_over_eps_b": r.normal_residual_norm / (1e-8 * bn),
                      "normal_residual_rel_to_Atb": r.normal_residual_norm / atb}), flush=True)
