"""Short driver for ncu captures: build one BASELINE config, run a few solves.
Use with TS_NO_GRAPH=1 (ncu cannot profile kernel nodes of conditional graphs)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = W.make(name)
dm = ts.DeviceMatrix(w.a)
bn = float(np.linalg.norm(w.b))
for _ in range(reps):
    if name in ("c1", "c2", "c3", "c4"):
        r = ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-8, max_iters=40))
    else:
        r = ts.solve_adaptive(dm, w.b, eps=0.0, max_iters=40)
    print(name, r.status, r.iterations, f"{r.device_ms:.2f} ms", r.kernel_ms, r.kernel_count)
