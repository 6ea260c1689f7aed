"""Fixed per-solve cost on C5 (not the bench contract): device_ms and wall time
of TA-LP solves capped at 1, 2, 5 and 11 iterations; the intercept of the line
is the per-solve overhead (input staging, init, graph launch, final
honest-residual passes, x read-back, host glue)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

w = W.make("c5")
dm = ts.DeviceMatrix(w.a)
bn = float(np.linalg.norm(w.b))
for cap in (1, 2, 5, 11, 1, 11):
    ds, ws = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        r = ts.nonnegative_feasibility(dm, w.b, eps=1e-6 * bn, max_iters=cap)
        ws.append((time.perf_counter() - t0) * 1e3)
        ds.append(r.device_ms)
    print(f"cap {cap:3d}: it {r.iterations:3d} {r.status:14s} device {np.median(ds):7.3f} ms  wall {np.median(ws):7.3f} ms  "
          f"kernels {r.kernel_launches}", flush=True)
