"""Fixed per-solve cost (not the bench contract): device_ms of C2 CTA solves
capped at 1, 2, 5 and 23 iterations; the intercept of the line is the
per-solve overhead (init, graph launch, final honest-residual passes, copies)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = W.make(name)
dm = ts.DeviceMatrix(w.a)
b = torch.from_numpy(w.b).cuda()
for cap in (1, 2, 5, 23, 1, 23):
    ds, ws = [], []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ts.centering_solve(dm, b, ts.CenteringOptions(epsilon=1e-8, max_iters=cap))
        ws.append((time.perf_counter() - t0) * 1e3)
        ds.append(r.device_ms)
    print(f"cap {cap:3d}: it {r.iterations:3d} device {np.median(ds):8.3f} ms  wall {np.median(ws):8.3f} ms  "
          f"kernels {r.kernel_launches}", flush=True)
