"""Does the speed of a pass depend on WHERE its arrays land in device memory?
C5 solves with X MB of dummy device memory allocated before the matrix is
created (X shifts every later cudaMalloc); prints the live A v / A^T v times.

    python tools/placement_probe.py 0 2 6 14 30 62 126
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

w = W.make("c5")
bn = float(np.linalg.norm(w.b))
keep = []
for x in [int(a) for a in sys.argv[1:]] or [0, 2, 6, 14, 30, 62, 126]:
    if x:
        keep.append(torch.empty(x << 20, dtype=torch.uint8, device="cuda"))
    import os
    os.environ["TS_MATRIX_POOL"] = "0"
    dm = ts.DeviceMatrix(w.a)
    km = np.zeros(4)
    kc = np.zeros(4)
    for _ in range(50):
        r = ts.nonnegative_feasibility(dm, w.b, eps=1e-6 * bn)
        km += np.array(r.kernel_ms)
        kc += np.array(r.kernel_count)
    print(f"dummy +{x:4d} MB: A v {1e3 * km[0] / kc[0]:6.2f} us  A^T v {1e3 * km[1] / kc[1]:6.2f} us", flush=True)
    del dm
    torch.cuda.synchronize()
