"""Host-side phase timing of one end-to-end solve (not the bench contract):
matrix upload / handle creation, the solve call (split into device time and
host overhead), result read-back, handle destruction.

    python tools/e2e_phases.py c2 c5
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W


def pinned(arr):
    t = torch.empty(arr.shape, dtype=torch.float64 if arr.dtype == np.float64 else torch.int32,
                    pin_memory=True)
    out = t.numpy()
    out[...] = arr
    return out, t


def solve(name, dm, b, bn):
    if name in ("c1", "c2", "c3", "c4"):
        cap = {"c1": 2000, "c2": 100000, "c3": 2000, "c4": 200}[name]
        return ts.centering_solve(dm, b, ts.CenteringOptions(epsilon=1e-8, max_iters=cap))
    return ts.nonnegative_feasibility(dm, b, eps=1e-6 * bn)


for name in sys.argv[1:] or ["c2", "c5"]:
    w = W.make(name)
    bn = float(np.linalg.norm(w.b))
    keep = []
    import scipy.sparse as sp
    if sp.issparse(w.a):
        d, t1 = pinned(w.a.data)
        i, t2 = pinned(w.a.indices.astype(np.int32))
        p, t3 = pinned(w.a.indptr.astype(np.int32))
        keep += [t1, t2, t3]
        a_host = sp.csr_array((d, i, p), shape=w.a.shape)
        a_host.indices = i
        a_host.indptr = p
    else:
        a_host, t1 = pinned(w.a)
        keep.append(t1)
    b_host, t4 = pinned(w.b)
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dm = ts.DeviceMatrix(a_host)
        t1_ = time.perf_counter()
        r = solve(name, dm, b_host, bn)
        t2_ = time.perf_counter()
        r2 = solve(name, dm, b_host, bn)
        t3_ = time.perf_counter()
        del dm
        torch.cuda.synchronize()
        t4_ = time.perf_counter()
        print(f"[{name} rep{rep}] create {1e3*(t1_-t0):.2f} ms | first solve {1e3*(t2_-t1_):.2f} ms "
              f"(device {r.device_ms:.2f}) | cached solve {1e3*(t3_-t2_):.2f} ms (device {r2.device_ms:.2f}) "
              f"| destroy {1e3*(t4_-t3_):.2f} ms | it={r.iterations} kernels={r.kernel_ms}", flush=True)
