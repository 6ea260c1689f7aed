"""Events-timed matvec passes per BASELINE config (ts_time_pass): avg us, GB/s."""
import ctypes as C, json, os, sys
sys.path.insert(0, ".")
import numpy as np
import scipy.sparse as sp
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import _native as N, workloads as W

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
for name in names:
    w = W.make(name)
    dm = ts.DeviceMatrix(w.a)
    m, n = w.a.shape
    for trans in (0, 1):
        if sp.issparse(w.a):
            nnz = w.a.nnz
            byt = 12 * nnz + 4 * ((n if trans else m) + 1) + 8 * (m + n)
        else:
            byt = 8 * m * n + 8 * (m + n)
        out = C.c_double()
        N.check(N.lib().ts_time_pass(dm.handle, trans, 20, C.byref(out), None))
        us = out.value * 1e3
        gbs = byt / (us * 1e-6) / 1e9
        print(f"{name} {'A^T v' if trans else 'A v  '} {us:9.2f} us  {gbs:8.1f} GB/s  frac={gbs/peak:.3f}  "
              f"bpsm={os.environ.get('TS_BLOCKS_PER_SM','4')}", flush=True)
