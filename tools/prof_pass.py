"""Time (or, under ncu, profile) single matvec passes of a BASELINE config
through ts_time_pass: back-to-back launches of one pass kernel on
device-resident vectors (every launch active, unlike TS_NO_GRAPH solves).

    python tools/prof_pass.py c4 [reps]      # prints avg us per pass, GB/s
"""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import _native as N
from paper_2304_12168_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
w = W.make(name)
dm = ts.DeviceMatrix(w.a)
m, n = w.a.shape
out = {}
for trans in (0, 1):
    avg = C.c_double()
    N.check(N.lib().ts_time_pass(dm.handle, trans, reps, C.byref(avg), None))
    if dm.kind == "csr":
        nnz = dm.nnz
        byt = 12 * nnz + 4 * ((n if trans else m) + 1) + 8 * (m + n)
    else:
        byt = 8 * m * n + 8 * (m + n)
    us = avg.value * 1e3
    out["A^T v" if trans else "A v"] = {"us": round(us, 2), "GB/s": round(byt / (us * 1e-6) / 1e9, 1)}
print(name, json.dumps(out), flush=True)
