"""Runs a fixed set of small device solves and prints digests of the results
(one JSON line): the body of tests/test_gpu_variants.py, which starts it once
per kernel-structure switch (the switches are read once per process)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W


def digest(r):
    x = np.ascontiguousarray(r.x, dtype=np.float64)
    rows = np.ascontiguousarray(np.array([[float(v) for v in row[:4]] for row in r.trace.rows], dtype=np.float64))
    return {"status": r.status, "iterations": int(r.iterations),
            "x_sha": hashlib.sha256(x.tobytes()).hexdigest(),
            "trace_sha": hashlib.sha256(rows.tobytes()).hexdigest(),
            "x_head": [float(v) for v in x[:64]]}


out = {}
# square banded, L2-resident: band-pair kernel, period graph, mid-period rechecks
w = W.clement_variant(n=4001, seed=3)
dm = ts.DeviceMatrix(w.a)
out["clement_cta"] = digest(ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-10, max_iters=140)))
out["clement_cta_recheck3"] = digest(ts.centering_solve(
    dm, w.b, ts.CenteringOptions(epsilon=1e-10, max_iters=61, recheck_every=3, t_max=4)))
out["clement_cta_t1"] = digest(ts.centering_solve(
    dm, w.b, ts.CenteringOptions(epsilon=1e-10, max_iters=30, recheck_every=7, t_max=1)))
bn = float(np.linalg.norm(w.b))
out["clement_ta_reval"] = digest(ts.solve_adaptive(dm, w.b, eps=1e-9 * bn, max_iters=1100))
# 5-point stencil (wider band)
w = W.convdiff_upwind(grid=40, seed=1)
dm = ts.DeviceMatrix(w.a)
out["convdiff_cta"] = digest(ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-10, max_iters=90)))
# small dense: warp-per-row kernel both ways
w = W.dense_gaussian(300, 200, seed=5)
dm = ts.DeviceMatrix(w.a)
out["dense_cta"] = digest(ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-10, max_iters=40, recheck_every=5)))
bn = float(np.linalg.norm(w.b))
out["dense_ta"] = digest(ts.solve_adaptive(dm, w.b, eps=1e-8 * bn, max_iters=60))
print(json.dumps(out))
