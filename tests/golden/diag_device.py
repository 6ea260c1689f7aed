import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from conftest import Golden, rel_l2, trace_rows_numeric
from test_gpu_parity import run_device
for name in sys.argv[1:]:
    g = Golden(name); r = run_device(g)
    print(name, "status", r.status, g.status, "iters", r.iterations, g.iterations, "detail", repr(r.detail), repr(g.detail))
    print("  x rel", rel_l2(r.x, g.x), "res", r.residual_norm, g.residual_norm)
    tr = trace_rows_numeric(r.trace.rows, r.trace.columns)
    n = min(len(tr), len(g.trace))
    if n:
        d = np.abs(tr[:n]-g.trace[:n]) / np.maximum(np.abs(g.trace[:n]), 1e-300)
        print("  trace maxrel per col", d.max(axis=0))
        bad = np.nonzero(d.max(axis=1) > 1e-9)[0]
        print("  first bad row", bad[:5], tr[bad[:2]] if len(bad) else None, g.trace[bad[:2]] if len(bad) else None)
