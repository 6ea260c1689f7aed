import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from conftest import Golden, trace_rows_numeric, rel_l2
from test_gpu_parity import run_device, x_tolerance
for name in sys.argv[1:]:
    g = Golden(name); res = run_device(g)
    tr = trace_rows_numeric(res.trace.rows, res.trace.columns)
    colmax = np.abs(g.trace).max(axis=0)
    bound = x_tolerance(name) * np.maximum(np.abs(g.trace), colmax)
    viol = np.abs(tr - g.trace) / bound
    i, j = np.unravel_index(np.argmax(viol), viol.shape)
    print(name, g.trace_columns, "worst row", i, "col", j, "dev", tr[i], "ref", g.trace[i], "ratio", viol[i, j], "x", rel_l2(res.x, g.x))
