"""Quick device timing probe (not the bench contract): solve-level times."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

def t_solve(fn, reps=3):
    best = None
    for _ in range(reps):
        r = fn()
        best = r if best is None or r.device_ms < best.device_ms else best
    return best

which = sys.argv[1:] or ["c2", "c5", "c4", "c1", "c3"]
for name in which:
    t0 = time.time()
    w = W.make(name)
    print(f"[{name}] generated in {time.time()-t0:.1f}s", flush=True)
    t0 = time.time(); dm = ts.DeviceMatrix(w.a); up = time.time() - t0
    bn = float(np.linalg.norm(w.b))
    if name in ("c1", "c2", "c3", "c4"):
        cap = {"c1": 2000, "c2": 100000, "c3": 2000, "c4": 200}[name]
        r = t_solve(lambda: ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-8, max_iters=cap)))
        print(f"  CTA {r.status} it={r.iterations} dev_ms={r.device_ms:.2f} it/s={r.iterations/r.device_ms*1e3:.1f} "
              f"kernels={r.kernel_launches} relres={r.residual_norm/bn:.3e} upload={up:.2f}s", flush=True)
        rb = t_solve(lambda: ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-300, max_iters=64)))
        print(f"  CTA bench64 it={rb.iterations} dev_ms={rb.device_ms:.2f} ms/it={rb.device_ms/rb.iterations:.3f}", flush=True)
    if name in ("c1", "c5"):
        r = t_solve(lambda: ts.solve_adaptive(dm, w.b, eps=0.0, max_iters=200))
        print(f"  TA200 {r.status} it={r.iterations} dev_ms={r.device_ms:.2f} ms/it={r.device_ms/r.iterations:.4f}", flush=True)
    if name == "c5":
        r = t_solve(lambda: ts.nonnegative_feasibility(dm, w.b, eps=1e-6 * bn))
        print(f"  LP {r.status} it={r.iterations} dev_ms={r.device_ms:.2f}", flush=True)
