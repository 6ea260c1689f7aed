"""Per-class live kernel time of one solve (graph mode), per iteration."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

for name, iters in [(n, int(i)) for n, i in (a.split(":") for a in sys.argv[1:])]:
    w = W.make(name)
    dm = ts.DeviceMatrix(w.a)
    for _ in range(2):
        r = ts.centering_solve(dm, w.b, ts.CenteringOptions(epsilon=1e-300, max_iters=iters))
    it = r.iterations
    names = ["A v", "A^T v", "vector", "hankel"]
    print(f"{name}: {it} it, device {r.device_ms:.2f} ms = {r.device_ms/it*1e3:.1f} us/it, "
          f"kernels {r.kernel_launches} ({r.kernel_launches/it:.1f}/it)")
    tot = 0.0
    for k in range(4):
        if r.kernel_count[k]:
            tot += r.kernel_ms[k]
            print(f"   {names[k]:7s} n={r.kernel_count[k]:6d} avg={r.kernel_ms[k]/r.kernel_count[k]*1e3:7.2f} us "
                  f"per-it={r.kernel_ms[k]/it*1e3:7.2f} us")
    print(f"   kernels sum per-it {tot/it*1e3:.1f} us; gaps/launch per-it {(r.device_ms-tot)/it*1e3:.1f} us")
