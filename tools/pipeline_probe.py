"""Per-phase timing of the double-buffered e2e loop (probe, not the contract)."""
import sys, time
sys.path.insert(0, ".")
from concurrent.futures import ThreadPoolExecutor
import numpy as np, torch
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

w = W.make("c2")
t = torch.empty(w.a.shape, dtype=torch.float64, pin_memory=True)
a_host = t.numpy(); a_host[...] = w.a
tb = torch.empty(w.b.shape, dtype=torch.float64, pin_memory=True)
b_host = tb.numpy(); b_host[...] = w.b
s = torch.cuda.Stream()
opts = ts.CenteringOptions(epsilon=1e-8)
up = lambda: ts.DeviceMatrix(a_host, stream=s)
with ThreadPoolExecutor(max_workers=1) as pool:
    nxt = pool.submit(up)
    for k in range(8):
        t0 = time.perf_counter()
        dm = nxt.result(); t1 = time.perf_counter()
        nxt = pool.submit(up); t2 = time.perf_counter()
        r = ts.centering_solve(dm, b_host, opts); t3 = time.perf_counter()
        del dm; t4 = time.perf_counter()
        print(f"wait {1e3*(t1-t0):6.2f}  submit {1e3*(t2-t1):5.2f}  solve {1e3*(t3-t2):6.2f} (device {r.device_ms:6.2f})  release {1e3*(t4-t3):5.2f}", flush=True)
