"""Does a DeviceMatrix upload on a non-blocking stream overlap a solve? (probe)"""
import sys, time, threading
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W

w = W.make("c2")
from paper_2304_12168_b200 import _native as N
mode = sys.argv[1] if len(sys.argv) > 1 else "torch"
if mode == "lib":  # pinned through the library's own runtime (ts_host_alloc)
    a_host = N.pinned_empty(w.a.size).reshape(w.a.shape); a_host[...] = w.a
else:
    t = torch.empty(w.a.shape, dtype=torch.float64, pin_memory=True)
    a_host = t.numpy(); a_host[...] = w.a
print("mode", mode, flush=True)
b = w.b
import ctypes, glob, os
rt = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))[0])
ts_ = torch.cuda.Stream()
fl = ctypes.c_uint()
rt.cudaStreamGetFlags(ctypes.c_void_p(ts_.cuda_stream), ctypes.byref(fl))
print("torch stream flags:", fl.value, flush=True)
h = ctypes.c_void_p()
print("create rc", rt.cudaStreamCreateWithFlags(ctypes.byref(h), 1), flush=True)
s = h.value
dm0 = ts.DeviceMatrix(a_host, stream=s)
dm1 = ts.DeviceMatrix(a_host, stream=s)
del dm1
opts = ts.CenteringOptions(epsilon=1e-8)
for rep in range(3):
    t0 = time.perf_counter(); d = ts.DeviceMatrix(a_host, stream=s); tu = time.perf_counter() - t0; del d
    t0 = time.perf_counter(); ts.centering_solve(dm0, b, opts); tsol = time.perf_counter() - t0
    res = {}
    def up():
        t1 = time.perf_counter(); res["d"] = ts.DeviceMatrix(a_host, stream=s); res["t"] = time.perf_counter() - t1
    th = threading.Thread(target=up)
    t0 = time.perf_counter(); th.start(); ts.centering_solve(dm0, b, opts); th.join(); tb = time.perf_counter() - t0
    del res["d"]
    print(f"upload {tu*1e3:.1f} ms  solve {tsol*1e3:.1f} ms  both {tb*1e3:.1f} ms (upload in thread {res['t']*1e3:.1f})", flush=True)
# torch's own async H2D on a side stream vs our solve
dst = torch.empty(w.a.shape, dtype=torch.float64, device="cuda")
src = torch.from_numpy(a_host)
ts_side = torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(ts_side):
        dst.copy_(src, non_blocking=True)
    t_enq = time.perf_counter() - t0
    ts.centering_solve(dm0, b, opts)
    t_sol = time.perf_counter() - t0
    ts_side.synchronize()
    t_all = time.perf_counter() - t0
    print(f"torch copy enqueue {t_enq*1e3:.2f} ms, solve done at {t_sol*1e3:.1f} ms, all {t_all*1e3:.1f} ms", flush=True)
