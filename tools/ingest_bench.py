"""Ingest timing (not the bench contract): a C4-sized Matrix Market file
(5-point operator, n = 1e6, 4,996,000 entries) read (a) straight to a device
matrix (native parser + device CSR assembly), (b) to a host CSR (same parser +
scipy conversion) and then uploaded as a DeviceMatrix.  Prints one JSON line."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
import numpy as np

from paper_2304_12168_b200 import mmio
from paper_2304_12168_b200 import workloads as W

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
a = W.convdiff_upwind(grid).a
path = os.path.join(tempfile.mkdtemp(), "c4.mtx")
t0 = time.perf_counter()
mmio.write_matrix_market(a, path)
t_write = time.perf_counter() - t0
size = os.path.getsize(path)
res = {"file_mb": size / 1e6, "nnz": int(a.nnz), "write_s": t_write}
import paper_2304_12168_b200 as ts
for rep in range(2):
    t0 = time.perf_counter()
    dm, info = mmio.read_matrix_market_device(path)
    res["file_to_device_matrix_s"] = time.perf_counter() - t0
    del dm
    t0 = time.perf_counter()
    host = mmio.read_matrix_market(path)
    res["file_to_host_csr_s"] = time.perf_counter() - t0
    dm2 = ts.DeviceMatrix(host)
    res["file_to_host_csr_to_device_matrix_s"] = time.perf_counter() - t0
    del dm2
v = np.random.default_rng(0).standard_normal(a.shape[1])
dm, info = mmio.read_matrix_market_device(path)
res["same_operator"] = bool(np.array_equal(dm.matvec(v), a @ v))
res["cores"] = os.cpu_count()
print(json.dumps(res))
