"""Dump the C5 CSR as raw arrays (/tmp/c5.indptr|indices|data) for the
standalone microbenchmarks (tools/microbench/spmv_long.cu)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2304_12168_b200 import workloads as W
a = W.make("c5").a
a.indptr.astype(np.int32).tofile("/tmp/c5.indptr")
a.indices.astype(np.int32).tofile("/tmp/c5.indices")
a.data.astype(np.float64).tofile("/tmp/c5.data")
print(a.shape, a.nnz)
