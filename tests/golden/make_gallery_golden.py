"""Record the REAL reference's gallery matrices (small members of every
family) as tests/golden/gallery.npz.

    PYTHONPATH=/root/repo python tests/golden/make_gallery_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy.sparse as sparse

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from trisolve import gallery  # noqa: E402  (the reference)

CASES = [("diag-pd", 9, [], 3), ("diag-psd", 9, [], 4), ("diag-indef", 9, [], 5), ("gram-psd", 6, [], 2),
         ("clement", 7, [], 0), ("clement", 8, [], 0), ("dorr", 9, [], 0), ("dorr", 10, [0.05], 0),
         ("lotkin", 6, [], 0), ("poisson-d", 5, [], 0), ("poisson-n", 5, [], 0),
         ("convdiff", 5, [], 0), ("convdiff", 6, [2.0, 0.5, 3.0], 0), ("ode", 7, [], 0),
         ("ode", 6, [0.3, 0.1], 0)]


def main():
    out = {}
    for i, (fam, n, params, seed) in enumerate(CASES):
        a = gallery.make(fam, n, params, seed)
        out[f"c{i}_spec"] = np.array([fam, str(n), ",".join(map(str, params)), str(seed)])
        if sparse.issparse(a):
            a = sparse.csr_array(a)
            out[f"c{i}_indptr"] = a.indptr
            out[f"c{i}_indices"] = a.indices
            out[f"c{i}_data"] = a.data
            out[f"c{i}_shape"] = np.array(a.shape)
        else:
            out[f"c{i}_dense"] = np.asarray(a)
        out[f"c{i}_rowsum"] = gallery.row_sum_rhs(a)
    out["count"] = np.array(len(CASES))
    np.savez_compressed(os.path.join(HERE, "gallery.npz"), **out)
    print("recorded", len(CASES), "gallery members")


if __name__ == "__main__":
    main()
