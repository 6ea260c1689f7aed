"""ctypes binding of ``oracle/mirror.c`` — TEST INFRASTRUCTURE ONLY.

The C restatement of the device arithmetic of the dense TA path (see the
header of mirror.c).  Built by ``oracle/Makefile`` into
``oracle/_build/libmirror.so`` (``__graft_entry__.build()`` runs it).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libmirror.so")
_lib = None

TAG_PIVOT, TAG_EXPAND = 0, 1
STATUS = {0: "running", 1: "approx_solution", 2: "normal_eq_solution", 7: "iteration_cap",
          8: "numerical_failure"}


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", HERE], check=True, capture_output=True)
        lib = C.CDLL(LIB)
        lib.ts_mirror_ta_dense.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_double,
                                           C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_int64,
                                           C.c_void_p]
        lib.ts_mirror_ta_dense.restype = C.c_int64
        _lib = lib
    return _lib


def ta_dense(a, b, eps, max_iters, sms=148):
    """Run the mirrored device TA (solve_adaptive, x0 = None) on a dense
    matrix.  Returns dict(x, status, iterations, residual_norm,
    normal_residual_norm, rho, x_norm, trace) with trace rows
    (iter, tag, rho, gap_norm, c_norm).  Mirrors the tiled dense plans, which
    the library picks for n >= 128 and m n >= 2048 (smaller or narrower
    matrices run thread-per-row)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] < 128 or a.size < 2048:
        raise ValueError("the mirror models the tiled dense plans (n >= 128)")
    b = np.ascontiguousarray(b, dtype=np.float64)
    m, n = a.shape
    cap = int(max_iters) + 2
    x = np.empty(n)
    tr = np.zeros((cap, 5))
    out = np.zeros(8)
    rows = load().ts_mirror_ta_dense(a.ctypes.data, m, n, b.ctypes.data, float(eps), int(max_iters),
                                     int(sms), x.ctypes.data, tr.ctypes.data, cap, out.ctypes.data)
    return {"x": x, "status": STATUS.get(int(out[0]), str(int(out[0]))), "iterations": int(out[1]),
            "residual_norm": float(out[2]), "normal_residual_norm": float(out[3]),
            "rho": float(out[4]), "x_norm": float(out[5]), "trace": tr[: min(rows, cap)]}
