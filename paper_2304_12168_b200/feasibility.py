"""Feasibility of ``{x : Ax = b, x >= 0}`` via nonnegative-cone pivots (TA-LP)
on the B200 — drop-in for reference ``pkg/src/trisolve/feasibility.py``.

The projected step (c -> c+ = max(c, 0)) is fused into the device kernels:
||c+|| is reduced alongside ||c|| in the A^T pass, the pivot matvec scales
c+ on load, and the update kernel rebuilds the preimage and reduces min(x)
for the nonnegativity guard and the trace (feasibility.py:94-132).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from ._solve import build_result, host_vec, rows_to_trace, trace_buffer
from .linalg import as_device_matrix, frobenius_norm, local_rows, matvec, norm2, shape_of
from .results import FEASIBILITY_TRACE_COLUMNS, SolveResult


def nonnegative_part(c) -> np.ndarray:
    """Componentwise ``max(c, 0)`` (feasibility.py:32-34)."""
    return np.maximum(np.asarray(c, dtype=np.float64), 0.0)


def cone_pivot_point(a, c_plus, rho):
    """``v = rho A c+ / ||c+||`` and its nonnegative preimage (feasibility.py:37-46)."""
    cp_norm = norm2(c_plus)
    if cp_norm == 0.0:
        raise ValueError("no ascent direction: c+ is zero")
    if rho <= 0.0:
        raise ValueError("rho must be positive")
    preimage = (rho / cp_norm) * np.asarray(c_plus, dtype=np.float64)
    return matvec(a, preimage), preimage


def default_rho_max(a, b) -> float:
    """``10 n max(1, ||b|| / sigma)``, sigma = ||A||_F / sqrt(m) (feasibility.py:49-56)."""
    m, n = shape_of(a)
    sigma = frobenius_norm(a) / math.sqrt(m)
    if sigma == 0.0:
        sigma = 1.0
    return 10.0 * n * max(1.0, norm2(b) / sigma)


def nonnegative_feasibility(a, b, eps, rho_max=None, max_iters=100_000) -> SolveResult:
    """Search for nonnegative x with ||Ax - b|| <= eps (feasibility.py:59-140)."""
    m, n = shape_of(a)
    b = host_vec(b, m, f"b has shape {np.shape(b)}, expected ({m},)")
    if rho_max is not None and rho_max <= 0.0:
        if norm2(b) == 0.0:
            raise ValueError("b must be nonzero")
        raise ValueError("rho_max must be positive")
    b = local_rows(a, b)  # row layouts keep their block of b
    dm, gram = as_device_matrix(a)
    nn = dm.shape[1]
    o = N.LpOptions()
    o.eps = float(eps)
    o.rho_max = -1.0 if rho_max is None else float(rho_max)
    o.max_iters = int(max_iters)
    o.gram = int(gram)
    buf, cap = trace_buffer(max_iters)
    x = N.pinned_empty(nn)
    res = N.Result()
    N.check(N.lib().ts_lp_feasibility(dm.handle, N.ptr(b), C.byref(o), x.ctypes.data,
                                      buf.ctypes.data, cap, C.byref(res), None))
    trace = rows_to_trace("lp", buf, res.trace_rows, FEASIBILITY_TRACE_COLUMNS)
    lb = float(res.lower_bound) if res.has_lower_bound else None
    return build_result("lp", res, x, trace, rho=float(res.rho), lower_bound=lb,
                        min_x_entry=float(res.min_x_entry))
