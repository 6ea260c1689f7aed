"""Ellipsoid-membership solvers (Triangle Algorithm) on the B200.

Drop-in for reference ``pkg/src/trisolve/triangle.py``: ``solve_in_ball``
(fixed radius, Alg. 2.1) and ``solve_adaptive`` (growing radius, Alg. 2.2)
keep the reference's arguments, return values, statuses, trace schema and
stopping rules; their iteration loops run on the device (``csrc/ts_state.cuh``:
c = A^T(b - b') with fused ||c||, the pivot matvec with fused d.d / gap.d, and
the convex-combination update with fused ||gap|| / gap.b).  The per-step
helpers (``pivot_direction`` ...) are thin conveniences over the device
operator layer.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from ._solve import build_result, host_vec, rows_to_trace, trace_buffer
from .linalg import as_device_matrix, dot, local_slice, matvec, matvec_transpose, norm2, shape_of
from .results import APPROX_SOLUTION, TRIANGLE_TRACE_COLUMNS, SolveResult, Trace

_REVALIDATE_EVERY = 512   # triangle.py:37 (device cadence)
_INNER_EPS_FACTOR = 0.25  # triangle.py:43


def pivot_direction(a, b, b_prime) -> np.ndarray:
    """``c = A^T (b - b')`` (triangle.py:46-48)."""
    return matvec_transpose(a, np.asarray(b, dtype=np.float64) - np.asarray(b_prime, dtype=np.float64))


def pivot_point(a, c, rho):
    """``v = rho A c / ||c||`` and its preimage (triangle.py:51-60)."""
    c_norm = norm2(c)
    if c_norm == 0.0:
        raise ValueError("pivot direction is zero; caller must branch to the witness case")
    if rho <= 0.0:
        raise ValueError("rho must be positive")
    preimage = (rho / c_norm) * np.asarray(c, dtype=np.float64)
    return matvec(a, preimage), preimage


def is_strict_pivot(rho, c, b, b_prime) -> bool:
    """``rho ||c|| >= (b - b')^T b`` (triangle.py:63-66)."""
    gap = np.asarray(b, dtype=np.float64) - np.asarray(b_prime, dtype=np.float64)
    return rho * norm2(c) >= dot(gap, b)


def move_to_pivot(b_prime, x_prime, v, preimage, b):
    """Nearest point of segment [b', v] to b (triangle.py:69-81)."""
    b_prime = np.asarray(b_prime, dtype=np.float64)
    d = np.asarray(v, dtype=np.float64) - b_prime
    denom = dot(d, d)
    if denom == 0.0:
        raise ValueError("degenerate pivot: v coincides with the iterate")
    alpha = dot(np.asarray(b, dtype=np.float64) - b_prime, d) / denom
    alpha = min(1.0, max(0.0, alpha))
    return (b_prime + alpha * d,
            (1.0 - alpha) * np.asarray(x_prime, dtype=np.float64) + alpha * np.asarray(preimage),
            alpha)


def _dims(a):
    dm, gram = as_device_matrix(a)
    n = dm.shape[1]
    mo = n if gram else dm.shape[0]
    return dm, gram, mo, n


def solve_in_ball(a, b, rho, eps, eps_prime=None, max_iters=100_000, x0=None) -> SolveResult:
    """Membership test at fixed radius (triangle.py:92-113)."""
    m, n = shape_of(a)
    b = host_vec(b, m, f"b has shape {np.shape(b)}, expected ({m},)")
    if rho <= 0.0:
        # the reference checks b != 0 first
        if norm2(b) == 0.0:
            raise ValueError("b must be nonzero")
        raise ValueError("rho must be positive")
    dm, gram, mo, nn = _dims(a)
    o = N.BallOptions()
    o.rho = float(rho)
    o.eps = float(eps)
    o.eps_prime = float(eps if eps_prime is None else eps_prime)
    o.max_iters = int(max_iters)
    x0v = host_vec(local_slice(a, x0, nn), nn, "x0 has wrong shape") if x0 is not None else None
    o.x0 = N.ptr(x0v) if x0v is not None else None
    o.gram = int(gram)
    buf, cap = trace_buffer(max_iters)
    x = np.empty(nn)
    bp = np.empty(mo)
    res = N.Result()
    N.check(N.lib().ts_ta_in_ball(dm.handle, N.ptr(b), C.byref(o), x.ctypes.data, bp.ctypes.data,
                                  buf.ctypes.data, cap, C.byref(res), None))
    trace = rows_to_trace("ta", buf, res.trace_rows, TRIANGLE_TRACE_COLUMNS)
    extra = {"rho": float(rho), "b_prime": bp}
    if res.has_lower_bound and N.STATUS_NAMES[int(res.status)] == "witness":
        extra["lower_bound"] = float(res.lower_bound)
    return build_result("ta", res, x, trace, **extra)


def solve_adaptive(a, b, eps, eps_prime=None, rho_cap=None, max_iters=100_000,
                   x0=None, restart_halvings: int = 0) -> SolveResult:
    """Growing-radius solver (triangle.py:170-251), loop on the device."""
    m, n = shape_of(a)
    b = host_vec(b, m, f"b has shape {np.shape(b)}, expected ({m},)")
    dm, gram, mo, nn = _dims(a)
    o = N.TaOptions()
    o.eps = float(eps)
    o.eps_prime = -1.0 if eps_prime is None else float(eps_prime)
    o.rho_cap = -1.0 if rho_cap is None else float(rho_cap)
    o.max_iters = int(max_iters)
    o.restart_halvings = int(max(0, restart_halvings))
    o.gram = int(gram)
    x0v = host_vec(local_slice(a, x0, nn), nn, "x0 has wrong shape") if x0 is not None else None
    o.x0 = N.ptr(x0v) if x0v is not None else None
    buf, cap = trace_buffer(max_iters)
    x = np.empty(nn)
    res = N.Result()
    N.check(N.lib().ts_ta_adaptive(dm.handle, N.ptr(b), C.byref(o), x.ctypes.data,
                                   buf.ctypes.data, cap, C.byref(res), None))
    trace = rows_to_trace("ta", buf, res.trace_rows, TRIANGLE_TRACE_COLUMNS)
    if res.trivial:
        return SolveResult(APPROX_SOLUTION, np.zeros(nn), 0.0, 0.0, 0,
                           Trace(TRIANGLE_TRACE_COLUMNS), rho=0.0)
    return build_result("ta", res, x, trace, rho=float(res.rho))
