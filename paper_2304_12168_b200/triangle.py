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
import math
import time

import numpy as np

from . import _native as N
from ._solve import build_result, host_vec, rows_to_trace, trace_buffer
from .linalg import (GramProduct, as_device_matrix, dot, local_rows, local_slice, matvec, matvec_transpose, norm2,
                     residual, shape_of)
from .results import (
    APPROX_SOLUTION,
    ITERATION_CAP,
    MIN_NORM_SOLUTION,
    NORMAL_EQ_SOLUTION,
    TRIANGLE_TRACE_COLUMNS,
    WITNESS,
    SolveResult,
    Trace,
)

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
    b = local_rows(a, b)  # row layouts keep their block of b
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
    x = N.pinned_empty(nn)
    bp = N.pinned_empty(mo)
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
    b = local_rows(a, b)  # row-block shards keep their block of b
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
    x = N.pinned_empty(nn)
    res = N.Result()
    N.check(N.lib().ts_ta_adaptive(dm.handle, N.ptr(b), C.byref(o), x.ctypes.data,
                                   buf.ctypes.data, cap, C.byref(res), None))
    trace = rows_to_trace("ta", buf, res.trace_rows, TRIANGLE_TRACE_COLUMNS)
    if res.trivial:
        return SolveResult(APPROX_SOLUTION, np.zeros(nn), 0.0, 0.0, 0,
                           Trace(TRIANGLE_TRACE_COLUMNS), rho=0.0)
    return build_result("ta", res, x, trace, rho=float(res.rho))


def min_norm_solve(a, b, eps, x_eps, inner_cap=250_000, max_iters=4_000_000) -> SolveResult:
    """Approximate minimum-norm solution by bisection on the ellipsoid radius
    (triangle.py:254-330).  Each bisection step is one warm-started device
    membership loop (``solve_in_ball`` on the cached instance, CUDA-graph
    WHILE loop); the host keeps only the bracket ``[rho_lo, rho_hi]`` and the
    outer trace rows, exactly like the reference's driver."""
    m, n = shape_of(a)
    b = host_vec(b, m, f"b has shape {np.shape(b)}, expected ({m},)")
    if norm2(b) == 0.0:
        raise ValueError("b must be nonzero")
    dm, gram = as_device_matrix(a)
    # the operand of the inner solves and residuals: A, or the implicit A^T A
    # (a GramProduct: every apply is the device pass pair A^T (A v))
    op = GramProduct(dm) if gram else dm
    x_eps = host_vec(local_slice(a, x_eps, dm.shape[1]), dm.shape[1], "x_eps has wrong shape")
    start_gap, _ = residual(op, x_eps, b, want_normal=False)
    if start_gap > eps * (1.0 + 1e-9):
        raise ValueError(
            f"x_eps is not an eps-approximate solution: ||Ax-b|| = {start_gap:.3e} > {eps:.3e}")
    zero_floor = 1e-14 * op.frobenius_norm() * norm2(b)  # floating floor for "||c|| > 0"

    rho_hi = norm2(x_eps)
    rho_lo = 0.0
    best_x = np.array(x_eps, copy=True)
    warm = None
    trace = Trace(TRIANGLE_TRACE_COLUMNS)
    t0 = time.perf_counter_ns()
    iterations = 0
    status = MIN_NORM_SOLUTION
    detail = ""
    device_ms = 0.0
    launches = 0

    def finish(st, x, **extra):
        rn, an = residual(op, x, b)
        out = SolveResult(st, x, rn, an, iterations, trace, **extra)
        out.device_ms = device_ms
        out.kernel_launches = launches
        return out

    outer_budget = max(8, int(math.ceil(math.log2(max(rho_hi / eps, 2.0)))) + 8)
    for _ in range(outer_budget):
        if rho_hi - rho_lo <= eps or iterations >= max_iters:
            break
        rho = 0.5 * (rho_hi + rho_lo)
        if rho <= 0.0:
            break
        inner = solve_in_ball(op, b, rho, 0.25 * eps, eps_prime=zero_floor,
                              max_iters=min(inner_cap, max_iters - iterations), x0=warm)
        device_ms += inner.device_ms or 0.0
        launches += inner.kernel_launches or 0
        for row in inner.trace.rows:  # iteration_offset (triangle.py:300)
            trace.rows.append((iterations + row[0],) + tuple(row[1:]))
        iterations += inner.iterations
        wall = time.perf_counter_ns() - t0
        gap = inner.gap_norm
        if inner.status == APPROX_SOLUTION:
            best_x = inner.x
            rho_hi = min(rho, inner.x_norm)
            warm = inner.x
            trace.append(iterations, rho_hi, gap, 0.0, "shrink", wall)
        elif inner.status == WITNESS:
            rho_lo = min(max(rho_lo, inner.lower_bound), rho_hi)
            warm = inner.x
            trace.append(iterations, rho_lo, gap, 0.0, "expand", wall)
        elif inner.status == NORMAL_EQ_SOLUTION:
            return finish(NORMAL_EQ_SOLUTION, inner.x, rho=rho, rho_interval=(rho_lo, rho_hi),
                          detail="pivot direction vanished during bisection")
        else:
            status = inner.status
            detail = ("inner membership test exhausted its budget"
                      if inner.status == ITERATION_CAP else "non-finite iterate")
            break

    if status == MIN_NORM_SOLUTION and rho_hi - rho_lo > eps:
        status, detail = ITERATION_CAP, "bisection budget exhausted"
    return finish(status, best_x, rho=rho_hi, rho_interval=(rho_lo, rho_hi), detail=detail)
