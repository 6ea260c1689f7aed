"""Residual-centering solver family (CTA) on the B200.

Drop-in for reference ``pkg/src/trisolve/centering.py``: same
``CenteringOptions`` (fields, defaults, validation messages), same
``centering_solve`` arguments / return / stopping rules, same
``moments`` / ``min_norm_coefficients`` / ``centering_step`` helpers — but
every H-application, moment, Hankel solve and update runs in the native
library, and the whole ``while`` loop of ``centering_solve`` runs on the
device as a CUDA-graph WHILE loop (see ``csrc/ts_cta.cuh``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as N
from ._solve import build_result, host_vec, rows_to_trace, trace_buffer
from .linalg import (
    H_MODE_GRAM,
    H_MODE_SYMMETRIC,
    HOperator,
    as_device_matrix,
    dot,
    local_rows,
    local_slice,
    norm2,
    shape_of,
)
from .results import (
    APPROX_SOLUTION,
    CENTERING_TRACE_COLUMNS,
    SolveResult,
    Trace,
)

MOMENT_RCOND = 1e-13     # centering.py:44
_MONOTONE_SLACK = 1e-13  # centering.py:47 (applied on the device)
DEVICE_T_MAX = 8         # largest order the device kernels are built for


class NormalEquationReached(Exception):
    """Raised by the step when ``H r = 0`` (centering.py:50-52)."""


@dataclass
class Moments:
    """``phi_1..phi_2t`` and the Krylov vectors (centering.py:55-64)."""

    t: int
    phi: np.ndarray
    krylov: list
    transposed: list | None


@dataclass
class CenteringState:
    x: np.ndarray
    r: np.ndarray
    iterations: int = 0
    schedule_pos: int = 0
    trace: Trace = field(default_factory=lambda: Trace(CENTERING_TRACE_COLUMNS))


@dataclass
class CenteringOptions:
    """Driver knobs (centering.py:124-169); identical fields and defaults."""

    epsilon: float = 1e-15
    t_max: int = 5
    max_iters: int = 100_000
    h_mode: str = H_MODE_GRAM
    enhanced: bool = False
    known_solvable: bool = False
    recheck_every: int = 250
    start: str = "zero"
    start_seed: int = 0
    rcond: float = MOMENT_RCOND
    accelerate: bool = False
    accel_ratio: float = 0.95
    accel_patience: int = 3

    def validated(self, m: int) -> "CenteringOptions":
        if not 0.0 < self.epsilon < 1.0:
            raise ValueError("epsilon must lie in (0, 1)")
        if self.t_max < 1:
            raise ValueError("t_max must be at least 1")
        if self.h_mode not in (H_MODE_SYMMETRIC, H_MODE_GRAM):
            raise ValueError(f"unknown h_mode {self.h_mode!r}")
        if self.start not in ("zero", "random"):
            raise ValueError(f"unknown start {self.start!r}")
        out = self
        if self.t_max > m:
            out = replace(out, t_max=m)
        return out


def _order_schedule(t_max: int):
    """Triangle wave 1..t_max..2 (centering.py:254-260); the device uses the
    same closed form (ts_cta.cuh: sched_order)."""
    if t_max == 1:
        while True:
            yield 1
    cycle = list(range(1, t_max + 1)) + list(range(t_max - 1, 1, -1))
    while True:
        yield from cycle


def _hmode_code(mode: str) -> int:
    return 0 if mode == H_MODE_GRAM else 1


def moments(h: HOperator, r, t: int) -> Moments:
    """``phi_k = r^T H^k r`` for k = 1..2t from t device H-applications
    (centering.py:67-84)."""
    if not 1 <= t <= h.dim:
        raise ValueError(f"order t={t} outside 1..{h.dim}")
    if t > DEVICE_T_MAX:
        raise ValueError(f"order t={t} exceeds the device limit {DEVICE_T_MAX}")
    dm = h.device_matrix
    m, n = dm.shape
    r = host_vec(r, m, f"r has wrong shape, expected ({m},)")
    phi = np.empty(2 * t)
    kry = np.empty((t + 1, m))
    gram = h.mode == H_MODE_GRAM
    tra = np.empty((t, n)) if gram else None
    N.check(N.lib().ts_moments(dm.handle, _hmode_code(h.mode), N.ptr(r), t, phi.ctypes.data,
                               kry.ctypes.data, tra.ctypes.data if gram else None, None))
    h.apply_count += t
    return Moments(t, phi, list(kry), list(tra) if gram else None)


def min_norm_coefficients(mom: Moments, order: int | None = None,
                          rcond: float = MOMENT_RCOND) -> np.ndarray:
    """Equilibrated min-norm Hankel solve, on the device (centering.py:87-110)."""
    t = mom.t if order is None else order
    if not 1 <= t <= mom.t:
        raise ValueError(f"order {t} outside 1..{mom.t}")
    phi = np.ascontiguousarray(np.asarray(mom.phi, dtype=np.float64))
    out = np.empty(t)
    rc = N.lib().ts_hankel_min_norm(phi.ctypes.data, mom.t, t, float(rcond), out.ctypes.data, None)
    if rc == N.TS_EINVAL and "SVD" in N.lib().ts_last_error().decode():
        raise np.linalg.LinAlgError("SVD did not converge in Linear Least Squares")
    N.check(rc)
    return out


def centering_step(state: CenteringState, t: int, h: HOperator, a, b) -> CenteringState:
    """One order-t step (centering.py:216-224); raises NormalEquationReached
    when ``H r = 0``."""
    dm = h.device_matrix
    m, n = dm.shape
    if not 1 <= t <= h.dim:
        raise ValueError(f"order t={t} outside 1..{h.dim}")
    x = host_vec(state.x, n, f"x has wrong shape, expected ({n},)")
    r = host_vec(state.r, m, f"r has wrong shape, expected ({m},)")
    x_out, r_out = np.empty(n), np.empty(m)
    order, atr, st = C.c_int32(), C.c_double(), C.c_int32()
    N.check(N.lib().ts_cta_step(dm.handle, _hmode_code(h.mode), N.ptr(x), N.ptr(r), t,
                                MOMENT_RCOND, x_out.ctypes.data, r_out.ctypes.data,
                                C.byref(order), C.byref(atr), C.byref(st), None))
    h.apply_count += t
    if st.value == 2:
        raise NormalEquationReached
    return CenteringState(x_out, r_out, state.iterations + 1, state.schedule_pos, state.trace)


def first_order_probe(x, r, h: HOperator, j_max: int, threshold: float, hr=None, atr=None):
    """Short first-order orbit search (centering.py:227-251): follow
    ``y <- y - (y^T H y / y^T H^2 y) H y`` for up to ``j_max - 1``
    compositions; return ``(x_hat, j)`` for the first image with
    ``|y^T H y| <= threshold``, else None.  The H-applications and inner
    products run on the device (``centering_solve(enhanced=True)`` runs the
    same probe inside its device loop)."""
    y = np.asarray(r, dtype=np.float64)
    x_hat = np.asarray(x, dtype=np.float64).copy()
    if hr is None:
        hr, atr = h.apply_with_transpose(y)
    for j in range(1, j_max):
        phi1 = dot(y, hr)
        phi2 = dot(hr, hr)
        if phi2 == 0.0:
            return None  # orbit terminated without triggering
        alpha = phi1 / phi2
        x_hat += alpha * (atr if h.mode == H_MODE_GRAM else y)
        y = y - alpha * hr
        hr, atr = h.apply_with_transpose(y)
        if abs(dot(y, hr)) <= threshold:
            return x_hat, j
    return None


def centering_solve(a, b, options: CenteringOptions | None = None) -> SolveResult:
    """Solve ``Ax = b`` (or its normal equation) by cycled centering steps
    (centering.py:263-358), entirely on the device."""
    opts = options or CenteringOptions()
    m, n = shape_of(a)
    opts = opts.validated(m)
    b = host_vec(b, m, f"b has shape {np.shape(b)}, expected ({m},)")
    b = local_rows(a, b)  # row-block shards keep their block of b
    if opts.h_mode == H_MODE_SYMMETRIC and m != n:
        # the reference returns the b = 0 early exit before building H
        if norm2(b) == 0.0:
            return SolveResult(APPROX_SOLUTION, np.zeros(n), 0.0, 0.0, 0,
                               Trace(CENTERING_TRACE_COLUMNS))
        raise ValueError("symmetric mode requires a square matrix")
    if opts.t_max > DEVICE_T_MAX:
        raise ValueError(f"t_max={opts.t_max} exceeds the device limit {DEVICE_T_MAX}")
    dm, gram = as_device_matrix(a)
    # gram: `a` is a GramProduct, the implicit normal matrix A^T A of dm (the
    # device applies it as the pass pair A^T (A v); centering.py:278)
    n_local = dm.shape[1]  # == n unless `a` is a column-sharded ShardedMatrix
    x_start = None
    if opts.start == "random":
        x_start = local_slice(a, np.random.default_rng(opts.start_seed).standard_normal(n), n_local)
    o = N.CtaOptions()
    o.epsilon = float(opts.epsilon)
    o.t_max = int(opts.t_max)
    o.h_mode = _hmode_code(opts.h_mode)
    o.max_iters = int(opts.max_iters)
    o.enhanced = int(bool(opts.enhanced))
    o.known_solvable = int(bool(opts.known_solvable))
    o.recheck_every = int(opts.recheck_every or 0)
    o.rcond = float(opts.rcond)
    o.accelerate = int(bool(opts.accelerate))
    o.accel_patience = int(opts.accel_patience)
    o.accel_ratio = float(opts.accel_ratio)
    o.x_start = x_start.ctypes.data if x_start is not None else None
    o.normal_operand = int(bool(gram))
    buf, cap = trace_buffer(opts.max_iters)
    x = N.pinned_empty(n_local)
    res = N.Result()
    N.check(N.lib().ts_cta_solve(dm.handle, N.ptr(b), C.byref(o), x.ctypes.data,
                                 buf.ctypes.data, cap, C.byref(res), None))
    trace = rows_to_trace("cta", buf, res.trace_rows, CENTERING_TRACE_COLUMNS)
    if res.trivial:
        return SolveResult(APPROX_SOLUTION, np.zeros(n_local), 0.0, 0.0, 0, trace)
    return build_result("cta", res, x, trace)
