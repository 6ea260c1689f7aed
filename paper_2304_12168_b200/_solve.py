"""Shared host glue for the device solvers: argument staging, trace buffers,
and mapping the C ABI's ``ts_result`` / ``ts_trace_row`` back onto the
reference's ``SolveResult`` / ``Trace`` (results.py:23-101)."""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .linalg import _is_torch
from .results import SolveResult, Trace

# detail strings, verbatim from the reference
_DETAILS = {
    0: lambda v: "",
    1: lambda v: "non-finite residual",                                   # centering.py:299
    2: lambda v: "moment solve failed: SVD did not converge in Linear Least Squares",  # :315
    3: lambda v: f"certified ||A^T A x - A^T b|| <= {v:.3e}",            # centering.py:322
    4: lambda v: "residual drift exceeded budget",                        # centering.py:349
    5: lambda v: "non-finite iterate",                                    # triangle.py:214
    6: lambda v: "pivot direction vanished",                              # triangle.py:229
    7: lambda v: f"certified ||A^T(b - Ax)|| <= {v:.3e}",                # triangle.py:230
    8: lambda v: f"radius exceeded cap {v:.3e}",                         # triangle.py:247
    9: lambda v: "no ascent direction in the nonnegative cone section",   # feasibility.py:433
    10: lambda v: "iterate left the nonnegative cone",                   # feasibility.py:447
    11: lambda v: f"radius budget {v:.3e} exhausted",                    # feasibility.py:460
    12: lambda v: "iteration budget exhausted",                          # feasibility.py:411
    13: lambda v: "device loop watchdog tripped",                        # library-side
}

TRACE_ROW_CAP = 1 << 24


def host_vec(v, length, msg):
    """float64 contiguous numpy view (or CUDA torch tensor) of length `length`."""
    if _is_torch(v):
        if tuple(v.shape) != (length,):
            raise ValueError(msg)
        return v.contiguous().double()
    arr = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    if arr.shape != (length,):
        raise ValueError(msg)
    return arr


def trace_buffer(max_iters: int):
    cap = int(min(max(int(max_iters), 0) + 2, TRACE_ROW_CAP))
    return np.empty(cap, dtype=N.TRACE_DTYPE), cap


def detail_text(res: N.Result) -> str:
    return _DETAILS.get(int(res.detail), lambda v: "")(float(res.detail_value))


def rows_to_trace(kind: str, buf: np.ndarray, count: int, columns) -> Trace:
    tr = Trace(columns)
    count = min(int(count), len(buf))
    rows = buf[:count]
    it = rows["iter"].tolist()
    wall = rows["wall_ns"].tolist()
    tag = rows["tag"].tolist()
    v = rows["v"].tolist()
    if kind == "cta":
        tr.rows = [(it[i], tag[i], v[i][0], v[i][1], wall[i]) for i in range(count)]
    elif kind == "ta":
        tr.rows = [(it[i], v[i][0], v[i][1], v[i][2], N.EVENT_NAMES[tag[i]], wall[i])
                   for i in range(count)]
    else:
        tr.rows = [(it[i], v[i][0], v[i][1], v[i][2], N.EVENT_NAMES[tag[i]], v[i][3], wall[i])
                   for i in range(count)]
    return tr


def build_result(kind, res: N.Result, x, trace: Trace, **extra) -> SolveResult:
    out = SolveResult(
        status=N.STATUS_NAMES[int(res.status)],
        x=x,
        residual_norm=float(res.residual_norm),
        normal_residual_norm=float(res.normal_residual_norm),
        iterations=int(res.iterations),
        trace=trace,
        detail=detail_text(res),
        **extra,
    )
    out.device_ms = float(res.elapsed_ms)
    out.kernel_launches = int(res.kernel_launches)
    out.kernel_ms = tuple(float(v) for v in res.kernel_ms)
    out.kernel_count = tuple(int(v) for v in res.kernel_count)
    out.gap_norm = float(res.gap_norm)
    out.x_norm = float(res.x_norm)
    return out


def null_if_none(a):
    return None if a is None else N.ptr(a)


def isfinite(v) -> bool:
    return math.isfinite(float(v))


def stream_arg():
    return None
