"""ctypes binding of ``libtrisolve_b200.so`` (the C ABI in include/trisolve_b200.h).

The library is built in-tree (``make`` / ``__graft_entry__.build()``) into
``paper_2304_12168_b200/_lib/``.  There is no fallback: if the library or a
CUDA device is missing, every entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TS_LIB_PATH") or os.path.join(_HERE, "_lib", "libtrisolve_b200.so")

ABI_VERSION = 2  # TS_ABI_VERSION of include/trisolve_b200.h

EXPORTS = (
    "ts_abi_version", "ts_last_error", "ts_device_count",
    "ts_matrix_create_dense", "ts_matrix_create_csr", "ts_matrix_destroy", "ts_matrix_info",
    "ts_matrix_plans",
    "ts_matvec", "ts_rmatvec", "ts_gram_matvec", "ts_norm2", "ts_dot", "ts_residual", "ts_gram_residual",
    "ts_moments", "ts_hankel_min_norm", "ts_cta_step", "ts_time_pass",
    "ts_cta_solve", "ts_ta_adaptive", "ts_ta_in_ball", "ts_lp_feasibility",
    "ts_comm_create", "ts_comm_connect", "ts_comm_destroy", "ts_matrix_set_shard",
    "ts_pool_trim", "ts_host_alloc", "ts_host_free",
    "ts_mm_parse", "ts_mm_coo", "ts_mm_dense", "ts_mm_to_device", "ts_mm_free",
    "ts_matrix_create_csr_pair", "ts_matrix_set_row_shard", "ts_matrix_set_tall_shard",
    "ts_comm_create_local",
    "ts_matrix_gen_stencil5", "ts_matrix_gen_clement",
)

# statuses (results.py:11-18)
STATUS_NAMES = {
    1: "approx_solution", 2: "normal_eq_solution", 3: "min_norm_solution", 4: "witness",
    5: "feasible", 6: "inconclusive", 7: "iteration_cap", 8: "numerical_failure",
}
EVENT_NAMES = ("pivot", "expand", "witness")

TS_EINVAL = -1
TS_EDEGENERATE = -2


class TraceRow(C.Structure):
    _fields_ = [("iter", C.c_int64), ("wall_ns", C.c_int64), ("tag", C.c_int32),
                ("reserved", C.c_int32), ("v", C.c_double * 4)]


TRACE_DTYPE = np.dtype([("iter", "<i8"), ("wall_ns", "<i8"), ("tag", "<i4"),
                        ("reserved", "<i4"), ("v", "<f8", (4,))])
assert TRACE_DTYPE.itemsize == C.sizeof(TraceRow)


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("detail", C.c_int32), ("iterations", C.c_int64),
                ("residual_norm", C.c_double), ("normal_residual_norm", C.c_double),
                ("rho", C.c_double), ("lower_bound", C.c_double), ("min_x_entry", C.c_double),
                ("detail_value", C.c_double), ("trace_rows", C.c_int64),
                ("has_lower_bound", C.c_int32), ("trivial", C.c_int32),
                ("elapsed_ms", C.c_double), ("kernel_launches", C.c_int64),
                ("kernel_ms", C.c_double * 4), ("kernel_count", C.c_int64 * 4),
                ("gap_norm", C.c_double), ("x_norm", C.c_double)]


class CtaOptions(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("t_max", C.c_int32), ("h_mode", C.c_int32),
                ("max_iters", C.c_int64), ("enhanced", C.c_int32), ("known_solvable", C.c_int32),
                ("recheck_every", C.c_int64), ("rcond", C.c_double), ("accelerate", C.c_int32),
                ("accel_patience", C.c_int32), ("accel_ratio", C.c_double),
                ("x_start", C.c_void_p), ("normal_operand", C.c_int32), ("reserved", C.c_int32)]


class TaOptions(C.Structure):
    _fields_ = [("eps", C.c_double), ("eps_prime", C.c_double), ("rho_cap", C.c_double),
                ("max_iters", C.c_int64), ("restart_halvings", C.c_int32),
                ("gram", C.c_int32), ("x0", C.c_void_p)]


class BallOptions(C.Structure):
    _fields_ = [("rho", C.c_double), ("eps", C.c_double), ("eps_prime", C.c_double),
                ("max_iters", C.c_int64), ("x0", C.c_void_p), ("gram", C.c_int32),
                ("reserved", C.c_int32)]


class LpOptions(C.Structure):
    _fields_ = [("eps", C.c_double), ("rho_max", C.c_double), ("max_iters", C.c_int64),
                ("gram", C.c_int32), ("reserved", C.c_int32)]


_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double


def _declare(lib):
    sig = {
        "ts_abi_version": ([], C.c_int),
        "ts_last_error": ([], C.c_char_p),
        "ts_device_count": ([C.POINTER(C.c_int)], C.c_int),
        "ts_matrix_create_dense": ([_P, _I64, _I64, _I64, C.c_int, _P, C.POINTER(_P)], C.c_int),
        "ts_matrix_create_csr": ([_P, _P, _P, _I64, _I64, _I64, C.c_int, _P, C.POINTER(_P)],
                                 C.c_int),
        "ts_matrix_destroy": ([_P], C.c_int),
        "ts_pool_trim": ([C.c_int], C.c_int),
        "ts_host_alloc": ([C.c_size_t, C.POINTER(_P)], C.c_int),
        "ts_host_free": ([_P], C.c_int),
        "ts_matrix_info": ([_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64),
                            C.POINTER(_I32), C.POINTER(_D)], C.c_int),
        "ts_matrix_plans": ([_P, C.POINTER(_I32), C.POINTER(_I32)], C.c_int),
        "ts_matvec": ([_P, _P, _P, _P], C.c_int),
        "ts_rmatvec": ([_P, _P, _P, _P], C.c_int),
        "ts_gram_matvec": ([_P, _P, _P, _P], C.c_int),
        "ts_norm2": ([_P, _I64, _P, _P], C.c_int),
        "ts_dot": ([_P, _P, _I64, _P, _P], C.c_int),
        "ts_residual": ([_P, _P, _P, _P, C.POINTER(_D), C.POINTER(_D), _P], C.c_int),
        "ts_gram_residual": ([_P, _P, _P, _P, C.POINTER(_D), C.POINTER(_D), _P], C.c_int),
        "ts_moments": ([_P, _I32, _P, _I32, _P, _P, _P, _P], C.c_int),
        "ts_hankel_min_norm": ([_P, _I32, _I32, _D, _P, _P], C.c_int),
        "ts_cta_step": ([_P, _I32, _P, _P, _I32, _D, _P, _P, C.POINTER(_I32), C.POINTER(_D),
                         C.POINTER(_I32), _P], C.c_int),
        "ts_time_pass": ([_P, _I32, _I32, C.POINTER(_D), _P], C.c_int),
        "ts_comm_create": ([C.c_int, C.c_int, C.c_int, _I64, C.POINTER(_P), _P], C.c_int),
        "ts_comm_connect": ([_P, _P], C.c_int),
        "ts_comm_destroy": ([_P], C.c_int),
        "ts_matrix_set_shard": ([_P, _P, _I64, _I64, _D], C.c_int),
        "ts_matrix_set_row_shard": ([_P, _P, _I64, _I64, _D], C.c_int),
        "ts_matrix_set_tall_shard": ([_P, _P, _I64, _I64, _D], C.c_int),
        "ts_comm_create_local": ([C.c_int, C.c_int, _I64, _P, _P], C.c_int),
        "ts_matrix_gen_stencil5": ([_I64, _D, _D, _D, _D, _D, _I32, C.c_int, _P, C.POINTER(_P)],
                                   C.c_int),
        "ts_matrix_gen_clement": ([_I64, C.c_int, _P, C.POINTER(_P)], C.c_int),
        "ts_matrix_create_csr_pair": ([_P, _P, _P, _I64, _P, _P, _P, _I64, _I64, _I64, C.c_int, _P,
                                       C.POINTER(_P)], C.c_int),
        "ts_cta_solve": ([_P, _P, C.POINTER(CtaOptions), _P, _P, _I64, C.POINTER(Result), _P],
                         C.c_int),
        "ts_ta_adaptive": ([_P, _P, C.POINTER(TaOptions), _P, _P, _I64, C.POINTER(Result), _P],
                           C.c_int),
        "ts_ta_in_ball": ([_P, _P, C.POINTER(BallOptions), _P, _P, _P, _I64, C.POINTER(Result),
                          _P], C.c_int),
        "ts_lp_feasibility": ([_P, _P, C.POINTER(LpOptions), _P, _P, _I64, C.POINTER(Result), _P],
                              C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def load_library(path: str = LIB_PATH):
    """Load (once) and return the CDLL.  Raises RuntimeError when missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"trisolve_b200 native library not built: {path} is missing "
                    "(run `make` or __graft_entry__.build()); there is no CPU fallback")
            lib = C.CDLL(path)
            _declare(lib)
            if lib.ts_abi_version() != ABI_VERSION:  # structs would be misread: refuse a stale build
                raise RuntimeError(f"{path} implements ABI {lib.ts_abi_version()}, this package "
                                   f"expects {ABI_VERSION}: rebuild it (`make`)")
            _lib = lib
    return _lib


def lib():
    return load_library()


def check(rc: int):
    """Map a C ABI return code onto the reference's exception types."""
    if rc == 0:
        return
    msg = lib().ts_last_error().decode(errors="replace")
    if rc < 0:
        raise ValueError(msg)
    raise RuntimeError(f"trisolve_b200 CUDA failure ({rc}): {msg}")


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().ts_device_count(C.byref(n))
    if rc != 0:
        return 0
    return int(n.value)


class _PinnedBlock:
    """Owner of one page-locked host block from the library's pool, exposed
    to numpy through the array interface (the array keeps it alive)."""

    __slots__ = ("_p", "__array_interface__")

    def __init__(self, count: int, dtype):
        dt = np.dtype(dtype)
        p = C.c_void_p()
        check(lib().ts_host_alloc(max(count, 1) * dt.itemsize, C.byref(p)))
        self._p = p.value
        self.__array_interface__ = {"shape": (count,), "typestr": dt.str,
                                    "data": (self._p, False), "version": 3}

    def __del__(self):
        p = getattr(self, "_p", None)
        if p and _lib is not None:
            try:
                _lib.ts_host_free(p)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._p = None


def pinned_empty(count: int, dtype=np.float64) -> np.ndarray:
    """Uninitialised 1-D numpy array in pinned host memory (result vectors:
    the device->host copy then runs at full PCIe rate)."""
    return np.asarray(_PinnedBlock(int(count), dtype))


def trim_pools(device: int = -1) -> None:
    """Release retired matrix storage and cached pinned host blocks."""
    check(lib().ts_pool_trim(int(device)))


def ptr(arr) -> int | None:
    """Raw address of a contiguous float64/int32 numpy array or torch tensor."""
    if arr is None:
        return None
    if isinstance(arr, np.ndarray):
        return arr.ctypes.data
    if hasattr(arr, "data_ptr"):
        return int(arr.data_ptr())
    raise TypeError(f"cannot take the address of {type(arr)!r}")


def current_stream(device: int = 0):
    """The torch current stream on `device` when torch has CUDA, else NULL
    (the legacy default stream)."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream(device).cuda_stream or None
    except Exception:  # pragma: no cover - torch optional
        pass
    return None
