"""Operator layer on the B200: device-resident matrices and the reference's
``matvec`` / ``matvec_transpose`` / ``norm2`` / ``frobenius_norm`` /
``HOperator`` / ``GramProduct`` (reference ``pkg/src/trisolve/linalg.py:1-149``).

``DeviceMatrix`` is the plug-in point: it implements the reference's operator
protocol (``.matvec`` / ``.rmatvec`` / ``.shape`` / ``.frobenius_norm``,
linalg.py:4-8, 37-38, 48-49, 65-66), so even the unmodified reference drivers
accept it, while this package's drivers recognise it and run the whole
iteration on the device.  Upload once, solve many times::

    A = DeviceMatrix(a)          # ndarray, scipy sparse, or a CUDA torch tensor
    res = centering_solve(A, b)  # no host<->device traffic for A

Every product here runs in the native library; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sparse

from . import _native as N

H_MODE_SYMMETRIC = "a"
H_MODE_GRAM = "aat"


def is_sparse(a) -> bool:
    return sparse.issparse(a)


def shape_of(a) -> tuple[int, int]:
    m, n = a.shape
    return int(m), int(n)


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch") and hasattr(a, "data_ptr")


class DeviceMatrix:
    """Immutable device copy of a dense (row-major) or CSR fp64 matrix, with a
    device-built transposed CSR for deterministic ``A^T v``.

    Safe to share across threads and concurrent solves (linalg.py:10-13).
    """

    def __init__(self, a, device: int = 0, stream=None):
        """``stream``: a torch CUDA stream or a raw ``cudaStream_t`` for the
        upload and the device-side preparation (transpose, plans, Frobenius
        norm); the handle is ready when the constructor returns.  A
        non-blocking stream lets a new matrix upload while solves on other
        streams run (double-buffered pipelines of same-shaped problems)."""
        lib = N.lib()
        self.device = int(device)
        self._handle = C.c_void_p()
        if stream is not None and not isinstance(stream, int):
            stream = int(stream.cuda_stream)
        if isinstance(a, DeviceMatrix):
            raise TypeError("already a DeviceMatrix")
        if sparse.issparse(a):
            csr = a if a.format == "csr" else a.tocsr()
            m, n = shape_of(csr)
            if csr.nnz >= 2**31 - 1:
                raise ValueError("nnz exceeds the int32 index range")
            indptr = np.ascontiguousarray(csr.indptr, dtype=np.int32)
            indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
            data = np.ascontiguousarray(csr.data, dtype=np.float64)
            N.check(lib.ts_matrix_create_csr(
                indptr.ctypes.data, indices.ctypes.data if indices.size else None,
                data.ctypes.data if data.size else None, m, n, int(csr.nnz), self.device,
                stream, C.byref(self._handle)))
        elif _is_torch(a):
            if a.dim() != 2 or a.dtype.__str__() != "torch.float64":
                raise ValueError("torch matrices must be 2-D float64")
            t = a.contiguous()
            m, n = int(t.shape[0]), int(t.shape[1])
            N.check(lib.ts_matrix_create_dense(t.data_ptr(), m, n, n, self.device, stream,
                                               C.byref(self._handle)))
        else:
            arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
            if arr.ndim != 2:
                raise ValueError(f"matrix must be 2-D, got shape {arr.shape}")
            m, n = arr.shape
            N.check(lib.ts_matrix_create_dense(arr.ctypes.data, m, n, n, self.device, stream,
                                               C.byref(self._handle)))
        self._read_info()

    @classmethod
    def from_handle(cls, handle, device: int = 0) -> "DeviceMatrix":
        """Adopt a ``ts_matrix`` handle built by the native library (device-side
        ingest); the new object owns and destroys it."""
        obj = cls.__new__(cls)
        obj.device = int(device)
        obj._handle = handle if isinstance(handle, C.c_void_p) else C.c_void_p(handle)
        obj._read_info()
        return obj

    def _read_info(self):
        lib = N.lib()
        mm, nn, nz, kind, fro = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_double()
        N.check(lib.ts_matrix_info(self._handle, C.byref(mm), C.byref(nn), C.byref(nz),
                                   C.byref(kind), C.byref(fro)))
        self.shape = (int(mm.value), int(nn.value))
        self.nnz = int(nz.value)
        self.kind = "dense" if kind.value == 0 else "csr"
        self._fro = float(fro.value)

    @property
    def handle(self):
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and N._lib is not None:
            try:
                N._lib.ts_matrix_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._handle = C.c_void_p()

    def frobenius_norm(self) -> float:
        return self._fro

    def matvec(self, v):
        v = _as_vec(v, self.shape[1], "matvec: vector has length {got}, matrix has {want} columns")
        out = np.empty(self.shape[0])
        N.check(N.lib().ts_matvec(self._handle, N.ptr(v), out.ctypes.data, None))
        return out

    def rmatvec(self, v):
        v = _as_vec(v, self.shape[0],
                    "matvec_transpose: vector has length {got}, matrix has {want} rows")
        out = np.empty(self.shape[1])
        N.check(N.lib().ts_rmatvec(self._handle, N.ptr(v), out.ctypes.data, None))
        return out

    def gram_matvec(self, v):
        v = _as_vec(v, self.shape[1], "gram: vector has length {got}, expected {want}")
        out = np.empty(self.shape[1])
        N.check(N.lib().ts_gram_matvec(self._handle, N.ptr(v), out.ctypes.data, None))
        return out

    PLAN_NAMES = {0: "flat", 1: "thread_rows", 2: "dense_tiles", 7: "warp_rows", 9: "dense_transposed",
                  10: "sliced_ell", 11: "column_slabs",
                  12: "column_tiles_transposed_copy"}

    def plans(self) -> tuple[str, str]:
        """The kernels chosen for A v and A^T v."""
        pn, pt = C.c_int32(), C.c_int32()
        N.check(N.lib().ts_matrix_plans(self.handle, C.byref(pn), C.byref(pt)))
        return self.PLAN_NAMES.get(pn.value, str(pn.value)), self.PLAN_NAMES.get(pt.value, str(pt.value))

    def __repr__(self):
        return f"DeviceMatrix({self.kind}, shape={self.shape}, nnz={self.nnz}, device={self.device})"


def _as_vec(v, length, msg):
    if _is_torch(v):
        if tuple(v.shape) != (length,):
            raise ValueError(msg.format(got=tuple(v.shape), want=length))
        return v.contiguous().double()
    arr = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    if arr.shape != (length,):
        raise ValueError(msg.format(got=arr.shape, want=length))
    return arr


def as_device_matrix(a):
    """Return ``(DeviceMatrix, gram_flag)`` for any supported operand:
    ``DeviceMatrix``, ``GramProduct`` (implicit A^T A), ndarray, scipy sparse
    or CUDA torch tensor.  Other duck-typed operators cannot run on the
    device and raise ``TypeError`` (no CPU fallback)."""
    if isinstance(a, DeviceMatrix):
        return a, False
    if isinstance(a, GramProduct):
        return a.device_matrix, True
    if getattr(a, "_ts_shard", False):  # shard.py layouts
        return a.device_matrix, False
    if isinstance(a, np.ndarray) or sparse.issparse(a) or _is_torch(a):
        return DeviceMatrix(a), False
    if hasattr(a, "shape") and not hasattr(a, "matvec"):
        return DeviceMatrix(np.asarray(a, dtype=np.float64)), False
    raise TypeError(
        f"operator of type {type(a).__name__} cannot run on the device path; pass an ndarray, "
        "a scipy sparse matrix, a DeviceMatrix or a GramProduct")


def local_slice(a, v, n_local: int):
    """For a sharded matrix, this rank's part of an n-space vector given
    either globally or already locally; identity otherwise."""
    if v is None or not getattr(a, "_ts_shard", False):
        return v
    return a.local_x(v)


def local_rows(a, b):
    """For a sharded matrix, this rank's part of an m-space vector (b): its
    block on row layouts, the whole vector on column blocks; identity for
    unsharded operands."""
    if b is None or not getattr(a, "_ts_shard", False):
        return b
    return np.ascontiguousarray(a.local_b(b), dtype=np.float64)


def matvec(a, v) -> np.ndarray:
    """``A @ v`` (linalg.py:34-42) on the device."""
    if isinstance(a, (DeviceMatrix, GramProduct)):
        return a.matvec(v)
    if hasattr(a, "matvec") and not isinstance(a, np.ndarray) and not sparse.issparse(a):
        return a.matvec(np.asarray(v, dtype=np.float64))
    dm, _ = as_device_matrix(a)
    return dm.matvec(v)


def matvec_transpose(a, v) -> np.ndarray:
    """``A.T @ v`` from the same storage (linalg.py:45-56) on the device."""
    if isinstance(a, (DeviceMatrix, GramProduct)):
        return a.rmatvec(v)
    if hasattr(a, "rmatvec") and not isinstance(a, np.ndarray) and not sparse.issparse(a):
        return a.rmatvec(np.asarray(v, dtype=np.float64))
    dm, _ = as_device_matrix(a)
    return dm.rmatvec(v)


def norm2(v) -> float:
    """Euclidean norm (linalg.py:59-61), reduced on the device."""
    if _is_torch(v):
        v = v.contiguous().double()
        n = int(v.numel())
    else:
        v = np.ascontiguousarray(np.asarray(v, dtype=np.float64)).ravel()
        n = v.size
    out = C.c_double()
    N.check(N.lib().ts_norm2(N.ptr(v) if n else None, n, C.addressof(out), None))
    return float(out.value)


def residual(a, x, b, want_normal: bool = True, want_vector: bool = False):
    """``r = b - A x`` on the device: returns ``(||r||, ||A^T r||)`` (and ``r``
    with ``want_vector``) — the honest-residual step of the drivers
    (triangle.py:84-89, hybrid.py:102-104)."""
    dm, gram = as_device_matrix(a)
    m, n = dm.shape
    if gram:  # `a` is a GramProduct: r = b - A^T A x in n-space
        m = n
    x = _as_vec(x, n, "x has length {got}, expected {want}")
    b = _as_vec(b, m, "b has length {got}, expected {want}")
    rn, an = C.c_double(), C.c_double()
    r = np.empty(m) if want_vector else None
    fn = N.lib().ts_gram_residual if gram else N.lib().ts_residual
    N.check(fn(dm.handle, N.ptr(x), N.ptr(b), r.ctypes.data if r is not None else None,
               C.byref(rn), C.byref(an) if want_normal else None, None))
    out = (float(rn.value), float(an.value) if want_normal else None)
    return out + (r,) if want_vector else out


def dot(u, v) -> float:
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64)).ravel()
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64)).ravel()
    if u.shape != v.shape:
        raise ValueError("dot: shapes differ")
    out = C.c_double()
    N.check(N.lib().ts_dot(N.ptr(u) if u.size else None, N.ptr(v) if v.size else None, u.size,
                           C.addressof(out), None))
    return float(out.value)


def frobenius_norm(a) -> float:
    """``||A||_F`` (linalg.py:64-69), computed once on the device per matrix."""
    if isinstance(a, (DeviceMatrix, GramProduct)):
        return a.frobenius_norm()
    if hasattr(a, "frobenius_norm") and not isinstance(a, np.ndarray) and not sparse.issparse(a):
        return a.frobenius_norm()
    dm, _ = as_device_matrix(a)
    return dm.frobenius_norm()


class GramProduct:
    """Implicit ``A^T A`` (n x n) applied as ``A^T (A v)`` (linalg.py:93-114);
    symmetric, so ``rmatvec`` is ``matvec``."""

    def __init__(self, a):
        self._a = a
        self.device_matrix = a if isinstance(a, DeviceMatrix) else DeviceMatrix(a)
        m, n = shape_of(self.device_matrix)
        self.shape = (n, n)

    def matvec(self, v):
        return self.device_matrix.gram_matvec(v)

    rmatvec = matvec

    def frobenius_norm(self) -> float:
        return self.device_matrix.frobenius_norm() ** 2


class HOperator:
    """The solver-side operator H (linalg.py:117-149): ``"a"`` applies A
    (caller asserts symmetry), ``"aat"`` applies ``A (A^T r)`` without forming
    ``A A^T``.  Counts applications like the reference."""

    def __init__(self, a, mode: str = H_MODE_GRAM):
        if mode not in (H_MODE_SYMMETRIC, H_MODE_GRAM):
            raise ValueError(f"unknown H mode {mode!r}")
        m, n = shape_of(a)
        if mode == H_MODE_SYMMETRIC and m != n:
            raise ValueError("symmetric mode requires a square matrix")
        self.matrix = a
        self.device_matrix, _ = as_device_matrix(a) if not isinstance(a, GramProduct) else (None, True)
        if self.device_matrix is None:
            raise TypeError("HOperator over a GramProduct is not supported on the device path")
        self.mode = mode
        self.dim = m
        self.apply_count = 0

    def apply(self, r):
        return self.apply_with_transpose(r)[0]

    def apply_with_transpose(self, r):
        self.apply_count += 1
        dm = self.device_matrix
        if self.mode == H_MODE_SYMMETRIC:
            return dm.matvec(r), None
        at_r = dm.rmatvec(r)
        return dm.matvec(at_r), at_r

    def quadratic_form(self, r, hr) -> float:
        return dot(r, hr)


def nnz_of(a) -> int:
    """Stored nonzeros of a sparse matrix, else the nonzero count
    (linalg.py:72-76)."""
    if isinstance(a, DeviceMatrix):
        return int(a.nnz)
    if sparse.issparse(a):
        return int(a.nnz)
    return int(np.count_nonzero(np.asarray(a)))


def validate_symmetric(a, rel_tol: float = 1e-12) -> bool:
    """Debug check that ``a`` is square and symmetric (linalg.py:79-90).  A
    host-side O(n^2) helper, never called by the solvers (as in the reference)."""
    m, n = shape_of(a)
    if m != n:
        return False
    if sparse.issparse(a):
        d = a - a.T
        num = float(np.sqrt(abs((d.multiply(d)).sum())))
    else:
        arr = np.asarray(a)
        num = float(np.linalg.norm(arr - arr.T, "fro"))
    return num <= rel_tol * max(frobenius_norm(a), 1.0)
