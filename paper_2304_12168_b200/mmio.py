"""Matrix Market ingest — drop-in for reference ``pkg/src/trisolve/mmio.py``.

Parsing runs in the native library (``ts_mm_parse``: the reference's
acceptance rules and ``line N: ...`` error texts, entries parsed in parallel).
``read_matrix_market`` / ``read_matrix_market_with_info`` return what the
reference returns (scipy CSR for coordinate files, a dense ndarray for array
files); ``read_matrix_market_device`` goes straight to a ``DeviceMatrix``:
the coordinate triplets are uploaded once and mirrored, sorted,
de-duplicated and compressed into CSR on the device (``ts_mm_to_device``),
so neither a host CSR conversion nor a second transfer sits between the file
and the solver.  ``write_matrix_market`` renders every value with the
shortest decimal string that parses back to the same float64, so
``read(write(A))`` is bit-exact (as the reference guarantees).
"""

from __future__ import annotations

import ctypes as C
import io
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import scipy.sparse as sparse

from . import _native as N
from .linalg import DeviceMatrix

BANNER = "%%MatrixMarket"
_FORMATS = ("coordinate", "array")
_FIELDS = ("real", "integer", "pattern")
_SYMMETRIES = ("general", "symmetric", "skew-symmetric")


class MatrixMarketError(ValueError):
    """Malformed Matrix Market content; message carries the 1-based line number."""


@dataclass
class MmInfo:
    """Header facts plus bookkeeping from one read (mmio.py:29-39)."""

    format: str
    field: str
    symmetry: str
    rows: int
    cols: int
    entries: int
    duplicates: int = 0


class _Info(C.Structure):
    _fields_ = [("format", C.c_int32), ("field", C.c_int32), ("symmetry", C.c_int32),
                ("reserved", C.c_int32), ("rows", C.c_int64), ("cols", C.c_int64),
                ("entries", C.c_int64), ("stored", C.c_int64)]


def _lib():
    lib = N.lib()
    if not getattr(lib, "_mm_declared", False):
        lib.ts_mm_parse.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.POINTER(C.c_void_p),
                                    C.POINTER(_Info)]
        lib.ts_mm_coo.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ts_mm_dense.argtypes = [C.c_void_p, C.c_void_p]
        lib.ts_mm_to_device.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_int64)]
        lib.ts_mm_free.argtypes = [C.c_void_p]
        for f in ("ts_mm_parse", "ts_mm_coo", "ts_mm_dense", "ts_mm_to_device", "ts_mm_free"):
            getattr(lib, f).restype = C.c_int
        lib._mm_declared = True
    return lib


class _Parsed:
    """A parsed file held by the native library."""

    def __init__(self, source):
        lib = _lib()
        self.h = C.c_void_p()
        self.info = _Info()
        if isinstance(source, (str, Path)):
            rc = lib.ts_mm_parse(os.fsencode(str(source)), 0, 1, C.byref(self.h), C.byref(self.info))
        else:
            data = source.read()
            if isinstance(data, str):
                data = data.encode("utf-8")
            rc = lib.ts_mm_parse(data, len(data), 0, C.byref(self.h), C.byref(self.info))
        if rc < 0:
            raise MatrixMarketError(lib.ts_last_error().decode(errors="replace"))
        N.check(rc)

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value and N._lib is not None:
            N._lib.ts_mm_free(self.h)
            self.h = C.c_void_p()

    def mminfo(self, duplicates=0) -> MmInfo:
        i = self.info
        return MmInfo(_FORMATS[i.format], _FIELDS[i.field], _SYMMETRIES[i.symmetry], int(i.rows),
                      int(i.cols), int(i.entries), int(duplicates))

    def host_matrix(self):
        i = self.info
        lib = _lib()
        if i.format == 0:
            k = int(i.stored)
            rows = np.empty(k, dtype=np.int32)
            cols = np.empty(k, dtype=np.int32)
            vals = np.empty(k, dtype=np.float64)
            N.check(lib.ts_mm_coo(self.h, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data))
            coo = sparse.coo_array((vals, (rows.astype(np.int64), cols.astype(np.int64))),
                                   shape=(int(i.rows), int(i.cols)))
            csr = sparse.csr_array(coo)  # sums duplicate coordinates (mmio.py:114-117)
            return csr, k - csr.nnz
        a = np.empty((int(i.rows), int(i.cols)))
        N.check(lib.ts_mm_dense(self.h, a.ctypes.data))
        return a, 0


def read_matrix_market_with_info(source):
    """Parse ``source`` (path or file-like); return ``(matrix, MmInfo)``."""
    p = _Parsed(source)
    mat, dups = p.host_matrix()
    return mat, p.mminfo(dups)


def read_matrix_market(source):
    """Parse ``source``: sparse CSR for coordinate files, dense ndarray for array files."""
    return read_matrix_market_with_info(source)[0]


def read_matrix_market_device(source, device: int = 0):
    """Parse ``source`` and build the device matrix directly: ``(DeviceMatrix,
    MmInfo)``.  Coordinate files are assembled into CSR on the device."""
    p = _Parsed(source)
    if p.info.format == 1:
        a, _ = p.host_matrix()
        return DeviceMatrix(a, device=device), p.mminfo(0)
    h = C.c_void_p()
    dups = C.c_int64()
    N.check(_lib().ts_mm_to_device(p.h, int(device), None, C.byref(h), C.byref(dups)))
    return DeviceMatrix.from_handle(h, device), p.mminfo(int(dups.value))


def _shortest(v: float) -> str:
    # Python's float repr is the shortest string that reads back to the same
    # double, which makes write -> read bit-exact.
    return repr(float(v))


def write_matrix_market(a, target) -> None:
    """Coordinate/general for sparse input, array/general for dense input."""
    if isinstance(target, (str, Path)):
        with open(target, "w", encoding="utf-8") as fh:
            fh.write(_render(a))
    else:
        target.write(_render(a))


def _render(a) -> str:
    out = io.StringIO()
    if sparse.issparse(a):
        coo = sparse.coo_array(a)
        r, c = (np.asarray(x) for x in coo.coords)
        m, n = coo.shape
        out.write(f"{BANNER} matrix coordinate real general\n{m} {n} {coo.nnz}\n")
        for k in np.lexsort((c, r)):  # row-major entry order
            out.write(f"{r[k] + 1} {c[k] + 1} {_shortest(coo.data[k])}\n")
    else:
        arr = np.asarray(a, dtype=np.float64)
        m, n = arr.shape
        out.write(f"{BANNER} matrix array real general\n{m} {n}\n")
        out.writelines(f"{_shortest(v)}\n" for v in arr.T.ravel())  # column-major
    return out.getvalue()
