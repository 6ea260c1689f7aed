"""Column and row-block sharding of one solve across GPUs (one process per GPU).

BASELINE north_star: wide matrices (n >> m) are column-sharded; ``A^T r`` is
local and ``A x`` needs one m-vector all-reduce per pass.  This module does
the host plumbing — column partition, local slices, the IPC-handle exchange
over ``torch.distributed`` — and hands the solvers a :class:`ShardedMatrix`.
The exchange itself runs inside the solve's CUDA graph as a deterministic
one-shot all-reduce over NVLink peer memory fused into the pass epilogues
(``csrc/ts_comm.cuh``).

The drop-in solvers accept a ShardedMatrix like any other matrix; b is
replicated, the returned ``x`` is this rank's column slice (use
:meth:`ShardedMatrix.gather` for the full vector).

Square banded operators (C4: the 5-point stencil) shard by row blocks
instead (:class:`RowShardedMatrix`): rank p owns rows and
columns [r0, r1); both passes read their input vector only up to the band's
half-width past the block, so the exchange is a halo of that width with each
neighbour before every pass (8 KB on C4 at 8 ranks, instead of an 8 MB
all-reduce), plus the scalar all-reduces; every row and column is still
added in the reference's order, so operator results are bitwise those of the
unsharded path.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import scipy.sparse as sparse

from . import _native as N
from .linalg import DeviceMatrix


def column_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous column block of `rank` (same rule as the flat splits)."""
    return n * rank // world, n * (rank + 1) // world


def local_block(a, c0: int, c1: int):
    """Columns [c0, c1) of a dense array or scipy sparse matrix (CSR out)."""
    if sparse.issparse(a):
        return sparse.csr_array(sparse.csc_array(a)[:, c0:c1])
    return np.ascontiguousarray(np.asarray(a)[:, c0:c1])


class ShardedMatrix:
    """This rank's column block of A, attached to a communicator.

    ``a`` is either the full matrix (every rank slices its own block) or,
    with ``local=True``, the rank's block already (``n_global`` required).
    """

    def __init__(self, a, group=None, device: int | None = None, local: bool = False,
                 n_global: int | None = None):
        import torch
        import torch.distributed as dist

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        m, n_in = a.shape
        self.n_global = int(n_global if local else n_in)
        self.col_range = column_range(self.n_global, self.world, self.rank)
        blk = a if local else local_block(a, *self.col_range)
        self.device_matrix = DeviceMatrix(blk, device=self.device)
        self.shape = (int(m), self.n_global)
        self.local_shape = self.device_matrix.shape
        # communicator + IPC handle exchange (gloo side channel: plain bytes)
        lib = N.lib()
        self._comm = C.c_void_p()
        handles = (C.c_char * 128)()
        N.check(lib.ts_comm_create(self.device, self.rank, self.world, int(m), C.byref(self._comm),
                                   C.addressof(handles)))
        cpu_group = dist.new_group(backend="gloo") if dist.get_backend(group) != "gloo" else group
        gathered = [None] * self.world
        dist.all_gather_object(gathered, bytes(handles), group=cpu_group)
        allh = (C.c_char * (128 * self.world)).from_buffer_copy(b"".join(gathered))
        N.check(lib.ts_comm_connect(self._comm, C.addressof(allh)))
        fro2 = torch.tensor([self.device_matrix.frobenius_norm() ** 2], dtype=torch.float64)
        dist.all_reduce(fro2, group=cpu_group)
        self._fro = math.sqrt(float(fro2.item()))
        N.check(lib.ts_matrix_set_shard(self.device_matrix.handle, self._comm, self.n_global,
                                        self.col_range[0], self._fro))
        self._cpu_group = cpu_group

    def frobenius_norm(self) -> float:
        return self._fro

    def local(self, v):
        """This rank's slice of a global n-vector."""
        return np.ascontiguousarray(np.asarray(v, dtype=np.float64)[self.col_range[0]:self.col_range[1]])

    def gather(self, x_local):
        """Reassemble a global n-vector from every rank's slice (rank order)."""
        import torch.distributed as dist

        parts = [None] * self.world
        dist.all_gather_object(parts, np.asarray(x_local), group=self._cpu_group)
        return np.concatenate(parts)

    def __del__(self):
        h = getattr(self, "_comm", None)
        if h is not None and h.value and N._lib is not None:
            try:
                N._lib.ts_matrix_set_shard(self.device_matrix.handle, None, 0, 0, 0.0)
                N._lib.ts_comm_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._comm = C.c_void_p()


def row_blocks(a, r0: int, r1: int):
    """The rank's rows of a square matrix and its columns (as rows of A^T),
    both CSR with GLOBAL indices, and the halo width their indices need past
    the block [r0, r1)."""
    csr = sparse.csr_array(a)
    if csr.shape[0] != csr.shape[1]:
        raise ValueError("row-block sharding needs a square matrix")
    rows = csr[r0:r1]
    cols = sparse.csr_array(csr.T)[r0:r1]  # column j of A = row j of A^T, rows ascending
    lo, hi = r0, r1 - 1
    for blk in (rows, cols):
        if blk.nnz:
            lo = min(lo, int(blk.indices.min()))
            hi = max(hi, int(blk.indices.max()))
    return rows, cols, max(r0 - lo, hi - (r1 - 1), 0)


class RowShardedMatrix:
    """This rank's row block of a square sparse matrix (halo-exchange sharding).

    Every vector of a solve on it is split like the rows: pass the global ``b``
    (each rank keeps its block) and read back this rank's block of ``x``
    (:meth:`gather` reassembles it).
    """

    def __init__(self, a, group=None, device: int | None = None):
        import torch
        import torch.distributed as dist

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        n = int(a.shape[0])
        self.n_global = n
        self.col_range = self.row_range = column_range(n, self.world, self.rank)
        r0, r1 = self.row_range
        rows, cols, hw = row_blocks(a, r0, r1)
        cpu_group = dist.new_group(backend="gloo") if dist.get_backend(group) != "gloo" else group
        stats = torch.tensor([hw, -(r1 - r0)], dtype=torch.int64)
        dist.all_reduce(stats, op=dist.ReduceOp.MAX, group=cpu_group)
        hw, min_block = int(stats[0]), -int(stats[1])
        if hw > min_block:
            raise ValueError(f"band half-width {hw} exceeds the smallest row block ({min_block}); "
                             "use fewer ranks or ShardedMatrix")
        self.halo = hw
        lib = N.lib()
        loc = [np.ascontiguousarray(rows.indptr, dtype=np.int32),
               np.ascontiguousarray(rows.indices - r0, dtype=np.int32),
               np.ascontiguousarray(rows.data, dtype=np.float64),
               np.ascontiguousarray(cols.indptr, dtype=np.int32),
               np.ascontiguousarray(cols.indices - r0, dtype=np.int32),
               np.ascontiguousarray(cols.data, dtype=np.float64)]
        h = C.c_void_p()
        ptr = lambda v: v.ctypes.data if v.size else None  # noqa: E731
        N.check(lib.ts_matrix_create_csr_pair(ptr(loc[0]), ptr(loc[1]), ptr(loc[2]), int(rows.nnz),
                                              ptr(loc[3]), ptr(loc[4]), ptr(loc[5]), int(cols.nnz),
                                              r1 - r0, hw, self.device, None, C.byref(h)))
        self.device_matrix = DeviceMatrix.from_handle(h, self.device)
        self.shape = (n, n)
        self.local_shape = self.device_matrix.shape
        self._comm = C.c_void_p()
        handles = (C.c_char * 128)()
        N.check(lib.ts_comm_create(self.device, self.rank, self.world, max(2 * hw, 1),
                                   C.byref(self._comm), C.addressof(handles)))
        gathered = [None] * self.world
        dist.all_gather_object(gathered, bytes(handles), group=cpu_group)
        allh = (C.c_char * (128 * self.world)).from_buffer_copy(b"".join(gathered))
        N.check(lib.ts_comm_connect(self._comm, C.addressof(allh)))
        fro2 = torch.tensor([self.device_matrix.frobenius_norm() ** 2], dtype=torch.float64)
        dist.all_reduce(fro2, group=cpu_group)
        self._fro = math.sqrt(float(fro2.item()))
        N.check(lib.ts_matrix_set_row_shard(self.device_matrix.handle, self._comm, n, r0, self._fro))
        self._cpu_group = cpu_group

    def frobenius_norm(self) -> float:
        return self._fro

    def local(self, v):
        """This rank's block of a global vector (rows and columns split alike)."""
        r0, r1 = self.row_range
        return np.ascontiguousarray(np.asarray(v, dtype=np.float64)[r0:r1])

    local_rows = local

    def gather(self, x_local):
        import torch.distributed as dist

        parts = [None] * self.world
        dist.all_gather_object(parts, np.asarray(x_local), group=self._cpu_group)
        return np.concatenate(parts)

    def __del__(self):
        h = getattr(self, "_comm", None)
        if h is not None and h.value and N._lib is not None:
            try:
                N._lib.ts_matrix_set_shard(self.device_matrix.handle, None, 0, 0, 0.0)
                N._lib.ts_comm_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._comm = C.c_void_p()
