"""Sharding one solve across GPUs (one process per GPU), and emulated worlds.

BASELINE north_star / SURVEY.md 8(e): wide matrices (n >> m) are column-
sharded — ``A^T r`` is local, ``A x`` needs one m-vector all-reduce per pass;
tall matrices are row-sharded symmetrically — ``A x`` is local, ``A^T r``
needs one n-vector all-reduce per pass; square banded operators (C4: the
5-point stencil) shard by row blocks with a halo exchange of the band's
half-width instead of an all-reduce.  This module does the host plumbing —
partitions, local blocks, the communicators and their IPC-handle exchange
over ``torch.distributed`` — and hands the solvers a shard object.  The
exchanges themselves run inside the solve on the device: deterministic
one-shot all-reduces and halo copies over NVLink peer memory fused into the
pass epilogues (``csrc/ts_comm.cuh``), every sum in fixed rank order, so all
ranks hold bit-identical replicated vectors and take identical decisions.

Communicators are per process (one per (group, device), reused by every
shard built on that group and grown only when a larger vector is needed), as
is the gloo side channel the IPC handles travel on.

:class:`LocalWorld` runs the same sharded device code for ``world`` ranks
inside ONE process on ONE GPU (a rank per host thread, every exchange ordered
on the host between producer and consumer kernels): how the N > 1 paths are
exercised on a single B200, where ranks whose kernels spin on each other must
not share the GPU.

The drop-in solvers accept any shard object like a matrix.  ``b`` may be
given globally (row layouts keep their block); ``x`` comes back as the rank's
column slice (column layout) or replicated (row layouts: the rank's block
for square row blocks); :meth:`gather` reassembles global vectors.
"""

from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import math
import threading

import numpy as np
import scipy.sparse as sparse

from . import _native as N
from .linalg import DeviceMatrix

HANDLE_BYTES = 128  # IPC handles per rank (csrc: sym + flags)


def column_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous block of `rank` (same rule as the flat splits)."""
    return n * rank // world, n * (rank + 1) // world


def local_block(a, c0: int, c1: int):
    """Columns [c0, c1) of a dense array or scipy sparse matrix (CSR out)."""
    if sparse.issparse(a):
        return sparse.csr_array(sparse.csc_array(a)[:, c0:c1])
    return np.ascontiguousarray(np.asarray(a)[:, c0:c1])


def row_block(a, r0: int, r1: int):
    """Rows [r0, r1) of a dense array or scipy sparse matrix (CSR out)."""
    if sparse.issparse(a):
        return sparse.csr_array(a)[r0:r1]
    return np.ascontiguousarray(np.asarray(a)[r0:r1])


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


# ------------------------------------------------------------ communicators --
class Communicator:
    """One rank's ``ts_comm`` handle: symmetric slots + epoch flags."""

    def __init__(self, handle: C.c_void_p, rank: int, world: int, device: int, capacity: int,
                 side_group=None, local: bool = False):
        self.handle = handle
        self.rank, self.world, self.device = rank, world, device
        self.capacity = capacity
        self.side_group = side_group
        self.local = local

    def close(self, barrier: bool = True) -> None:
        """Free the slots.  Across processes every rank first meets on the side
        channel, so no peer still reads this rank's slots over NVLink."""
        if self.handle is None or not self.handle.value or N._lib is None:
            return
        if barrier and self.side_group is not None:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.barrier(group=self.side_group)
        N._lib.ts_comm_destroy(self.handle)
        self.handle = C.c_void_p()


_SIDE: dict = {}
_COMMS: dict = {}
_COMM_LOCK = threading.Lock()


def side_group(group=None):
    """The gloo side channel of `group` (created once per group and process)."""
    import torch.distributed as dist

    key = id(group)
    if key not in _SIDE:
        _SIDE[key] = group if dist.get_backend(group) == "gloo" else dist.new_group(backend="gloo")
    return _SIDE[key]


def communicator(group, device: int, capacity: int) -> Communicator:
    """This process's communicator on `group` with room for `capacity`
    doubles per slot.  Collective: every rank calls it with the same capacity
    (the shard constructors agree on it first), so every rank reuses or
    creates the same communicator."""
    import torch.distributed as dist

    key = (id(group), int(device))
    with _COMM_LOCK:
        for c in _COMMS.get(key, []):
            if c.capacity >= capacity and c.handle.value:
                return c
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    cpu = side_group(group)
    lib = N.lib()
    h = C.c_void_p()
    handles = (C.c_char * HANDLE_BYTES)()
    N.check(lib.ts_comm_create(device, rank, world, int(capacity), C.byref(h), C.addressof(handles)))
    gathered = [None] * world
    dist.all_gather_object(gathered, bytes(handles), group=cpu)
    allh = (C.c_char * (HANDLE_BYTES * world)).from_buffer_copy(b"".join(gathered))
    N.check(lib.ts_comm_connect(h, C.addressof(allh)))
    c = Communicator(h, rank, world, device, int(capacity), side_group=cpu)
    with _COMM_LOCK:
        _COMMS.setdefault(key, []).append(c)
    return c


def close_communicators() -> None:
    """Release every cached communicator of this process (collective)."""
    with _COMM_LOCK:
        comms = [c for cs in _COMMS.values() for c in cs]
        _COMMS.clear()
    for c in comms:
        c.close()


class _DistCtx:
    """torch.distributed plumbing of a shard constructor."""

    def __init__(self, group, device):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.cpu = side_group(group)

    def sum(self, v: float) -> float:
        import torch
        import torch.distributed as dist

        t = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(t, group=self.cpu)
        return float(t.item())

    def max_int(self, vals):
        import torch
        import torch.distributed as dist

        t = torch.tensor([int(v) for v in vals], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.cpu)
        return [int(v) for v in t.tolist()]

    def comm(self, capacity: int) -> Communicator:
        return communicator(self.group, self.device, capacity)


# ------------------------------------------------------------------- shards --
class _Shard:
    """Common protocol of the shard objects seen by the solvers."""

    _ts_shard = True
    layout = ""

    def frobenius_norm(self) -> float:
        return self._fro

    # vectors of the solve, given globally or already local
    def local_x(self, v):
        """This rank's part of an n-space vector (x0, x_start)."""
        return v

    def local_b(self, b):
        """This rank's part of an m-space vector (b)."""
        return b

    def gather(self, x_local):
        """Reassemble a global vector from every rank's part (rank order)."""
        if self.comm.local:
            raise RuntimeError("emulated world: use LocalWorld.gather")
        import torch.distributed as dist

        parts = [None] * self.world
        dist.all_gather_object(parts, np.asarray(x_local), group=self.comm.side_group)
        return np.concatenate(parts)

    def _finish(self, dm: DeviceMatrix, comm: Communicator, fro: float, attach) -> None:
        self.device_matrix = dm
        self.local_shape = dm.shape
        self.comm = comm
        self.rank, self.world, self.device = comm.rank, comm.world, comm.device
        self._fro = float(fro)
        N.check(attach(N.lib(), dm.handle, comm.handle, self._fro))

    def __del__(self):
        dm = getattr(self, "device_matrix", None)
        if dm is not None and N._lib is not None:
            try:
                N._lib.ts_matrix_set_shard(dm.handle, None, 0, 0, 0.0)  # detach
            except Exception:  # pragma: no cover - interpreter shutdown
                pass


class ShardedMatrix(_Shard):
    """This rank's column block of A (wide matrices: C5, C2).

    ``a`` is either the full matrix (every rank slices its own block) or,
    with ``local=True``, the rank's block already (``n_global`` required).
    m-vectors (b, r, ...) are replicated; x is the rank's column slice.
    """

    layout = "columns"

    def __init__(self, a, group=None, device: int | None = None, local: bool = False,
                 n_global: int | None = None):
        ctx = _DistCtx(group, device)
        m, n_in = a.shape
        n = int(n_global if local else n_in)
        cr = column_range(n, ctx.world, ctx.rank)
        blk = a if local else local_block(a, *cr)
        dm = DeviceMatrix(blk, device=ctx.device)
        fro = math.sqrt(ctx.sum(dm.frobenius_norm() ** 2))
        self._setup(dm, ctx.comm(int(m)), (int(m), n), cr, fro)

    def _setup(self, dm, comm, shape, cr, fro):
        self.shape = shape
        self.n_global = shape[1]
        self.col_range = cr
        self._finish(dm, comm, fro, lambda L, h, c, f: L.ts_matrix_set_shard(h, c, shape[1], cr[0], f))

    def local_x(self, v):
        if v is None:
            return v
        arr = np.asarray(v, dtype=np.float64)
        return self.local(arr) if arr.shape == (self.n_global,) else arr

    def local(self, v):
        """This rank's slice of a global n-vector."""
        return np.ascontiguousarray(np.asarray(v, dtype=np.float64)[self.col_range[0]:self.col_range[1]])


class RowShardedMatrix(_Shard):
    """This rank's row block of a square banded sparse matrix (halo sharding).

    Every vector of a solve on it is split like the rows: pass the global
    ``b`` (each rank keeps its block) and read back this rank's block of
    ``x`` (:meth:`gather` reassembles it).  Operator results are bitwise those
    of the unsharded path (each row / column added in the reference's order).
    """

    layout = "rows"

    def __init__(self, a, group=None, device: int | None = None, blocks=None):
        """``blocks``: this rank's ``row_blocks(a, r0, r1)`` already sliced
        (rows, columns as rows of A^T, halo width) — a caller building shards
        repeatedly slices once."""
        ctx = _DistCtx(group, device)
        n = int(a.shape[0])
        rr = column_range(n, ctx.world, ctx.rank)
        rows, cols, hw = blocks if blocks is not None else row_blocks(a, *rr)
        hw, neg_min_block = ctx.max_int([hw, -(rr[1] - rr[0])])
        _check_halo(hw, -neg_min_block)
        dm = _pair_matrix(rows, cols, rr, hw, ctx.device)
        fro = math.sqrt(ctx.sum(dm.frobenius_norm() ** 2))
        self._setup(dm, ctx.comm(max(2 * hw, 1)), n, rr, hw, fro)

    def _setup(self, dm, comm, n, rr, hw, fro):
        self.n_global = n
        self.shape = (n, n)
        self.col_range = self.row_range = rr
        self.halo = hw
        self._finish(dm, comm, fro, lambda L, h, c, f: L.ts_matrix_set_row_shard(h, c, n, rr[0], f))

    def local(self, v):
        """This rank's block of a global vector (rows and columns split alike)."""
        r0, r1 = self.row_range
        return np.ascontiguousarray(np.asarray(v, dtype=np.float64)[r0:r1])

    local_rows = local

    def local_x(self, v):
        if v is None:
            return v
        arr = np.asarray(v, dtype=np.float64)
        return self.local(arr) if arr.shape == (self.n_global,) else arr

    def local_b(self, b):
        if b is None:
            return b
        arr = np.asarray(b, dtype=np.float64)
        return self.local(arr) if arr.shape == (self.n_global,) else arr


class TallShardedMatrix(_Shard):
    """This rank's row block of a tall matrix (m >> n), all n columns.

    The mirror image of :class:`ShardedMatrix`: b-space vectors (b, b', r,
    the Krylov p-vectors) are the rank's row block, x-space vectors are
    replicated; ``A^T r`` sums an n-vector over ranks in rank order.  ``x``
    comes back replicated on every rank.
    """

    layout = "tall"

    def __init__(self, a, group=None, device: int | None = None):
        ctx = _DistCtx(group, device)
        m, n = (int(s) for s in a.shape)
        rr = column_range(m, ctx.world, ctx.rank)
        dm = DeviceMatrix(row_block(a, *rr), device=ctx.device)
        fro = math.sqrt(ctx.sum(dm.frobenius_norm() ** 2))
        self._setup(dm, ctx.comm(n), (m, n), rr, fro)

    def _setup(self, dm, comm, shape, rr, fro):
        self.shape = shape
        self.m_global, self.n_global = shape
        self.row_range = rr
        self._finish(dm, comm, fro, lambda L, h, c, f: L.ts_matrix_set_tall_shard(h, c, shape[0], rr[0], f))

    def local(self, v):
        """This rank's block of a global m-vector."""
        r0, r1 = self.row_range
        return np.ascontiguousarray(np.asarray(v, dtype=np.float64)[r0:r1])

    def local_b(self, b):
        if b is None:
            return b
        arr = np.asarray(b, dtype=np.float64)
        return self.local(arr) if arr.shape == (self.m_global,) else arr


def _check_halo(hw: int, min_block: int) -> None:
    if hw > min_block:
        raise ValueError(f"band half-width {hw} exceeds the smallest row block ({min_block}); "
                         "use fewer ranks or ShardedMatrix")


def _pair_matrix(rows, cols, rr, hw, device) -> DeviceMatrix:
    r0, r1 = rr
    loc = [np.ascontiguousarray(rows.indptr, dtype=np.int32),
           np.ascontiguousarray(rows.indices - r0, dtype=np.int32),
           np.ascontiguousarray(rows.data, dtype=np.float64),
           np.ascontiguousarray(cols.indptr, dtype=np.int32),
           np.ascontiguousarray(cols.indices - r0, dtype=np.int32),
           np.ascontiguousarray(cols.data, dtype=np.float64)]
    h = C.c_void_p()
    ptr = lambda v: v.ctypes.data if v.size else None  # noqa: E731
    N.check(N.lib().ts_matrix_create_csr_pair(ptr(loc[0]), ptr(loc[1]), ptr(loc[2]), int(rows.nnz),
                                              ptr(loc[3]), ptr(loc[4]), ptr(loc[5]), int(cols.nnz),
                                              r1 - r0, hw, device, None, C.byref(h)))
    return DeviceMatrix.from_handle(h, device)


def shard_matrix(a, group=None, device: int | None = None):
    """The north_star layout for `a`: square banded sparse -> row blocks with
    halos; tall (m > n) -> row blocks with an n-vector all-reduce; otherwise
    (wide) -> column blocks with an m-vector all-reduce."""
    import torch.distributed as dist

    m, n = a.shape
    if m == n and sparse.issparse(a):
        world = dist.get_world_size(group)
        rr = column_range(n, world, dist.get_rank(group))
        _, _, hw = row_blocks(a, *rr)
        if hw <= n // max(world, 1):
            return RowShardedMatrix(a, group, device)
    if m > n:
        return TallShardedMatrix(a, group, device)
    return ShardedMatrix(a, group, device)


# ---------------------------------------------------------- emulated worlds --
class LocalWorld:
    """``world`` ranks of this process on one GPU (see the module docstring).

    Build every rank's shard with :meth:`columns` / :meth:`rows` /
    :meth:`tall`, then run one solve per rank with :meth:`run` (one host
    thread per rank).  Solves of an emulated world take the direct launch path
    (one host-ordered iteration at a time), so they are a correctness vehicle
    for the sharded device code, not a performance one.
    """

    def __init__(self, world: int, device: int = 0, devices=None):
        """``devices``: the GPU of every rank (default: all on ``device``, an
        emulated world; distinct GPUs read each other's slots over NVLink)."""
        if world < 1:
            raise ValueError("world must be positive")
        self.world = int(world)
        self.device = int(device)
        self.devices = [int(d) for d in devices] if devices is not None else [self.device] * self.world
        if len(self.devices) != self.world:
            raise ValueError("one device per rank expected")
        self._comms: list[list[Communicator]] = []

    def comms(self, capacity: int) -> list[Communicator]:
        for cs in self._comms:
            if cs[0].capacity >= capacity:
                return cs
        arr = (C.c_void_p * self.world)()
        devs = (C.c_int32 * self.world)(*self.devices)
        N.check(N.lib().ts_comm_create_local(self.device, self.world, int(capacity), devs, arr))
        cs = [Communicator(C.c_void_p(arr[r]), r, self.world, self.devices[r], int(capacity), local=True)
              for r in range(self.world)]
        self._comms.append(cs)
        return cs

    def columns(self, a) -> list[ShardedMatrix]:
        m, n = (int(s) for s in a.shape)
        crs = [column_range(n, self.world, r) for r in range(self.world)]
        dms = [DeviceMatrix(local_block(a, *cr), device=d) for cr, d in zip(crs, self.devices)]
        fro = math.sqrt(sum(dm.frobenius_norm() ** 2 for dm in dms))
        cs = self.comms(m)
        out = []
        for r in range(self.world):
            s = ShardedMatrix.__new__(ShardedMatrix)
            s._setup(dms[r], cs[r], (m, n), crs[r], fro)
            out.append(s)
        return out

    def rows(self, a) -> list[RowShardedMatrix]:
        n = int(a.shape[0])
        rrs = [column_range(n, self.world, r) for r in range(self.world)]
        blocks = [row_blocks(a, *rr) for rr in rrs]
        hw = max(b[2] for b in blocks)
        _check_halo(hw, min(rr[1] - rr[0] for rr in rrs))
        dms = [_pair_matrix(b[0], b[1], rr, hw, d) for b, rr, d in zip(blocks, rrs, self.devices)]
        fro = math.sqrt(sum(dm.frobenius_norm() ** 2 for dm in dms))
        cs = self.comms(max(2 * hw, 1))
        out = []
        for r in range(self.world):
            s = RowShardedMatrix.__new__(RowShardedMatrix)
            s._setup(dms[r], cs[r], n, rrs[r], hw, fro)
            out.append(s)
        return out

    def tall(self, a) -> list[TallShardedMatrix]:
        m, n = (int(s) for s in a.shape)
        rrs = [column_range(m, self.world, r) for r in range(self.world)]
        dms = [DeviceMatrix(row_block(a, *rr), device=d) for rr, d in zip(rrs, self.devices)]
        fro = math.sqrt(sum(dm.frobenius_norm() ** 2 for dm in dms))
        cs = self.comms(n)
        out = []
        for r in range(self.world):
            s = TallShardedMatrix.__new__(TallShardedMatrix)
            s._setup(dms[r], cs[r], (m, n), rrs[r], fro)
            out.append(s)
        return out

    def shard(self, a) -> list:
        """Every rank's shard in the north_star layout for `a` (see
        shard_matrix): square banded sparse -> row blocks with halos, tall ->
        row blocks, else column blocks."""
        m, n = a.shape
        if m == n and sparse.issparse(a):
            try:
                return self.rows(a)
            except ValueError:  # band wider than a row block: column blocks
                pass
        return self.tall(a) if m > n else self.columns(a)

    def run(self, fn, shards, *args, **kw) -> list:
        """``fn(shard, *args, **kw)`` for every rank at once (one host thread
        each); results in rank order.  The first failure is re-raised."""
        if len(shards) != self.world:
            raise ValueError("one shard per rank expected")
        with cf.ThreadPoolExecutor(max_workers=self.world) as ex:
            futs = [ex.submit(fn, s, *args, **kw) for s in shards]
            return [f.result() for f in futs]

    @staticmethod
    def gather(parts) -> np.ndarray:
        return np.concatenate([np.asarray(p) for p in parts])

    def close(self) -> None:
        for cs in self._comms:
            for c in cs:
                c.close(barrier=False)
        self._comms = []
