"""World-size-2 gloo tests of the column-sharded path's host logic (CPU only).

Two processes each hold one column block; the sharded iteration model
(tests/sharded_model.py, the decomposition csrc/ts_comm.cuh implements) must
reproduce the unsharded reference oracle: same status, iteration count and
pivot/expand sequence, x and residuals to rounding.
"""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    import sharded_model as SM
    from paper_2304_12168_b200 import workloads as W
    from paper_2304_12168_b200.shard import column_range, local_block

    if case == "cta_dense":
        w = W.dense_lowrank(60, 240, 24, seed=3)
        c0, c1 = column_range(w.a.shape[1], world, rank)
        out = SM.cta_sharded(local_block(w.a, c0, c1), w.b, 1e-8, 200)
    elif case == "ta_dense":
        w = W.dense_gaussian(40, 90, seed=4)
        c0, c1 = column_range(w.a.shape[1], world, rank)
        out = SM.ta_adaptive_sharded(local_block(w.a, c0, c1), w.b,
                                     1e-8 * np.linalg.norm(w.b), 30)
    elif case == "cta_rows_convdiff":  # C4 family, row blocks + halo exchange
        from paper_2304_12168_b200.shard import row_blocks

        w = W.convdiff_upwind(24, seed=2)
        c0, c1 = column_range(w.a.shape[0], world, rank)
        rows, cols, hw = row_blocks(w.a, c0, c1)
        import torch
        t = torch.tensor([hw], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        hw = int(t.item())
        rows_ext, cols_ext = SM.shifted_blocks(rows, cols, c0, hw)
        out = SM.cta_row_sharded(rows_ext, cols_ext, hw, w.b[c0:c1], 1e-8, 40)
    elif case in ("cta_tall", "ta_tall"):  # tall row blocks, n-vector all-reduce
        from paper_2304_12168_b200.shard import row_block

        rng = np.random.default_rng(13)
        a = rng.standard_normal((300, 70))
        b = a @ rng.standard_normal(70)
        c0, c1 = column_range(300, world, rank)
        if case == "cta_tall":
            out = SM.cta_tall_sharded(row_block(a, c0, c1), b[c0:c1], 1e-8, 60)
        else:
            out = SM.ta_tall_sharded(row_block(a, c0, c1), b[c0:c1], 1e-8 * np.linalg.norm(b), 40)
    else:  # lp_sparse: the C5 family (cone stall)
        w = W.lp_columns(60, 3000, 10, seed=5)
        c0, c1 = column_range(w.a.shape[1], world, rank)
        out = SM.ta_adaptive_sharded(local_block(w.a, c0, c1), w.b,
                                     1e-6 * np.linalg.norm(w.b), 1000, lp=True)
    np.savez(os.path.join(outdir, f"{case}_{rank}.npz"), x=out["x"], c0=c0, c1=c1,
             iterations=out["iterations"], status=out["status"],
             residual_norm=out["residual_norm"], events=np.array(out.get("events", [])))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cta_dense", "ta_dense", "lp_sparse", "cta_rows_convdiff",
                                  "cta_tall", "ta_tall"])
def test_sharded_decomposition_matches_oracle(case, tmp_path):
    import torch.multiprocessing as mp

    from oracle import port
    from paper_2304_12168_b200 import workloads as W

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(os.path.join(tmp_path, f"{case}_{r}.npz")) for r in range(world)]
    x = np.concatenate([p["x"] for p in parts])
    if case.endswith("_tall"):  # x is replicated on tall row blocks
        assert np.array_equal(parts[0]["x"], parts[1]["x"])
        x = parts[0]["x"]
    if case == "cta_dense":
        w = W.dense_lowrank(60, 240, 24, seed=3)
        ref = port.cta_solve(w.a, w.b, epsilon=1e-8, max_iters=200)
    elif case == "ta_dense":
        w = W.dense_gaussian(40, 90, seed=4)
        ref = port.ta_adaptive(w.a, w.b, eps=1e-8 * np.linalg.norm(w.b), max_iters=30)
    elif case == "cta_rows_convdiff":
        w = W.convdiff_upwind(24, seed=2)
        ref = port.cta_solve(w.a, w.b, epsilon=1e-8, max_iters=40)
    elif case.endswith("_tall"):
        rng = np.random.default_rng(13)
        a = rng.standard_normal((300, 70))
        b = a @ rng.standard_normal(70)
        ref = (port.cta_solve(a, b, epsilon=1e-8, max_iters=60) if case == "cta_tall" else
               port.ta_adaptive(a, b, eps=1e-8 * np.linalg.norm(b), max_iters=40))
    else:
        w = W.lp_columns(60, 3000, 10, seed=5)
        ref = port.lp_feasibility(w.a, w.b, eps=1e-6 * np.linalg.norm(w.b), max_iters=1000)
    for p in parts:  # every rank takes identical decisions
        assert str(p["status"]) == ref["status"]
        assert int(p["iterations"]) == ref["iterations"]
        assert float(p["residual_norm"]) == pytest.approx(ref["residual_norm"], rel=1e-9)
    if "trace" in ref and not case.startswith("cta"):
        assert list(parts[0]["events"]) == [row[4] for row in ref["trace"]]
    assert np.linalg.norm(x - ref["x"]) <= 1e-9 * max(np.linalg.norm(ref["x"]), 1e-300)


def test_column_partition_covers_all_columns():
    from paper_2304_12168_b200.shard import column_range

    for n in (1, 7, 1000, 1_000_000):
        for world in (1, 2, 3, 8):
            ranges = [column_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(b - a for a, b in ranges) - min(b - a for a, b in ranges) <= 1


def test_local_block_dense_and_sparse():
    import scipy.sparse as sp

    from paper_2304_12168_b200.shard import local_block

    rng = np.random.default_rng(0)
    dense = rng.standard_normal((7, 11)) * (rng.random((7, 11)) < 0.4)
    csr = sp.csr_array(dense)
    for c0, c1 in ((0, 4), (4, 11), (3, 3)):
        assert np.array_equal(local_block(dense, c0, c1), dense[:, c0:c1])
        blk = local_block(csr, c0, c1)
        assert blk.format == "csr"
        assert np.array_equal(blk.toarray(), dense[:, c0:c1])


def test_row_blocks_halo_width():
    from paper_2304_12168_b200 import workloads as W
    from paper_2304_12168_b200.shard import column_range, row_blocks

    w = W.convdiff_upwind(10, seed=1)  # 5-point stencil: half-bandwidth = grid = 10
    n = w.a.shape[0]
    for world in (1, 2, 3):
        for rank in range(world):
            r0, r1 = column_range(n, world, rank)
            rows, cols, hw = row_blocks(w.a, r0, r1)
            assert hw == (0 if world == 1 else 10)
            assert rows.shape == (r1 - r0, n) and cols.shape == (r1 - r0, n)
            assert rows.indices.min() >= r0 - hw and rows.indices.max() < r1 + hw
            # columns of A as rows of A^T, row indices ascending (the reference's order)
            assert all(np.all(np.diff(cols.indices[cols.indptr[i]:cols.indptr[i + 1]]) > 0)
                       for i in range(r1 - r0))
            assert np.array_equal(cols.toarray(), w.a.toarray()[:, r0:r1].T)
