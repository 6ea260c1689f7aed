"""Column-sharded device path on one GPU (world size 1).

Exercises the full sharding machinery — communicator, IPC-handle exchange
over torch.distributed, symmetric buffers, epoch barriers, the fused
all-reduce kernels (k_ar_vec / k_ar_scalars) and the deferred finishers —
and checks it against the unsharded device path on the same inputs.  (Ranks
that wait on each other must not share one GPU, so N > 1 is covered by the
gloo host-logic tests in test_sharding_cpu.py.)
"""

from __future__ import annotations

import socket

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    import torch.distributed as dist

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1)
    yield None


def _pair(a):
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200.shard import ShardedMatrix

    return ts.DeviceMatrix(a), ShardedMatrix(a)


def test_sharded_cta_dense(group):
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import workloads as W

    w = W.dense_lowrank(120, 480, 48, seed=2)
    dm, sh = _pair(w.a)
    opts = ts.CenteringOptions(epsilon=1e-8)
    r0 = ts.centering_solve(dm, w.b, opts)
    r1 = ts.centering_solve(sh, w.b, opts)
    assert (r1.status, r1.iterations) == (r0.status, r0.iterations)
    assert rel_l2(r1.x, r0.x) <= 1e-11
    assert r1.residual_norm == pytest.approx(r0.residual_norm, rel=1e-9)
    assert r1.kernel_launches > r0.kernel_launches  # the all-reduce kernels ran


def test_sharded_ta_and_lp_sparse(group):
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import workloads as W

    w = W.lp_columns(60, 3000, 10, seed=5)
    dm, sh = _pair(w.a)
    bn = float(np.linalg.norm(w.b))
    for fn, kw in ((ts.solve_adaptive, dict(eps=1e-6 * bn)),
                   (ts.nonnegative_feasibility, dict(eps=1e-6 * bn))):
        r0 = fn(dm, w.b, **kw)
        r1 = fn(sh, w.b, **kw)
        assert (r1.status, r1.iterations) == (r0.status, r0.iterations)
        assert [row[4] for row in r1.trace.rows] == [row[4] for row in r0.trace.rows]
        assert rel_l2(r1.x, r0.x) <= 1e-11
    # random start + a short recheck cadence on the sharded CTA (sparse,
    # ill-conditioned: compare inside the parity window)
    w3 = W.clement_variant(301, seed=3)
    dm3, sh3 = _pair(w3.a)
    opts = ts.CenteringOptions(epsilon=1e-8, max_iters=40, start="random", start_seed=4,
                               recheck_every=16)
    r0 = ts.centering_solve(dm3, w3.b, opts)
    r1 = ts.centering_solve(sh3, w3.b, opts)
    assert (r1.status, r1.iterations) == (r0.status, r0.iterations)
    assert rel_l2(r1.x, r0.x) <= 1e-9
    assert r1.residual_norm == pytest.approx(r0.residual_norm, rel=1e-6)


def test_row_sharded_cta_and_ta_convdiff(group):
    """Row-block sharding (RowShardedMatrix: halo exchange kernel, both
    orientations given per rank, every reduction deferred to the scalar
    all-reduce) at world size 1 against the unsharded path: the passes add
    every row / column in the same order, so x must be bitwise equal."""
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import workloads as W
    from paper_2304_12168_b200.shard import RowShardedMatrix

    w = W.convdiff_upwind(40, seed=2)  # 1600 x 1600 five-point operator
    dm = ts.DeviceMatrix(w.a)
    rs = RowShardedMatrix(w.a)
    assert rs.halo == 0 and rs.local_shape == w.a.shape
    opts = ts.CenteringOptions(epsilon=1e-8, max_iters=50)
    r0 = ts.centering_solve(dm, w.b, opts)
    r1 = ts.centering_solve(rs, w.b, opts)
    assert (r1.status, r1.iterations) == (r0.status, r0.iterations)
    assert np.array_equal(r1.x, r0.x)
    assert r1.residual_norm == r0.residual_norm
    assert r1.kernel_launches > r0.kernel_launches  # halo + scalar all-reduce kernels ran
    bn = float(np.linalg.norm(w.b))
    t0 = ts.solve_adaptive(dm, w.b, eps=1e-6 * bn, max_iters=60)
    t1 = ts.solve_adaptive(rs, w.b, eps=1e-6 * bn, max_iters=60)
    assert (t1.status, t1.iterations) == (t0.status, t0.iterations)
    assert np.array_equal(t1.x, t0.x)
