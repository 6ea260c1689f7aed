"""Kernel-level device checks that the golden cases (all small) do not reach:

* the TMA-streamed short-row CSR kernel (k_rows_stream, the plan for
  HBM-sized short-row matrices such as C4 and C5's A^T v) must be bitwise
  equal to scipy's csr_matvec order for A v and to the reference's
  ``v @ csr`` row-order scatter for A^T v (linalg.py:42,55) on ragged
  inputs: empty rows, rows at the chunk-size limit, a single row, rows whose
  entries straddle 16-byte boundaries;
* matrix handles recycled by the storage pool (same shape, new entries,
  same or different sparsity) give the same answers as fresh handles;
* pinned result vectors come back correct and are recycled.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import scipy.sparse as sparse

pytestmark = pytest.mark.gpu

K_ST_CAP = 1024  # kStCap in csrc/ts_passes.cuh


def _ragged(m, n, seed, max_row=40, empty_frac=0.1, long_rows=()):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_row + 1, size=m)
    lens[rng.random(m) < empty_frac] = 0
    for r, ln in long_rows:
        lens[r] = ln
    rows, cols = [], []
    for r, ln in enumerate(lens):
        ln = min(int(ln), n)
        c = np.sort(rng.choice(n, size=ln, replace=False))
        rows.append(np.full(ln, r))
        cols.append(c)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = rng.standard_normal(rows.size)
    return sparse.csr_array((vals, (rows, cols)), shape=(m, n))


def _stream_matrix(a):
    import paper_2304_12168_b200 as ts

    old = os.environ.get("TS_CSR_SHORT")
    os.environ["TS_CSR_SHORT"] = "stream"
    try:
        return ts.DeviceMatrix(a)
    finally:
        if old is None:
            del os.environ["TS_CSR_SHORT"]
        else:
            os.environ["TS_CSR_SHORT"] = old


CASES = [
    ("ragged", dict(m=3000, n=2000, seed=1)),
    ("wide", dict(m=500, n=40000, seed=2, max_row=200)),
    ("tall_short", dict(m=50000, n=300, seed=3, max_row=6, empty_frac=0.3)),
    ("cap_rows", dict(m=4000, n=5000, seed=4, long_rows=((0, K_ST_CAP), (17, K_ST_CAP - 1),
                                                         (3999, K_ST_CAP), (2000, 1000)))),
    ("single_row", dict(m=1, n=3000, seed=5, max_row=K_ST_CAP, empty_frac=0.0)),
]


@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_stream_kernel_bitwise_scipy(name, kw):
    a = _ragged(**kw)
    dm = _stream_matrix(a)
    rng = np.random.default_rng(99)
    v = rng.standard_normal(a.shape[1])
    w = rng.standard_normal(a.shape[0])
    # long rows (>= 32 nnz on average in that orientation) take the flat split
    # kernel, which sums with FMA in four partial accumulators: 1e-14, not bitwise
    if a.nnz / a.shape[0] >= 32:
        ref = a @ v
        assert np.linalg.norm(dm.matvec(v) - ref) <= 1e-14 * np.linalg.norm(abs(a) @ abs(v))
    else:
        assert np.array_equal(dm.matvec(v), a @ v)
    if a.nnz / a.shape[1] >= 32:
        ref = w @ a
        assert np.linalg.norm(dm.rmatvec(w) - ref) <= 1e-14 * np.linalg.norm(abs(w) @ abs(a))
    else:
        assert np.array_equal(dm.rmatvec(w), w @ a)


def test_stream_kernel_cta_matches_warp_kernel():
    """A whole CTA solve on the streamed plan matches the warp-kernel plan: both
    add every row in scipy's order (bitwise products), only the fused scalar
    reductions (phi, norms) group rows differently."""
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import workloads as W

    w = W.convdiff_upwind(60)  # 3600 x 3600 five-point operator
    dm_s = _stream_matrix(w.a)
    old = os.environ.get("TS_CSR_SHORT")
    os.environ["TS_CSR_SHORT"] = "warp"
    try:
        dm_w = ts.DeviceMatrix(w.a.copy())
    finally:
        if old is None:
            del os.environ["TS_CSR_SHORT"]
        else:
            os.environ["TS_CSR_SHORT"] = old
    opts = ts.CenteringOptions(epsilon=1e-8, max_iters=60)
    rs = ts.centering_solve(dm_s, w.b, opts)
    rw = ts.centering_solve(dm_w, w.b, opts)
    assert rs.iterations == rw.iterations
    assert np.linalg.norm(rs.x - rw.x) <= 1e-10 * np.linalg.norm(rw.x)
    v = np.random.default_rng(5).standard_normal(w.a.shape[1])
    assert np.array_equal(dm_s.matvec(v), dm_w.matvec(v))
    assert np.array_equal(dm_s.rmatvec(v), dm_w.rmatvec(v))


def test_pool_recycles_dense_and_csr():
    """A handle recycled from the storage pool (same shape, new entries) solves
    exactly like a fresh one."""
    import paper_2304_12168_b200 as ts

    rng = np.random.default_rng(7)
    a1 = rng.standard_normal((300, 200))
    a2 = rng.standard_normal((300, 200))
    b = rng.standard_normal(300)
    opts = ts.CenteringOptions(epsilon=1e-8, max_iters=40)
    ref2 = ts.centering_solve(ts.DeviceMatrix(a2), b, opts)  # fresh (pool empty of this shape)
    d1 = ts.DeviceMatrix(a1)
    ts.centering_solve(d1, b, opts)  # builds instances on d1's storage
    del d1  # retired into the pool
    d2 = ts.DeviceMatrix(a2)  # recycles d1's storage, plans and graphs
    got = ts.centering_solve(d2, b, opts)
    assert got.iterations == ref2.iterations
    assert np.array_equal(got.x, ref2.x)
    assert d2.frobenius_norm() == pytest.approx(np.linalg.norm(a2), rel=1e-14)
    # CSR: same nnz, different sparsity (different plan tables)
    s1 = _ragged(4000, 3000, seed=11, max_row=8)
    nnz = s1.nnz
    s2 = _ragged(4000, 3000, seed=12, max_row=8)
    while s2.nnz != nnz:  # trim / pad to the same nnz
        s2 = _ragged(4000, 3000, seed=int(rng.integers(1 << 30)), max_row=8)
        if abs(s2.nnz - nnz) < 200:
            coo = s2.tocoo()
            k = min(s2.nnz, nnz)
            s2 = sparse.csr_array((coo.data[:k], (coo.row[:k], coo.col[:k])), shape=s2.shape)
            if s2.nnz != nnz:
                continue
    v = rng.standard_normal(3000)
    e1 = _stream_matrix(s1)
    assert np.array_equal(e1.matvec(v), s1 @ v)
    del e1
    e2 = _stream_matrix(s2)
    assert np.array_equal(e2.matvec(v), s2 @ v)
    assert np.array_equal(e2.rmatvec(np.ones(4000)), np.ones(4000) @ s2)


def test_pinned_results_are_recycled():
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import _native as N

    x = N.pinned_empty(1000)
    assert x.shape == (1000,) and x.dtype == np.float64 and x.flags.writeable
    x[:] = 3.0
    addr = x.ctypes.data
    del x
    y = N.pinned_empty(1000)
    assert y.ctypes.data == addr  # the freed block came back from the pool
    rng = np.random.default_rng(3)
    a = rng.standard_normal((50, 80))
    b = a @ rng.standard_normal(80)
    r = ts.solve_adaptive(a, b, eps=1e-6 * np.linalg.norm(b), max_iters=200)
    assert np.linalg.norm(a @ r.x - b) == pytest.approx(r.residual_norm, rel=1e-9, abs=1e-12)


def test_prefetching_warp_kernel_bitwise_scipy():
    """The prefetching short-row kernel (k_rows_warp_pf, opt-in
    TS_CSR_SHORT=pf) on HBM-sized rows of >= 8 entries (C5's A^T v shape):
    bitwise scipy in both orientations, incl. empty rows and rows spanning
    several prefetch chunks."""
    import paper_2304_12168_b200 as ts

    a = _ragged(300_000, 20_000, seed=21, max_row=24, empty_frac=0.05,
                long_rows=((5, 700), (299_999, 400), (150_000, 193)))
    assert a.nnz >= (1 << 21) and a.nnz >= 8 * a.shape[0]
    os.environ["TS_CSR_SHORT"] = "pf"
    try:
        dm = ts.DeviceMatrix(a)
        lp = sparse.random_array((2000, 400_000), density=0.005, random_state=22, format="csr")
        dm2 = ts.DeviceMatrix(lp)
    finally:
        del os.environ["TS_CSR_SHORT"]
    rng = np.random.default_rng(8)
    v = rng.standard_normal(a.shape[1])
    assert np.array_equal(dm.matvec(v), a @ v)
    w = rng.standard_normal(lp.shape[0])
    assert np.array_equal(dm2.rmatvec(w), w @ lp)


def test_thread_row_kernel_tails_bitwise_scipy():
    """The thread-per-row kernel (k_rows_short, L2-sized short-row plans)
    loads a row's last 0-3 entries as one batch and its first row's bounds
    before the state word: rows of every length 0..11 stay bitwise scipy in
    both orientations."""
    import paper_2304_12168_b200 as ts

    a = _ragged(50_000, 40_000, seed=31, max_row=11, empty_frac=0.08)
    assert a.nnz < (1 << 21)
    dm = ts.DeviceMatrix(a)
    rng = np.random.default_rng(9)
    v = rng.standard_normal(a.shape[1])
    w = rng.standard_normal(a.shape[0])
    assert np.array_equal(dm.matvec(v), a @ v)
    assert np.array_equal(dm.rmatvec(w), w @ a)


def test_split_dense_av_matches_fused():
    """TS_DENSE_N=split (tile kernel + combine kernel, the persistent loop's
    bodies) agrees with the default one-kernel dense A v to rounding: only
    the order of the per-row sum over tile partials differs."""
    import paper_2304_12168_b200 as ts

    rng = np.random.default_rng(12)
    a = rng.standard_normal((2300, 1700))
    os.environ["TS_DENSE_N"] = "split"
    try:
        d_split = ts.DeviceMatrix(a)
    finally:
        del os.environ["TS_DENSE_N"]
    d_fused = ts.DeviceMatrix(a)
    v = rng.standard_normal(1700)
    y1, y2, ref = d_split.matvec(v), d_fused.matvec(v), a @ v
    scale = np.abs(a) @ np.abs(v)
    assert np.all(np.abs(y1 - ref) <= 1e-13 * scale)
    assert np.all(np.abs(y2 - ref) <= 1e-13 * scale)
    # A^T v of this L2-sized matrix runs over a transposed copy (PLAN_TRANS)
    # with its own partial / counter layout next to the A v pass's
    w = rng.standard_normal(2300)
    for dm in (d_split, d_fused):
        for _ in range(3):  # alternate the two passes: counters stay consistent
            assert np.all(np.abs(dm.rmatvec(w) - a.T @ w) <= 1e-13 * (np.abs(a.T) @ np.abs(w)))
            assert np.all(np.abs(dm.matvec(v) - ref) <= 1e-13 * scale)
    b = a @ np.ones(1700)
    opts = ts.CenteringOptions(epsilon=1e-10, max_iters=15)
    r1, r2 = ts.centering_solve(d_split, b, opts), ts.centering_solve(d_fused, b, opts)
    assert r1.iterations == r2.iterations
    assert np.linalg.norm(r1.x - r2.x) <= 1e-9 * np.linalg.norm(r2.x)
