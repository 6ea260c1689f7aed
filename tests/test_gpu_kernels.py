"""Kernel-level device checks that the golden cases (all small) do not reach:

* the sliced-ELL short-row CSR kernel (k_rows_sell, the plan for HBM-sized
  short-row matrices such as C4 and C5's A^T v) must be bitwise equal to
  scipy's csr_matvec order for A v and to the reference's ``v @ csr``
  row-order scatter for A^T v (linalg.py:42,55) on ragged inputs: empty
  rows, one very long row in a slice of short ones, a single row, a last
  slice with fewer than 32 rows;
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

LONG = 1024  # a row far longer than its slice neighbours (padding-heavy slice)


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


def _forced_matrix(a, plan):
    """DeviceMatrix with the short-row plan forced (plans are chosen at creation)."""
    import paper_2304_12168_b200 as ts

    old = os.environ.get("TS_CSR_SHORT")
    os.environ["TS_CSR_SHORT"] = plan
    try:
        return ts.DeviceMatrix(a)
    finally:
        if old is None:
            del os.environ["TS_CSR_SHORT"]
        else:
            os.environ["TS_CSR_SHORT"] = old


def _sell_matrix(a):
    return _forced_matrix(a, "sell")


CASES = [
    ("ragged", dict(m=3000, n=2000, seed=1)),
    ("wide", dict(m=500, n=40000, seed=2, max_row=200)),
    ("tall_short", dict(m=50000, n=300, seed=3, max_row=6, empty_frac=0.3)),
    ("long_in_slice", dict(m=4001, n=5000, seed=4, long_rows=((0, LONG), (17, LONG - 1),
                                                              (4000, LONG), (2000, 1000)))),
    ("single_row", dict(m=1, n=3000, seed=5, max_row=LONG, empty_frac=0.0)),
    ("all_empty_slices", dict(m=3000, n=700, seed=6, max_row=3, empty_frac=0.9)),
]


@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_sell_kernel_bitwise_scipy(name, kw):
    a = _ragged(**kw)
    dm = _sell_matrix(a)
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


def test_sell_kernel_cta_matches_thread_kernel():
    """A whole CTA solve on the sliced-ELL plan matches the thread-per-row CSR
    plan: both add every row in scipy's order (bitwise products), only the
    fused scalar reductions (phi, norms) group rows differently."""
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import workloads as W

    w = W.convdiff_upwind(60)  # 3600 x 3600 five-point operator
    dm_s = _sell_matrix(w.a)
    dm_w = _forced_matrix(w.a.copy(), "thread")
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
    e1 = _sell_matrix(s1)
    assert np.array_equal(e1.matvec(v), s1 @ v)
    del e1
    e2 = _sell_matrix(s2)  # recycled storage; the SELL tables are rebuilt
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


def test_sell_is_the_default_for_hbm_sized_short_rows():
    """Without overrides, HBM-sized short rows (nnz >= 2^21) take the
    sliced-ELL plan in both orientations: bitwise scipy, incl. empty rows and
    rows far longer than their slice neighbours (C5's A^T v shape: 10 random
    entries per row of the transpose)."""
    import paper_2304_12168_b200 as ts

    a = _ragged(300_000, 20_000, seed=21, max_row=24, empty_frac=0.05,
                long_rows=((5, 700), (299_999, 400), (150_000, 193)))
    assert a.nnz >= (1 << 21)
    dm = ts.DeviceMatrix(a)
    lp = sparse.random_array((2000, 400_000), density=0.005, random_state=22, format="csr")
    dm2 = ts.DeviceMatrix(lp)
    rng = np.random.default_rng(8)
    v = rng.standard_normal(a.shape[1])
    assert np.array_equal(dm.matvec(v), a @ v)
    w = rng.standard_normal(lp.shape[0])
    assert np.array_equal(dm2.rmatvec(w), w @ lp)
    # the LP pivot's c+ transform (v -> s * max(v, 0)) rides on the gathers
    r = ts.nonnegative_feasibility(dm2, lp @ np.abs(rng.standard_normal(lp.shape[1])), eps=1e-9, max_iters=50)
    assert r.iterations >= 1


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


def test_dense_av_and_transposed_atv_alternate():
    """Dense A v (one fused kernel) and A^T v of an L2-sized matrix (over a
    transposed copy, PLAN_TRANS, with its own partial / counter layout next
    to the A v pass's) stay correct when the two passes alternate: the
    self-resetting group counters of one never leak into the other."""
    import paper_2304_12168_b200 as ts

    rng = np.random.default_rng(12)
    a = rng.standard_normal((2300, 1700))
    dm = ts.DeviceMatrix(a)
    v = rng.standard_normal(1700)
    w = rng.standard_normal(2300)
    ref = a @ v
    scale = np.abs(a) @ np.abs(v)
    for _ in range(3):
        assert np.all(np.abs(dm.rmatvec(w) - a.T @ w) <= 1e-13 * (np.abs(a.T) @ np.abs(w)))
        assert np.all(np.abs(dm.matvec(v) - ref) <= 1e-13 * scale)
    b = a @ np.ones(1700)
    opts = ts.CenteringOptions(epsilon=1e-10, max_iters=15)
    r1, r2 = ts.centering_solve(dm, b, opts), ts.centering_solve(ts.DeviceMatrix(a), b, opts)
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.x, r2.x)


def test_column_slab_plan_wide_long_rows():
    """Long rows of a wide matrix (the C5 shape, scaled) take the column-slab
    plan (k_slab_av + k_slab_combine): A v within 1e-14 of scipy (FMA chains
    per slab, slabs added in order), the LP pivot's c+ transform applied when
    the x slab is staged, identical bits run to run; a CSR whose rows hold
    unsorted column indices keeps the warp-per-row kernel."""
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import workloads as W

    w = W.lp_columns(2000, 200_000, 10, seed=41)
    dm = ts.DeviceMatrix(w.a)
    assert dm.plans()[0] == "column_slabs"
    rng = np.random.default_rng(4)
    v = rng.standard_normal(w.a.shape[1])
    y = dm.matvec(v)
    ref = w.a @ v
    assert np.all(np.abs(y - ref) <= 1e-14 * (abs(w.a) @ np.abs(v)))
    assert np.array_equal(dm.matvec(v), y)
    bn = float(np.linalg.norm(w.b))
    r = ts.nonnegative_feasibility(dm, w.b, eps=1e-6 * bn)
    r2 = ts.nonnegative_feasibility(ts.DeviceMatrix(w.a, ), w.b, eps=1e-6 * bn)
    assert (r.status, r.iterations) == (r2.status, r2.iterations) and np.array_equal(r.x, r2.x)
    # every row's entries in descending column order (a valid, unsorted CSR):
    # no slab plan (its runs need sorted rows), the same product
    a = w.a
    idx, dat = a.indices.copy(), a.data.copy()
    for r in range(a.shape[0]):
        lo, hi = a.indptr[r], a.indptr[r + 1]
        idx[lo:hi] = idx[lo:hi][::-1]
        dat[lo:hi] = dat[lo:hi][::-1]
    uns = sparse.csr_array((dat, idx, a.indptr.copy()), shape=a.shape)
    du = ts.DeviceMatrix(uns)
    assert du.plans()[0] == "warp_rows"
    assert np.all(np.abs(du.matvec(v) - ref) <= 1e-14 * (abs(w.a) @ np.abs(v)))
