"""Seeded synthetic inputs for the five BASELINE.json configurations.

These are host-side generators (numpy, PCG64 via ``default_rng``) so that the
device path, the CPU oracle and the golden fixtures all consume the *same*
arrays.  Draw order follows SURVEY.md Appendix A; the ambiguities listed in
SURVEY.md Appendix B are resolved as recorded in DESIGN.md:

* C2 uses the *variance* reading of ``N(0, 1/sqrt(2000))`` (entries of A have
  unit variance), i.e. U, V entries have std ``k**-0.25``.
* C3 is BASELINE's Clement variant (rows 0 and n-1 are zero), not
  ``gallery.gen_clement`` (reference ``pkg/src/trisolve/gallery.py:64-71``).
* C4 is the h^2-scaled *upwind* 5-point operator with ``cx = h*Pe``,
  ``cy = 0.5*h*Pe`` (not the central-difference ``gallery.gen_convdiff``).
* C5 draws 10 *distinct* rows per column so ``nnz == 10 * n`` exactly.

Every generator takes its size parameters so tests can build scaled-down
instances of the same families.  Nothing here runs on the solve path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sparse


@dataclass
class Workload:
    name: str
    a: object          # np.ndarray (C-order fp64) or scipy.sparse.csr_array
    b: np.ndarray
    x_star: np.ndarray
    note: str = ""


def dense_gaussian(m: int = 1000, n: int = 1000, seed: int = 0) -> Workload:
    """C1: A i.i.d. N(0,1), x* ~ N(0,1), b = A x*."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    xs = rng.standard_normal(n)
    return Workload("c1_dense_gaussian", a, a @ xs, xs)


def dense_lowrank(m: int = 5000, n: int = 20000, k: int = 2000, seed: int = 0,
                  noise: float = 1e-3) -> Workload:
    """C2: A = U V^T (rank k), U,V i.i.d. N(0, k**-0.5) (variance reading),
    b = A x* + noise * N(0,1) (inconsistent)."""
    rng = np.random.default_rng(seed)
    s = float(k) ** -0.25
    u = rng.standard_normal((m, k)) * s
    v = rng.standard_normal((n, k)) * s
    a = np.ascontiguousarray(u @ v.T)
    del u, v
    xs = rng.standard_normal(n)
    b = a @ xs + noise * rng.standard_normal(m)
    return Workload("c2_dense_lowrank", a, b, xs)


def clement_variant(n: int = 100001, seed: int = 0) -> Workload:
    """C3: BASELINE's Clement variant, CSR, zero diagonal.

    ``A[i,i+1] = sqrt(i (n-1-i)) / scale`` and
    ``A[i+1,i] = sqrt((i+1) (n-2-i)) / scale`` with ``scale = n/2``; explicit
    zeros (row 0's super-diagonal and row n-1's sub-diagonal) are dropped.
    """
    rng = np.random.default_rng(seed)
    i = np.arange(n - 1, dtype=np.float64)
    scale = n / 2.0
    up = np.sqrt(i * (n - 1 - i)) / scale
    lo = np.sqrt((i + 1) * (n - 2 - i)) / scale
    a = sparse.diags_array([lo, up], offsets=[-1, 1], shape=(n, n), format="csr")
    a = sparse.csr_array(a)
    a.eliminate_zeros()
    a.sort_indices()
    a.indices = a.indices.astype(np.int32)
    a.indptr = a.indptr.astype(np.int32)
    xs = rng.standard_normal(n)
    return Workload("c3_clement", a, a @ xs, xs)


def convdiff_upwind(grid: int = 1000, pe: float = 50.0, seed: int = 0) -> Workload:
    """C4: 5-point upwind convection-diffusion on a grid x grid mesh,
    h^2-scaled, Dirichlet (stencil truncated at the boundary), k = ix + grid*iy."""
    rng = np.random.default_rng(seed)
    nn = grid * grid
    h = 1.0 / (grid + 1)
    cx = 1.0 * h * pe
    cy = 0.5 * h * pe
    k = np.arange(nn, dtype=np.int64)
    ix = k % grid
    iy = k // grid
    rows = [k]
    cols = [k]
    vals = [np.full(nn, 4.0 + cx + cy)]
    for ok, off, val in (
        (ix > 0, -1, -1.0 - cx),        # west
        (ix < grid - 1, 1, -1.0),       # east
        (iy > 0, -grid, -1.0 - cy),     # south
        (iy < grid - 1, grid, -1.0),    # north
    ):
        kk = k[ok]
        rows.append(kk)
        cols.append(kk + off)
        vals.append(np.full(kk.size, val))
    a = sparse.coo_array(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(nn, nn),
    ).tocsr()
    a.sort_indices()
    a.indices = a.indices.astype(np.int32)
    a.indptr = a.indptr.astype(np.int32)
    xs = rng.uniform(-1.0, 1.0, nn)
    return Workload("c4_convdiff_upwind", a, a @ xs, xs)


def lp_columns(m: int = 10_000, n: int = 1_000_000, per_col: int = 10,
               seed: int = 0) -> Workload:
    """C5: m x n, ``per_col`` distinct uniformly random rows per column,
    values U(0.1, 1.0); x* ~ U(0,1) >= 0, b = A x*."""
    if per_col > m:
        raise ValueError("per_col exceeds the row count")
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, m, size=(n, per_col))
    rows.sort(axis=1)
    while True:
        bad = np.nonzero(np.any(np.diff(rows, axis=1) == 0, axis=1))[0]
        if bad.size == 0:
            break
        redraw = rng.integers(0, m, size=(bad.size, per_col))
        redraw.sort(axis=1)
        rows[bad] = redraw
    vals = rng.uniform(0.1, 1.0, size=(n, per_col))
    indptr = np.arange(0, n * per_col + 1, per_col, dtype=np.int64)
    csc = sparse.csc_array((vals.ravel(), rows.ravel().astype(np.int32), indptr),
                           shape=(m, n))
    a = sparse.csr_array(csc.tocsr())
    a.sort_indices()
    a.indices = a.indices.astype(np.int32)
    a.indptr = a.indptr.astype(np.int32)
    xs = rng.uniform(0.0, 1.0, n)
    return Workload("c5_lp_columns", a, a @ xs, xs)


CONFIGS = {
    "c1": dense_gaussian,
    "c2": dense_lowrank,
    "c3": clement_variant,
    "c4": convdiff_upwind,
    "c5": lp_columns,
}


def make(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
