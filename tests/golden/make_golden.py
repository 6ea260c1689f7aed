"""Record golden fixtures from the REAL reference implementation.

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONPATH=/root/repo python tests/golden/make_golden.py

It imports ``trisolve`` from ``/root/reference/pkg/src`` and, for every case in
``cases.py``, stores the inputs and the reference's outputs (status,
iterations, x, residual norms, extras, trace rows without ``wall_ns``) as
``tests/golden/<case>.npz``.  A second group records operator-layer and
moment-system known answers (``kat_*.npz``).  BLAS is pinned to one thread
so the recorded dense arithmetic is reproducible.
"""

from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np
import scipy.sparse as sparse

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import trisolve  # noqa: E402  (the reference)
from trisolve import centering, linalg  # noqa: E402

from cases import CASES  # noqa: E402

EVENT = {"pivot": 0, "expand": 1, "witness": 2}


def _store_matrix(d, a):
    if sparse.issparse(a):
        a = sparse.csr_array(a)
        d["a_kind"] = "csr"
        d["a_shape"] = np.array(a.shape, dtype=np.int64)
        d["a_indptr"] = a.indptr.astype(np.int64)
        d["a_indices"] = a.indices.astype(np.int32)
        d["a_data"] = a.data.astype(np.float64)
    else:
        d["a_kind"] = "dense"
        d["a"] = np.ascontiguousarray(a, dtype=np.float64)


def _call(solver, a, b, kw):
    kw = dict(kw)
    bn = linalg.norm2(b)
    if "eps_rel" in kw:
        kw["eps"] = kw.pop("eps_rel") * bn
    if solver == "cta":
        return trisolve.centering_solve(a, b, trisolve.CenteringOptions(**kw)), kw
    if solver == "ta":
        return trisolve.solve_adaptive(a, b, **kw), kw
    if solver == "ta_gram":
        g = linalg.matvec_transpose(a, b)
        kw["eps"] = kw["eps"] / bn * linalg.norm2(g)
        return trisolve.solve_adaptive(trisolve.GramProduct(a), g, **kw), kw
    if solver == "ball":
        if "rho_frac" in kw:
            xs = np.linalg.pinv(a) @ b
            kw["rho"] = kw.pop("rho_frac") * linalg.norm2(xs)
        return trisolve.solve_in_ball(a, b, **kw), kw
    if solver == "lp":
        return trisolve.nonnegative_feasibility(a, b, **kw), kw
    if solver == "hybrid":
        return trisolve.hybrid_solve(a, b, trisolve.HybridOptions(**kw)), kw
    if solver == "cta_gramop":
        return trisolve.centering_solve(trisolve.GramProduct(a), b, trisolve.CenteringOptions(**kw)), kw
    if solver == "hybrid_gramop":
        return trisolve.hybrid_solve(trisolve.GramProduct(a), b, trisolve.HybridOptions(**kw)), kw
    raise KeyError(solver)


def record_case(name, builder, solver, kw):
    built = builder()
    a, b = built[0], built[1]
    if solver in ("mn", "mn_gramop"):
        op = trisolve.GramProduct(a) if solver == "mn_gramop" else a
        res = trisolve.min_norm_solve(op, b, x_eps=built[2], **kw)
        resolved = dict(kw)
    else:
        res, resolved = _call(solver, a, b, kw)
    d = {}
    _store_matrix(d, a)
    d["b"] = np.asarray(b, dtype=np.float64)
    if len(built) > 2:
        d["x_eps"] = np.asarray(built[2], dtype=np.float64)
    if res.rho_interval is not None:
        d["rho_interval"] = np.asarray(res.rho_interval, dtype=np.float64)
    if res.stage_results:
        d["stage_status"] = np.array([r.status for r in res.stage_results])
        d["stage_iterations"] = np.array([r.iterations for r in res.stage_results])
    d["solver"] = solver
    d["kwargs"] = json.dumps(resolved)
    d["status"] = res.status
    d["detail"] = res.detail
    d["iterations"] = res.iterations
    d["x"] = np.asarray(res.x, dtype=np.float64)
    d["residual_norm"] = res.residual_norm
    d["normal_residual_norm"] = res.normal_residual_norm
    for key in ("rho", "lower_bound", "min_x_entry"):
        val = getattr(res, key)
        if val is not None:
            d[key] = float(val)
    if res.b_prime is not None:
        d["b_prime"] = np.asarray(res.b_prime, dtype=np.float64)
    cols = res.trace.columns
    rows = res.trace.rows
    d["trace_columns"] = np.array(cols)
    num = []
    for row in rows:
        vals = []
        for col, v in zip(cols, row):
            if col == "wall_ns":
                continue
            if col == "event":
                vals.append(float(EVENT.get(v, {"shrink": 3}.get(v, 4))))
            elif col == "stage":
                vals.append(1.0 if v == "stage1" else 2.0)
            else:
                vals.append(float(v))
        num.append(vals)
    d["trace"] = np.array(num, dtype=np.float64).reshape(len(rows), len(cols) - 1)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    return res


def record_kats():
    rng = np.random.default_rng(2024)
    # operator layer: dense + CSR, including empty rows/cols and a 1 x n row
    mats = []
    for (m, n, dens) in ((7, 5, 1.0), (30, 17, 0.3), (1, 300, 1.0), (200, 3, 0.5), (64, 64, 0.05)):
        dense = rng.standard_normal((m, n)) * (rng.random((m, n)) < dens)
        mats.append(dense)
    out = {}
    for i, dense in enumerate(mats):
        m, n = dense.shape
        v = rng.standard_normal(n)
        w = rng.standard_normal(m)
        csr = sparse.csr_array(dense)
        out[f"m{i}_dense"] = dense
        out[f"m{i}_v"] = v
        out[f"m{i}_w"] = w
        out[f"m{i}_mv_dense"] = linalg.matvec(dense, v)
        out[f"m{i}_rmv_dense"] = linalg.matvec_transpose(dense, w)
        out[f"m{i}_mv_csr"] = linalg.matvec(csr, v)
        out[f"m{i}_rmv_csr"] = linalg.matvec_transpose(csr, w)
        out[f"m{i}_norm_v"] = linalg.norm2(v)
        out[f"m{i}_fro"] = linalg.frobenius_norm(dense)
    out["count"] = len(mats)
    np.savez_compressed(os.path.join(HERE, "kat_linalg.npz"), **out)

    # moment systems: phi vectors from real CTA runs + synthetic rank-deficient ones
    phis, orders, alphas = [], [], []
    for seed in range(12):
        r2 = np.random.default_rng(seed)
        m = int(r2.integers(3, 12))
        a = r2.standard_normal((m, int(r2.integers(2, 12))))
        r = r2.standard_normal(m)
        t = int(min(5, m))
        h = linalg.HOperator(a, "aat")
        mom = centering.moments(h, r, t)
        for order in range(1, t + 1):
            phis.append(np.pad(mom.phi, (0, 10 - mom.phi.size)))
            orders.append((t, order))
            alphas.append(np.pad(centering.min_norm_coefficients(mom, order), (0, 5 - order)))
    for t in (1, 2, 3, 4, 5):  # identity operator: rank-one Hankel
        h = linalg.HOperator(np.eye(4), "a")
        mom = centering.moments(h, np.array([2.0, -1.0, 0.5, 1.0]), min(t, 4))
        for order in range(1, mom.t + 1):
            phis.append(np.pad(mom.phi, (0, 10 - mom.phi.size)))
            orders.append((mom.t, order))
            alphas.append(np.pad(centering.min_norm_coefficients(mom, order), (0, 5 - order)))
    np.savez_compressed(os.path.join(HERE, "kat_moments.npz"), phi=np.array(phis),
                        orders=np.array(orders, dtype=np.int64), alpha=np.array(alphas))


def main():
    only = set(sys.argv[1:])  # record just these cases (default: everything)
    if not only:
        record_kats()
    for name, builder, solver, kw in CASES:
        if only and name not in only:
            continue
        res = record_case(name, builder, solver, kw)
        print(f"{name:24s} {res.status:20s} iters={res.iterations:6d} "
              f"res={res.residual_norm:.3e} nres={res.normal_residual_norm:.3e}")


if __name__ == "__main__":
    main()
