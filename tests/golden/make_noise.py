"""Record the REFERENCE's own self-noise on every golden case.

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONPATH=/root/repo python tests/golden/make_noise.py

For each recorded case the real reference (``trisolve`` from
``/root/reference/pkg/src``) is re-run on the recorded inputs

* with b perturbed by 1e-15 relative (DRAWS seeded draws, one BLAS thread,
  plus the recorded unperturbed run),
* unperturbed with 8 OpenBLAS threads (the blocked dense reduction order
  changes with the thread count),

and the largest relative l2 distance of the final iterate from the recorded
one among the runs that reach the recorded status (``x_noise``; likewise the
largest trace deviation relative to each column's scale, ``trace_noise``; a boundary
case such as ball_inside flips between approx and witness under a 1e-15
perturbation), plus the spread of final residual norms, iteration counts and
statuses, is stored in ``self_noise.json``.  ``tests/test_gpu_parity.py`` holds
the device to ``max(1e-9, 10 x_noise)`` (iterates) and
``max(1e-9, 10 trace_noise)`` (trace rows) on every window case: north_star's
1e-9 where the reference reproduces itself that well, ten times the
reference's own spread where it does not (these replace round 1's hand-set
per-case tolerances).
"""

from __future__ import annotations

import json
import os
import sys

THREADS = int(os.environ.get("TS_NOISE_THREADS", "1"))  # the 8-thread pass runs in a child process
os.environ["OPENBLAS_NUM_THREADS"] = str(THREADS)
os.environ["OMP_NUM_THREADS"] = str(THREADS)

import subprocess  # noqa: E402

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from conftest import Golden, golden_names, trace_rows_numeric  # noqa: E402
from make_golden import _call  # noqa: E402  (imports the reference)

import trisolve  # noqa: E402

DRAWS = 8
SKIP = {"mn_underdetermined", "mn_bisection", "hy_min_norm", "hy_c2_lowrank",
        "mn_gram_operand"}  # OUTCOME cases


def _run(g, b):
    """The recorded call on (a, b); the recorded kwargs are already resolved."""
    if g.solver in ("mn", "mn_gramop"):
        op = trisolve.GramProduct(g.a) if g.solver == "mn_gramop" else g.a
        return trisolve.min_norm_solve(op, b, x_eps=g.x_eps, **g.kwargs)
    if g.solver == "ta_gram":  # _call would rescale the resolved eps a second time
        rhs = trisolve.linalg.matvec_transpose(g.a, b)
        return trisolve.solve_adaptive(trisolve.GramProduct(g.a), rhs, **g.kwargs)
    return _call(g.solver, g.a, b, dict(g.kwargs))[0]


def _rel(x, y):
    ny = float(np.linalg.norm(y))
    return float(np.linalg.norm(np.asarray(x) - y)) / (ny if ny > 0 else 1.0)


def _trace_dev(g, r):
    """Largest |trace - recorded| / max(|recorded|, column max) over the
    numeric trace entries (0 when the run's trace has another shape)."""
    if r.status != g.status or not g.trace.size:
        return 0.0
    try:
        tr = trace_rows_numeric(r.trace.rows, r.trace.columns)
    except ValueError:
        return 0.0
    if tr.shape != g.trace.shape:
        return 0.0
    colmax = np.abs(g.trace).max(axis=0)
    den = np.maximum(np.abs(g.trace), colmax)
    den[den == 0] = 1.0
    return float((np.abs(tr - g.trace) / den).max())


def _one(g, b):
    r = _run(g, b)
    return (_rel(r.x, g.x) if r.status == g.status else 0.0, float(r.residual_norm),
            int(r.iterations), r.status, _trace_dev(g, r))


def noise(name, threaded):
    g = Golden(name)
    rng = np.random.default_rng(4321)
    runs = [threaded[name]]
    for k in range(DRAWS + 1):  # k = 0: the recorded run itself (sanity)
        b = g.b if k == 0 else g.b * (1.0 + 1e-15 * rng.standard_normal(g.b.size))
        runs.append(_one(g, b))
    xs = [r[0] for r in runs]
    res = [r[1] for r in runs]
    its = [r[2] for r in runs]
    stats = {r[3] for r in runs}
    return {"x_noise": max(xs), "trace_noise": max(r[4] for r in runs), "residual_lo": min(res), "residual_hi": max(res),
            "iterations_lo": min(its), "iterations_hi": max(its), "statuses": sorted(stats),
            "runs": len(xs)}


def main():
    names = [n for n in golden_names() if n not in SKIP]
    if THREADS != 1:  # child: the unperturbed runs at this thread count, as JSON
        print(json.dumps({n: _one(Golden(n), Golden(n).b) for n in names}))
        return
    env = dict(os.environ, TS_NOISE_THREADS="8")
    threaded = json.loads(subprocess.run([sys.executable, os.path.abspath(__file__)], env=env,
                                         check=True, capture_output=True, text=True).stdout)
    out = {}
    for name in names:
        out[name] = noise(name, threaded)
        print(f"{name:24s} x_noise={out[name]['x_noise']:.2e} its={out[name]['iterations_lo']}.."
              f"{out[name]['iterations_hi']} {out[name]['statuses']}", flush=True)
    with open(os.path.join(HERE, "self_noise.json"), "w") as fh:
        json.dump({"how": "reference re-run with b * (1 + 1e-15 N(0,1)) (8 draws, 1 BLAS thread) "
                          "and unperturbed with 8 OpenBLAS threads; x_noise = max rel l2 of x from "
                          "the recorded run", "cases": out}, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
