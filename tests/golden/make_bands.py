"""Record the REFERENCE's own reproducibility band for the chaotic golden cases.

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONPATH=/root/repo python tests/golden/make_bands.py

The chaotic cases (ill-conditioned runs far past the ~50-iteration parity
window) reach an outcome that depends on rounding: the
reference itself lands elsewhere when only the last bit of its input moves.
For each such case this script re-runs the real reference (``trisolve`` from
``/root/reference/pkg/src``, one BLAS thread) on the recorded inputs and
records two bands separately:

* ``perturbation``: b perturbed by 1e-15 relative (PERT_DRAWS seeded draws
  plus the unperturbed run), the reference's code unchanged — the band the
  device is held to;
* ``solver_swap``: for the CTA cases, the same perturbations with the moment
  system's least-squares call
(``np.linalg.lstsq`` at centering.py:109) swapped for mathematically
equivalent solvers of the same equilibrated system (SVD or symmetric-eigen
pseudo-inverse with the same rcond cut, Cholesky, LU): an ill-conditioned
run's outcome moves with the last bits of that solve (cta_c4_convdiff: 237
iterations with gelsd, 205 with numpy's SVD, 193 and a normal-equation stop
with eigh) — recorded for reference only.

Each band stores the range of final residual norms and iteration counts, the
statuses, and the largest rel l2 distance of x from the recorded run.
``tests/test_gpu_parity.py`` accepts a device run whose status is among the
perturbation band's, whose residual lies inside [lo / 2, 2 hi] of it
(north_star's factor of 2 on the reference's own spread), whose iteration
count lies inside it widened by +-1 %, and whose x is no farther from the
recorded x than 10 x the band's x spread.
"""

from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np
import scipy.linalg

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from conftest import Golden  # noqa: E402
from make_golden import _call  # noqa: E402  (imports the reference)

CHAOTIC = ("cta_c1_cap", "ta_c1_500", "ta_c1_revalidate", "cta_c3_clement", "ta_sparse_c3",
           "cta_c4_convdiff")
PERT_DRAWS = 200
SWAP_DRAWS = 24
_LSTSQ = np.linalg.lstsq


def _alt_lstsq(kind):
    """np.linalg.lstsq stand-in for a square symmetric system, same cut rule."""

    def solve(a, b, rcond=None):
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        cut = (rcond if rcond is not None else 1e-15)
        if kind == "svd":
            u, sv, vt = np.linalg.svd(a)
            keep = sv > cut * sv[0]
            x = vt[keep].T @ ((u[:, keep].T @ b) / sv[keep])
        elif kind == "eigh":
            w, v = np.linalg.eigh(a)
            keep = np.abs(w) > cut * np.abs(w).max()
            x = v[:, keep] @ ((v[:, keep].T @ b) / w[keep])
        elif kind == "chol":
            try:
                x = scipy.linalg.cho_solve(scipy.linalg.cho_factor(a, lower=True), b)
            except np.linalg.LinAlgError:
                return _LSTSQ(a, b, rcond=rcond)
        else:  # "lu"
            x = np.linalg.solve(a, b)
        return x, None, None, None

    return solve


def _spread(g, kinds, draws):
    res, its, xs, statuses = [], [], [], set()
    nx = float(np.linalg.norm(g.x)) or 1.0
    for kind in kinds:
        rng = np.random.default_rng(1234)
        np.linalg.lstsq = _LSTSQ if kind is None else _alt_lstsq(kind)
        try:
            for k in range(draws + 1):
                b = g.b if k == 0 else g.b * (1.0 + 1e-15 * rng.standard_normal(g.b.size))
                # the recorded kwargs are already resolved (absolute eps etc.)
                r, _ = _call(g.solver, g.a, b, dict(g.kwargs))
                res.append(float(r.residual_norm))
                its.append(int(r.iterations))
                xs.append(float(np.linalg.norm(np.asarray(r.x) - g.x)) / nx)
                statuses.add(r.status)
        finally:
            np.linalg.lstsq = _LSTSQ
    return {"residual_lo": min(res), "residual_hi": max(res), "iterations_lo": min(its),
            "iterations_hi": max(its), "statuses": sorted(statuses), "runs": len(res),
            "x_spread": max(xs)}


def band(name):
    g = Golden(name)
    out = {"perturbation": dict(_spread(g, [None], PERT_DRAWS),
                                how="b * (1 + 1e-15 N(0,1)), reference code unchanged")}
    if g.solver == "cta":
        out["solver_swap"] = dict(_spread(g, ["svd", "eigh", "chol", "lu"], SWAP_DRAWS),
                                  how="as perturbation, moment solve by svd / eigh / cholesky / lu "
                                      "instead of lstsq (recorded, not asserted)")
    return out


def main():
    out = {name: band(name) for name in CHAOTIC}
    with open(os.path.join(HERE, "chaotic_bands.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    for k, v in out.items():
        print(k, v)


if __name__ == "__main__":
    main()
