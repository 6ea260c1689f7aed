"""Pin the CPU oracle (``oracle/port.py``) against fixtures recorded from the
real reference (``tests/golden/make_golden.py``).  CPU only."""

from __future__ import annotations

import os

import numpy as np
import pytest
import scipy.sparse as sparse

from conftest import GOLDEN, rel_l2
from oracle import port

pytestmark = pytest.mark.filterwarnings("ignore")


def run_oracle(g):
    kw = dict(g.kwargs)
    if g.solver == "cta":
        return port.cta_solve(g.a, g.b, **kw)
    if g.solver == "ta":
        return port.ta_adaptive(g.a, g.b, **kw)
    if g.solver == "ta_gram":
        return port.ta_adaptive(port.Gram(g.a), port.rmv(g.a, g.b), **kw)
    if g.solver == "ball":
        return port.ta_in_ball(g.a, g.b, **kw)
    if g.solver == "lp":
        return port.lp_feasibility(g.a, g.b, **kw)
    if g.solver == "mn":
        return port.min_norm_solve(g.a, g.b, x_eps=g.x_eps, **kw)
    if g.solver == "hybrid":
        return port.hybrid_solve(g.a, g.b, **kw)
    if g.solver == "cta_gramop":
        return port.cta_solve(port.Gram(g.a), g.b, **kw)
    if g.solver == "mn_gramop":
        return port.min_norm_solve(port.Gram(g.a), g.b, x_eps=g.x_eps, **kw)
    if g.solver == "hybrid_gramop":
        return port.hybrid_solve(port.Gram(g.a), g.b, **kw)
    raise KeyError(g.solver)


def test_oracle_matches_reference(golden):
    g = golden
    out = run_oracle(g)
    assert out["status"] == g.status
    assert out["detail"] == g.detail
    assert out["iterations"] == g.iterations
    # same numpy primitives in the same order: bit-for-bit, with a
    # last-ulp allowance only for BLAS kernel selection differences
    assert rel_l2(out["x"], g.x) <= 1e-14
    assert out["residual_norm"] == pytest.approx(g.residual_norm, rel=1e-12, abs=1e-300)
    if g.solver.startswith("hybrid"):  # merged trace is host bookkeeping; check the stages instead
        assert list(out["stage_status"]) == g.stage_status
        assert list(out["stage_iterations"]) == g.stage_iterations
        return
    if g.rho_interval is not None:
        np.testing.assert_allclose(out["rho_interval"], g.rho_interval, rtol=1e-12, atol=1e-300)
    tr = np.array([[float(v) if not isinstance(v, str) else
                    float(("pivot", "expand", "witness", "shrink").index(v)) for v in row]
                   for row in out["trace"]], dtype=np.float64).reshape(len(out["trace"]), g.trace.shape[1])
    assert tr.shape == g.trace.shape
    np.testing.assert_allclose(tr, g.trace, rtol=1e-12, atol=0)
    for key, val in g.extras.items():
        got = out[key]
        if isinstance(val, np.ndarray):
            assert rel_l2(got, val) <= 1e-13
        else:
            assert got == pytest.approx(val, rel=1e-12)


def test_operator_kats():
    z = np.load(os.path.join(GOLDEN, "kat_linalg.npz"))
    for i in range(int(z["count"])):
        dense = z[f"m{i}_dense"]
        csr = sparse.csr_array(dense)
        v, w = z[f"m{i}_v"], z[f"m{i}_w"]
        assert np.array_equal(port.mv(csr, v), z[f"m{i}_mv_csr"])
        assert np.array_equal(port.rmv(csr, w), z[f"m{i}_rmv_csr"])
        assert rel_l2(port.mv(dense, v), z[f"m{i}_mv_dense"]) <= 1e-15
        assert rel_l2(port.rmv(dense, w), z[f"m{i}_rmv_dense"]) <= 1e-15
        assert port.nrm(v) == pytest.approx(float(z[f"m{i}_norm_v"]), rel=1e-15)
        assert port.fro(dense) == pytest.approx(float(z[f"m{i}_fro"]), rel=1e-15)


def test_moment_kats():
    z = np.load(os.path.join(GOLDEN, "kat_moments.npz"))
    for phi, (t, order), alpha in zip(z["phi"], z["orders"], z["alpha"]):
        got = port.hankel_coeffs(phi[: 2 * t], int(order))
        np.testing.assert_allclose(got, alpha[:order], rtol=1e-12, atol=1e-14)


def test_schedule_wave():
    gen = port.schedule(5)
    assert [next(gen) for _ in range(12)] == [1, 2, 3, 4, 5, 4, 3, 2, 1, 2, 3, 4]
    gen = port.schedule(1)
    assert [next(gen) for _ in range(3)] == [1, 1, 1]


def test_chaotic_bands_cover_the_recorded_and_oracle_runs():
    """tests/golden/chaotic_bands.json (the reference's own spread under 1e-15
    input perturbations, recorded by make_bands.py) contains the recorded
    reference run, and the oracle lands inside the band the device tests use."""
    import json

    from conftest import Golden

    with open(os.path.join(GOLDEN, "chaotic_bands.json")) as fh:
        bands = {k: v["perturbation"] for k, v in json.load(fh).items()}
    assert set(bands) == {"cta_c1_cap", "ta_c1_500", "ta_c1_revalidate", "cta_c3_clement",
                          "ta_sparse_c3", "cta_c4_convdiff"}
    for name, bd in bands.items():
        g = Golden(name)
        assert bd["residual_lo"] <= g.residual_norm <= bd["residual_hi"]
        assert bd["iterations_lo"] <= g.iterations <= bd["iterations_hi"]
        if name in ("cta_c1_cap", "ta_c1_500", "ta_c1_revalidate"):
            continue  # dense: the oracle's BLAS order is the recorded one (checked above)
        out = run_oracle(g)
        assert 0.5 * bd["residual_lo"] <= out["residual_norm"] <= 2.0 * bd["residual_hi"]
        assert np.linalg.norm(out["x"] - g.x) <= 10 * bd["x_spread"] * np.linalg.norm(g.x)


def test_self_noise_table_covers_the_window_cases():
    """tests/golden/self_noise.json (make_noise.py) holds the reference's own
    x spread for every non-OUTCOME golden case, and the recorded run sits
    inside its recorded spread of statuses / iterations."""
    import json

    from conftest import Golden, golden_names

    with open(os.path.join(GOLDEN, "self_noise.json")) as fh:
        noise = json.load(fh)["cases"]
    outcome = {"mn_underdetermined", "mn_bisection", "hy_min_norm", "hy_c2_lowrank", "mn_gram_operand"}
    assert set(noise) == set(golden_names()) - outcome
    for name, nd in noise.items():
        g = Golden(name)
        assert g.status in nd["statuses"]
        assert nd["iterations_lo"] <= g.iterations <= nd["iterations_hi"]
        assert 0.0 <= nd["x_noise"] < 1e-2
