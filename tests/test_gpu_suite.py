"""The reference's own test suites, replayed through this package on the GPU.

``tests/golden/make_suite.py`` ran the reference's tests
(``pkg/tests/test_{linalg,centering,triangle,feasibility,hybrid,acceptance}.py``)
against the REAL reference with a recording layer in front of every public
function of the iteration path, and stored each top-level call (inputs,
outputs or raised exception, the test that made it, the reference's own x
spread for solver calls) in ``tests/golden/suite_calls.pkl.gz``.  Here every
recorded call is re-issued against this package's same-named function —
public API -> C ABI -> CUDA kernels — and compared:

* a call that raised in the reference must raise the same exception type
  with the same message (the reference's error contract);
* solver results (``SolveResult``) against the reference's OWN band on that
  call (recorded from re-runs with b * (1 + 1e-15 N(0,1))): status among the
  band's statuses; iteration count inside the band +-1 %; final residual
  norms within [lo / 2, 2 hi] of the band (north_star's factor of 2, floored
  at the cancellation level); x, rho, lower bound and min(x) within
  max(1e-9, 10 x the band's spread) (north_star's 1e-9 wherever the
  reference reproduces itself that well); where every re-run kept the
  recorded status, count and detail: the same detail, trace length and
  trace event sequence;
* operator results (matvec, norms, moments, pivot points, centering steps,
  the Hankel coefficients): 1e-12 relative to the scale of the operands
  (|A| |v| for products: dense BLAS and device reduction orders differ),
  booleans and integers exactly;
* side effects the tests assert on (``HOperator.apply_count``) equal.

One pytest case per reference test; a case fails on the first mismatching
call and reports which one.
"""

from __future__ import annotations

import gzip
import os
import pickle

import numpy as np
import pytest
import scipy.sparse as sparse

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

_PATH = os.path.join(GOLDEN, "suite_calls.pkl.gz")
if not os.path.exists(_PATH):  # regenerate with tests/golden/make_suite.py
    pytest.skip("suite_calls.pkl.gz not recorded", allow_module_level=True)
with gzip.open(_PATH, "rb") as _fh:
    _DATA = pickle.load(_fh)
RECORDS = _DATA["records"]
TESTS = sorted({r["test"] for r in RECORDS})
# calls of one reference test, in order
BY_TEST = {t: [r for r in RECORDS if r["test"] == t] for t in TESTS}


def _ours():
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import centering, feasibility, hybrid, linalg, triangle

    return {"trisolve.linalg": linalg, "trisolve.centering": centering, "trisolve.triangle": triangle,
            "trisolve.feasibility": feasibility, "trisolve.hybrid": hybrid, "ts": ts}


def revive(obj, mods):
    """Plain tagged tuples -> this package's classes."""
    if isinstance(obj, tuple) and obj and isinstance(obj[0], str):
        tag = obj[0]
        if tag == "GramProduct":
            return mods["trisolve.linalg"].GramProduct(revive(obj[1], mods))
        if tag == "HOperator":
            h = mods["trisolve.linalg"].HOperator(revive(obj[1], mods), obj[2])
            h.apply_count = obj[3]
            return h
        if tag == "CenteringOptions":
            return mods["trisolve.centering"].CenteringOptions(**revive(obj[1], mods))
        if tag == "HybridOptions":
            return mods["trisolve.hybrid"].HybridOptions(**revive(obj[1], mods))
        if tag == "CenteringState":
            d = revive(obj[1], mods)
            tr = d.pop("trace", None)
            st = mods["trisolve.centering"].CenteringState(**d)
            if isinstance(tr, tuple) and tr[0] == "Trace":
                st.trace.rows = list(tr[2])
            return st
        if tag == "Moments":
            return mods["trisolve.centering"].Moments(**revive(obj[1], mods))
    if isinstance(obj, list):
        return [revive(v, mods) for v in obj]
    if isinstance(obj, tuple):
        return tuple(revive(v, mods) for v in obj)
    if isinstance(obj, dict):
        return {k: revive(v, mods) for k, v in obj.items()}
    if isinstance(obj, np.ndarray):
        return obj.copy()
    if sparse.issparse(obj):
        return obj.copy()
    return obj


def _vec_close(got, want, rtol, what):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    if want.size == 0:
        return
    scale = max(float(np.abs(want).max()), 1e-300)
    err = float(np.abs(got - want).max())
    assert err <= rtol * scale or np.array_equal(got, want), (what, err / scale, rtol)


def _num_close(got, want, rtol, floor, what):
    if want is None:
        assert got is None, (what, got)
        return
    assert got is not None, (what, want)
    if isinstance(want, (bool, np.bool_)) or isinstance(want, (int, np.integer)) and not isinstance(want, bool):
        assert got == want, (what, got, want)
        return
    assert abs(float(got) - float(want)) <= rtol * abs(float(want)) + floor, (what, got, want)


def _trace_numeric(rows, columns):
    cols = [c for c in columns if c not in ("wall_ns",)]
    num, ev = [], []
    for row in rows:
        vals = []
        for c, v in zip(columns, row):
            if c == "wall_ns":
                continue
            if isinstance(v, str):
                ev.append(v)
                vals.append(0.0)
            else:
                vals.append(float(v))
        num.append(vals)
    return np.array(num, dtype=np.float64).reshape(len(rows), len(cols)), ev


def _tag(obj):
    return obj[0] if isinstance(obj, tuple) and obj and isinstance(obj[0], str) else None


def _dense(a):
    if _tag(a) == "GramProduct":
        a = a[1]
    if _tag(a) == "HOperator":
        a = a[1]
    return a.toarray() if sparse.issparse(a) else np.asarray(a, dtype=np.float64)


def _scale_vector(rec):
    """|A| |v| (or |A|^T |v|) of a recorded operator call: the scale its
    rounding error lives on."""
    fn = rec["fn"].rsplit(".", 1)[1]
    a0, v = rec["args"][0], np.asarray(rec["args"][1], dtype=np.float64)
    ad = np.abs(_dense(a0))
    if _tag(a0) == "GramProduct":
        return ad.T @ (ad @ np.abs(v))
    return ad.T @ np.abs(v) if fn == "matvec_transpose" else ad @ np.abs(v)


def _compare_outcome(got, w, rec, what, bn):
    """Bisections and staged solves (min_norm_solve, hybrid_solve): their
    inner iteration totals move by tens of percent in the reference itself
    under 1e-15 perturbations (test_gpu_parity OUTCOME cases), so they are
    held to their outcome: the stage statuses, and for a min-norm outcome the
    certified bracket (<= eps), ||x|| within 2 eps of the reference's and the
    residual within eps; a normal-equation outcome to its certified normal
    residual."""
    if w.get("stage_results"):
        assert [r.status for r in got.stage_results] == [s[1]["status"] for s in w["stage_results"]], what
    fn = what.rsplit(".", 1)[1]
    if got.status == "min_norm_solution":
        if fn == "min_norm_solve":
            eps = rec["args"][2] if len(rec["args"]) > 2 else rec["kwargs"]["eps"]
        else:
            opts = rec["args"][2][1] if len(rec["args"]) > 2 else rec["kwargs"]["options"][1]
            eps = max(opts["eps_ta"] * bn, 1.01 * got.stage_results[0].residual_norm)
        lo, hi = got.rho_interval
        assert hi - lo <= eps * (1 + 1e-9), (what, "bracket", hi - lo, eps)
        assert abs(np.linalg.norm(got.x) - np.linalg.norm(w["x"])) <= 2 * eps, (what, "||x||")
        assert got.residual_norm <= eps * (1 + 1e-9), (what, "residual", got.residual_norm, eps)
    elif w.get("normal_residual_norm") is not None:
        band = rec.get("band") or {}
        rlo, rhi = band.get("normal_residual_norm", [w["normal_residual_norm"]] * 2)
        assert got.normal_residual_norm <= 2.0 * rhi + 1e-10 * max(bn, 1.0), (what, "normal residual")


def _compare_solve(got, w, rec, what):
    band = rec.get("band") or {}
    tol = max(1e-9, 10.0 * float(band.get("x_spread", 0.0)))
    b = rec["args"][1] if len(rec["args"]) > 1 else None
    bn = float(np.linalg.norm(b)) if isinstance(b, np.ndarray) else 1.0
    floor = 1e-12 * max(bn, 1.0)
    statuses = band.get("statuses", [w["status"]])
    assert got.status in statuses, (what, got.status, statuses, got.detail, w["detail"])
    if what.rsplit(".", 1)[1] in ("min_norm_solve", "hybrid_solve") and not band.get("same_trace", True):
        _compare_outcome(got, w, rec, what, bn)
        return
    lo, hi = band.get("iterations", [w["iterations"]] * 2)
    assert int(np.floor(0.99 * lo)) <= got.iterations <= int(np.ceil(1.01 * hi)), \
        (what, "iterations", got.iterations, lo, hi)
    if got.status == w["status"]:
        x_ref = np.asarray(w["x"], dtype=np.float64)
        nx = max(float(np.linalg.norm(x_ref)), 1e-300)
        err = float(np.linalg.norm(np.asarray(got.x) - x_ref)) / nx
        assert err <= tol or float(np.linalg.norm(np.asarray(got.x) - x_ref)) <= floor, (what, "x", err, tol)
    for key in ("residual_norm", "normal_residual_norm"):
        if w.get(key) is not None:
            rlo, rhi = band.get(key, [w[key]] * 2)
            val = float(getattr(got, key))
            assert 0.5 * rlo - 1e2 * floor <= val <= 2.0 * rhi + 1e2 * floor, (what, key, val, rlo, rhi)
    for key in ("rho", "lower_bound", "min_x_entry"):
        if w.get(key) is not None and got.status == w["status"]:
            klo, khi = band.get(key, [w[key]] * 2)
            val = getattr(got, key)
            assert val is not None, (what, key)
            slack = tol * max(abs(klo), abs(khi)) + floor
            assert klo - slack <= float(val) <= khi + slack, (what, key, val, klo, khi)
    if band.get("same_trace", True):
        assert got.detail == w["detail"], (what, got.detail, w["detail"])
        if w.get("stage_results"):
            assert [r.status for r in got.stage_results] == [s[1]["status"] for s in w["stage_results"]]
        tr = w["trace"]
        if _tag(tr) == "Trace":
            assert len(got.trace.rows) == len(tr[2]), (what, len(got.trace.rows), len(tr[2]))
            _, ev_got = _trace_numeric(got.trace.rows, got.trace.columns)
            _, ev_ref = _trace_numeric(tr[2], tr[1])
            assert ev_got == ev_ref, (what, "trace events")
        if w.get("b_prime") is not None:
            _vec_close(got.b_prime, w["b_prime"], tol, (what, "b_prime"))


def compare_result(got, want, rec, mods):
    """Compare our return value with the recorded (plain) reference value."""
    what = rec["fn"]
    fn = what.rsplit(".", 1)[1]
    if _tag(want) == "SolveResult":
        _compare_solve(got, want[1], rec, what)
        return
    if fn in ("matvec", "matvec_transpose") and isinstance(want, np.ndarray):
        got = np.asarray(got, dtype=np.float64)
        assert got.shape == want.shape, (what, got.shape, want.shape)
        sc = _scale_vector(rec)
        assert np.all(np.abs(got - want) <= 1e-12 * sc + 1e-300), (what, float(np.max(np.abs(got - want) - 1e-12 * sc)))
        return
    if _tag(want) == "Moments":
        w = want[1]
        assert got.t == w["t"]
        _vec_close(got.phi, w["phi"], 1e-12, (what, "phi"))
        for k, (gk, wk) in enumerate(zip(got.krylov, w["krylov"])):
            _vec_close(gk, wk, 1e-12, (what, f"krylov {k}"))
        if w["transposed"] is not None:
            for k, (gk, wk) in enumerate(zip(got.transposed, w["transposed"])):
                _vec_close(gk, wk, 1e-12, (what, f"transposed {k}"))
        return
    if _tag(want) == "CenteringState":
        w = want[1]
        st_in = rec["args"][0][1]  # the state the step started from
        sx = max(float(np.abs(w["x"]).max(initial=0.0)), float(np.abs(st_in["x"]).max(initial=0.0)), 1e-300)
        sr = max(float(np.abs(w["r"]).max(initial=0.0)), float(np.abs(st_in["r"]).max(initial=0.0)), 1e-300)
        assert float(np.abs(np.asarray(got.x) - w["x"]).max(initial=0.0)) <= 1e-9 * max(sx, sr), (what, "x")
        assert float(np.abs(np.asarray(got.r) - w["r"]).max(initial=0.0)) <= 1e-9 * sr, (what, "r")
        assert got.iterations == w["iterations"]
        return
    if want is None:
        assert got is None, (what, got)
        return
    if isinstance(want, (bool, np.bool_)):
        assert bool(got) == bool(want), (what, got, want)
        return
    if isinstance(want, (int, np.integer)):
        assert int(got) == int(want), (what, got, want)
        return
    if isinstance(want, float):
        _num_close(got, want, 1e-12, 0.0, what)
        return
    if isinstance(want, np.ndarray):
        rtol = 1e-12
        if fn == "min_norm_coefficients":
            rtol = _hankel_rtol(rec)
        _vec_close(got, want, rtol, what)
        return
    if isinstance(want, tuple):
        assert isinstance(got, tuple) and len(got) == len(want), (what, got)
        for g_, w_ in zip(got, want):
            compare_result(g_, w_, dict(rec, band=None, fn=rec["fn"] + "[]"), mods)
        return
    raise AssertionError(f"{what}: cannot compare {type(want)}")


def _hankel_rtol(rec):
    """Both sides are backward-stable solves of the equilibrated Hankel system
    (LAPACK gelsd vs the device's Cholesky / Jacobi): agreement is bounded by
    eps * cond (as test_gpu_parity.test_moment_kats)."""
    mom = rec["args"][0]
    if _tag(mom) != "Moments":
        return 1e-8
    phi = np.asarray(mom[1]["phi"], dtype=np.float64)
    order = rec["args"][1] if len(rec["args"]) > 1 and rec["args"][1] is not None else \
        rec["kwargs"].get("order") or mom[1]["t"]
    idx = np.add.outer(np.arange(order), np.arange(order)) + 1
    hk = phi[idx]
    s = np.sqrt(np.abs(np.diag(hk)))
    s[s == 0] = 1.0
    sv = np.linalg.svd(hk / np.outer(s, s), compute_uv=False)
    kept = sv[sv > 1e-13 * sv[0]] if sv[0] > 0 else sv[:1]
    cond = sv[0] / kept[-1] if kept.size and kept[-1] > 0 else 1.0
    return max(1e-10, 50 * 2.2e-16 * cond)


def replay(rec, mods):
    modname, fname = rec["fn"].rsplit(".", 1)
    fn = getattr(mods[modname], fname)
    args = revive(rec["args"], mods)
    kwargs = revive(rec["kwargs"], mods)
    if "error" in rec:
        etype, emsg = rec["error"]
        with pytest.raises(Exception) as ei:
            fn(*args, **kwargs)
        got = type(ei.value).__name__
        assert got == etype or (etype == "LinAlgError" and got == "LinAlgError"), \
            (rec["fn"], got, etype, str(ei.value), emsg)
        assert str(ei.value) == emsg, (rec["fn"], str(ei.value), emsg)
        return
    got = fn(*args, **kwargs)
    compare_result(got, rec["result"], rec, mods)
    for a, post in zip(args, rec.get("post", [])):
        if _tag(post) == "HOperator":
            assert a.apply_count == post[3], (rec["fn"], "apply_count", a.apply_count, post[3])


@pytest.mark.parametrize("test", TESTS)
def test_reference_suite_call(test):
    mods = _ours()
    for k, rec in enumerate(BY_TEST[test]):
        try:
            replay(rec, mods)
        except AssertionError as e:
            raise AssertionError(f"{test}: call {k} {rec['fn']}: {e}") from None


def test_suite_fixture_is_complete():
    """The recording covered every suite and nothing was left unrepresentable."""
    assert _DATA["pytest_rc"] == 0
    assert not _DATA["skipped"]
    suites = {t.split("::")[0].rsplit("/", 1)[-1] for t in TESTS}
    assert suites == set(_DATA["suites"])
