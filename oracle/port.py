"""numpy restatement of the reference TA / CTA / TA-LP loops (TEST INFRASTRUCTURE).

See ``oracle/__init__.py`` for the import rules.  Every function below names
the reference lines it restates (paths relative to
``/root/reference/pkg/src/trisolve/``).  The arithmetic deliberately goes
through the same numpy entry points the reference uses (``ndarray @``,
``csr @`` / ``v @ csr``, ``np.linalg.norm``, ``np.dot``, ``np.linalg.lstsq``)
so that, for a fixed BLAS thread count, results agree with the reference bit
for bit; ``tests/test_oracle_golden.py`` pins that against fixtures recorded
from the reference itself.

Results are returned as plain dicts (``status``, ``x``, ``iterations``,
``trace`` rows without ``wall_ns``, ...) so that the oracle has no dependency
on the product's result classes.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

APPROX = "approx_solution"
NORMAL_EQ = "normal_eq_solution"
MIN_NORM = "min_norm_solution"
WITNESS = "witness"
FEASIBLE = "feasible"
INCONCLUSIVE = "inconclusive"
CAP = "iteration_cap"
NUMFAIL = "numerical_failure"


# --------------------------------------------------------------------------
# operator layer — linalg.py:34-69
# --------------------------------------------------------------------------
def _is_op(a) -> bool:
    return (not isinstance(a, np.ndarray)) and (not sp.issparse(a)) and hasattr(a, "matvec")


def mv(a, v):
    """A @ v (linalg.py:34-42)."""
    v = np.asarray(v, dtype=np.float64)
    if _is_op(a):
        return a.matvec(v)
    if v.shape != (a.shape[1],):
        raise ValueError("matvec: length mismatch")
    return a @ v


def rmv(a, v):
    """A^T @ v from the same storage (linalg.py:45-56): dense strided view,
    sparse ``v @ csr`` (row-order scatter)."""
    v = np.asarray(v, dtype=np.float64)
    if _is_op(a):
        return a.rmatvec(v)
    if v.shape != (a.shape[0],):
        raise ValueError("matvec_transpose: length mismatch")
    if sp.issparse(a):
        return np.asarray(v @ a)
    return a.T @ v


def nrm(v) -> float:
    """linalg.py:59-61."""
    return float(np.linalg.norm(np.asarray(v, dtype=np.float64)))


def fro(a) -> float:
    """linalg.py:64-69."""
    if _is_op(a) and hasattr(a, "frobenius_norm"):
        return a.frobenius_norm()
    if sp.issparse(a):
        return float(np.sqrt((a.multiply(a)).sum()))
    return float(np.linalg.norm(np.asarray(a), "fro"))


class Gram:
    """Implicit A^T A applied as A^T (A v) (linalg.py:93-114)."""

    def __init__(self, a):
        self.a = a
        self.shape = (a.shape[1], a.shape[1])

    def matvec(self, v):
        return rmv(self.a, mv(self.a, v))

    rmatvec = matvec

    def frobenius_norm(self):
        return fro(self.a) ** 2


# --------------------------------------------------------------------------
# CTA — centering.py
# --------------------------------------------------------------------------
def krylov(a, r, t, gram=True):
    """Moments phi_1..phi_2t and the Krylov vectors (centering.py:67-84,
    HOperator.apply_with_transpose linalg.py:138-145)."""
    p = [np.asarray(r, dtype=np.float64)]
    q = [] if gram else None
    for _ in range(t):
        if gram:
            at = rmv(a, p[-1])
            p.append(mv(a, at))
            q.append(at)
        else:
            p.append(mv(a, p[-1]))
    phi = np.empty(2 * t)
    for k in range(1, 2 * t + 1):
        lo = k // 2
        phi[k - 1] = float(np.dot(p[lo], p[k - lo]))
    return phi, p, q


def hankel_coeffs(phi, order, rcond=1e-13):
    """Equilibrated min-norm Hankel solve (centering.py:87-110)."""
    idx = np.add.outer(np.arange(order), np.arange(order)) + 1
    hk = np.asarray(phi, dtype=np.float64)[idx]
    s = np.sqrt(np.abs(np.diag(hk)))
    s[s == 0.0] = 1.0
    beta = np.linalg.lstsq(hk / np.outer(s, s), np.asarray(phi[:order]) / s, rcond=rcond)[0]
    return beta / s


class _NE(Exception):
    pass


def cta_step(x, r, t, a, gram=True, rcond=1e-13):
    """One order-t step with monotone retry (centering.py:172-213, without
    the optional probe).  Returns (x_new, r_new, order, atr_norm)."""
    phi, p, q = krylov(a, r, t, gram)
    if phi[1] == 0.0:
        raise _NE
    atr_norm = nrm(q[0]) if gram else nrm(p[1])
    r_norm = nrm(r)
    pick = None
    for order in range(t, 0, -1):
        al = hankel_coeffs(phi, order, rcond)
        cand = r.copy()
        for i in range(order):
            cand -= al[i] * p[i + 1]
        cn = nrm(cand)
        if pick is None or cn < pick[0]:
            pick = (cn, order, al, cand)
        if cn <= r_norm * (1.0 + 1e-13):
            pick = (cn, order, al, cand)
            break
    _, order, al, r_new = pick
    dirs = q if gram else p
    x_new = x.copy()
    for i in range(order):
        x_new += al[i] * dirs[i]
    return x_new, r_new, order, atr_norm, (phi, p, q)


def _probe(x, r, a, gram, j_max, thr, hr, atr):
    """first_order_probe (centering.py:227-251)."""
    y = np.asarray(r, dtype=np.float64)
    xh = np.asarray(x, dtype=np.float64).copy()
    for j in range(1, j_max):
        f1 = float(np.dot(y, hr))
        f2 = float(np.dot(hr, hr))
        if f2 == 0.0:
            return None
        al = f1 / f2
        xh += al * (atr if gram else y)
        y = y - al * hr
        if gram:
            atr = rmv(a, y)
            hr = mv(a, atr)
        else:
            hr = mv(a, y)
            atr = None
        if abs(float(np.dot(y, hr))) <= thr:
            return xh, j
    return None


def schedule(t_max):
    """Triangle wave 1..t_max..2 (centering.py:254-260)."""
    if t_max == 1:
        while True:
            yield 1
    wave = list(range(1, t_max + 1)) + list(range(t_max - 1, 1, -1))
    while True:
        yield from wave


def cta_solve(a, b, epsilon=1e-15, t_max=5, max_iters=100_000, h_mode="aat",
              enhanced=False, known_solvable=False, recheck_every=250,
              start="zero", start_seed=0, rcond=1e-13, accelerate=False,
              accel_ratio=0.95, accel_patience=3):
    """centering_solve (centering.py:263-358)."""
    m, n = a.shape
    if not 0.0 < epsilon < 1.0:
        raise ValueError("epsilon must lie in (0, 1)")
    if t_max < 1:
        raise ValueError("t_max must be at least 1")
    if h_mode not in ("a", "aat"):
        raise ValueError("unknown h_mode")
    t_max = min(t_max, m)
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (m,):
        raise ValueError("b has wrong shape")
    gram = h_mode == "aat"
    bn = nrm(b)
    out = dict(trace=[], detail="")
    if bn == 0.0:
        out.update(status=APPROX, x=np.zeros(n), residual_norm=0.0,
                   normal_residual_norm=0.0, iterations=0)
        return out
    if start == "random":
        x = np.random.default_rng(start_seed).standard_normal(n)
        r = b - mv(a, x)
    else:
        x = np.zeros(n)
        r = b.copy()
    eps_abs = epsilon * bn
    quad = eps_abs * eps_abs
    afro = fro(a)
    sched = schedule(t_max)
    status, detail, it, slow = CAP, "", 0, 0
    while it < max_iters:
        rn = nrm(r)
        if not np.isfinite(rn):
            status, detail = NUMFAIL, "non-finite residual"
            break
        if rn <= eps_abs:
            status = APPROX
            break
        t = next(sched)
        try:
            x_new, r_new, _, atrn, (phi, p, q) = cta_step(x, r, t, a, gram, rcond)
        except _NE:
            status = NORMAL_EQ
            break
        except np.linalg.LinAlgError as exc:
            status, detail = NUMFAIL, f"moment solve failed: {exc}"
            break
        prb = None
        if enhanced and not known_solvable and t >= 2:
            prb = _probe(x, r, a, gram, t, quad, p[1], q[0] if gram else None)
        out["trace"].append((it, t, rn, atrn))
        if not known_solvable and atrn * atrn <= quad:
            status = NORMAL_EQ
            detail = f"certified ||A^T A x - A^T b|| <= {eps_abs:.3e}"
            break
        if accelerate:
            ratio = nrm(r_new) / rn if rn > 0 else 0.0
            slow = slow + 1 if ratio > accel_ratio else 0
            if slow >= accel_patience:
                w = ratio / (1.0 + ratio)
                x_new = w * x + (1.0 - w) * x_new
                r_new = w * r + (1.0 - w) * r_new
                slow = 0
        x, r = x_new, r_new
        it += 1
        if prb is not None:
            xh, _ = prb
            if nrm(rmv(a, b - mv(a, xh))) < nrm(rmv(a, b - mv(a, x))):
                x = xh
                r = b - mv(a, x)
            status = NORMAL_EQ
            break
        if recheck_every and it % recheck_every == 0:
            fresh = b - mv(a, x)
            drift = nrm(fresh - r)
            if drift > 1e-10 * (bn + afro * nrm(x)):
                status, detail = NUMFAIL, "residual drift exceeded budget"
                r = fresh
                break
            r = fresh
    fr = b - mv(a, x)
    out.update(status=status, detail=detail, x=x, iterations=it,
               residual_norm=nrm(fr), normal_residual_norm=nrm(rmv(a, fr)))
    return out


# --------------------------------------------------------------------------
# TA — triangle.py
# --------------------------------------------------------------------------
def _segment_step(bp, xp, v, pre, b):
    """move_to_pivot (triangle.py:69-81)."""
    d = np.asarray(v) - np.asarray(bp)
    dd = float(np.dot(d, d))
    if dd == 0.0:
        raise ValueError("degenerate pivot: v coincides with the iterate")
    al = float(np.dot(np.asarray(b) - bp, d)) / dd
    al = min(1.0, max(0.0, al))
    return bp + al * d, (1.0 - al) * xp + al * pre, al


def _finish(out, a, b, x):
    """_result (triangle.py:84-89)."""
    fr = np.asarray(b) - mv(a, x)
    out.update(x=x, residual_norm=nrm(fr), normal_residual_norm=nrm(rmv(a, fr)))
    return out


def ta_adaptive(a, b, eps, eps_prime=None, rho_cap=None, max_iters=100_000,
                x0=None, restart_halvings=0):
    """solve_adaptive (triangle.py:170-251)."""
    m, n = a.shape
    b = np.asarray(b, dtype=np.float64)
    if nrm(b) == 0.0:
        return dict(status=APPROX, x=np.zeros(n), residual_norm=0.0,
                    normal_residual_norm=0.0, iterations=0, trace=[], rho=0.0, detail="")
    if eps_prime is None:
        eps_prime = eps
    if rho_cap is None:
        rho_cap = 4.0 * nrm(b) ** 2 / eps_prime
    if x0 is not None:
        x = np.asarray(x0, dtype=np.float64).copy()
        bp = mv(a, x)
        rho = nrm(x)
    else:
        x, bp, rho = np.zeros(n), np.zeros(m), 0.0
    trace = []
    status, detail, it, since, halv = CAP, "", 0, 0, max(0, restart_halvings)
    while it < max_iters:
        gap = b - bp
        gn = nrm(gap)
        if not math.isfinite(gn):
            status, detail = NUMFAIL, "non-finite iterate"
            break
        if gn <= eps:
            status = APPROX
            break
        c = rmv(a, gap)
        cn = nrm(c)
        if cn <= eps_prime:
            if cn > 0.0 and halv > 0:
                halv -= 1
                eps_prime *= 0.5
                continue
            status = NORMAL_EQ
            detail = ("pivot direction vanished" if cn == 0.0
                      else f"certified ||A^T(b - Ax)|| <= {eps_prime:.3e}")
            break
        gb = float(np.dot(gap, b))
        if rho > 0.0 and rho * cn >= gb:
            pre = (rho / cn) * c
            bp, x, _ = _segment_step(bp, x, mv(a, pre), pre, b)
            trace.append((it, rho, gn, cn, "pivot"))
            since += 1
            if since >= 512:
                bp = mv(a, x)
                since = 0
        else:
            rho = max(2.0 * rho, gb / cn)
            trace.append((it, rho, gn, cn, "expand"))
            if rho > rho_cap:
                status, detail = CAP, f"radius exceeded cap {rho_cap:.3e}"
                it += 1
                break
        it += 1
    out = dict(status=status, detail=detail, iterations=it, trace=trace, rho=rho)
    return _finish(out, a, b, x)


def ta_in_ball(a, b, rho, eps, eps_prime=None, max_iters=100_000, x0=None):
    """solve_in_ball + _membership_loop (triangle.py:92-167)."""
    m, n = a.shape
    b = np.asarray(b, dtype=np.float64)
    if nrm(b) == 0.0:
        raise ValueError("b must be nonzero")
    if rho <= 0.0:
        raise ValueError("rho must be positive")
    if eps_prime is None:
        eps_prime = eps
    if x0 is not None and nrm(x0) <= rho * (1.0 + 1e-9):
        x = np.asarray(x0, dtype=np.float64).copy()
        bp = mv(a, x)
    else:
        x, bp = np.zeros(n), np.zeros(m)
    trace = []
    wb = None
    status, it, since = CAP, 0, 0
    while it < max_iters:
        gap = b - bp
        gn = nrm(gap)
        if not math.isfinite(gn):
            status = NUMFAIL
            break
        if gn <= eps:
            status = APPROX
            break
        c = rmv(a, gap)
        cn = nrm(c)
        if cn <= eps_prime:
            status = NORMAL_EQ
            break
        gb = float(np.dot(gap, b))
        if rho * cn >= gb:
            pre = (rho / cn) * c
            bp, x, _ = _segment_step(bp, x, mv(a, pre), pre, b)
            trace.append((it, rho, gn, cn, "pivot"))
            since += 1
            if since >= 512:
                bp = mv(a, x)
                since = 0
        else:
            wb = gb / cn
            trace.append((it, rho, gn, cn, "witness"))
            status = WITNESS
            it += 1
            break
        it += 1
    out = dict(status=status, detail="", iterations=it, trace=trace, rho=rho, b_prime=bp)
    if status == WITNESS:
        out["lower_bound"] = wb
    return _finish(out, a, b, x)


# --------------------------------------------------------------------------
# TA-LP — feasibility.py
# --------------------------------------------------------------------------
def default_rho_max(a, b):
    """feasibility.py:49-56."""
    m, n = a.shape
    sigma = fro(a) / math.sqrt(m)
    if sigma == 0.0:
        sigma = 1.0
    return 10.0 * n * max(1.0, nrm(b) / sigma)


def lp_feasibility(a, b, eps, rho_max=None, max_iters=100_000):
    """nonnegative_feasibility (feasibility.py:59-140)."""
    m, n = a.shape
    b = np.asarray(b, dtype=np.float64)
    if nrm(b) == 0.0:
        raise ValueError("b must be nonzero")
    if rho_max is None:
        rho_max = default_rho_max(a, b)
    if rho_max <= 0.0:
        raise ValueError("rho_max must be positive")
    x, bp, rho = np.zeros(n), np.zeros(m), 0.0
    trace = []
    status, detail, lb, it, since = INCONCLUSIVE, "iteration budget exhausted", None, 0, 0
    while it < max_iters:
        gap = b - bp
        gn = nrm(gap)
        if not math.isfinite(gn):
            status, detail = NUMFAIL, "non-finite iterate"
            break
        if gn <= eps:
            status, detail = FEASIBLE, ""
            break
        c = rmv(a, gap)
        cp = np.maximum(c, 0.0)
        cpn = nrm(cp)
        if cpn == 0.0:
            status = WITNESS
            cn = nrm(c)
            lb = float(np.dot(gap, b)) / cn if cn > 0.0 else math.inf
            detail = "no ascent direction in the nonnegative cone section"
            trace.append((it, rho, gn, cn, "witness", float(x.min()) if n else 0.0))
            it += 1
            break
        gb = float(np.dot(gap, b))
        if rho > 0.0 and rho * cpn >= gb:
            pre = (rho / cpn) * cp
            bp, x, _ = _segment_step(bp, x, mv(a, pre), pre, b)
            xmin = float(x.min())
            if xmin < -1e-12:
                status, detail = NUMFAIL, "iterate left the nonnegative cone"
                break
            trace.append((it, rho, gn, nrm(c), "pivot", xmin))
            since += 1
            if since >= 512:
                bp = mv(a, x)
                since = 0
        else:
            rho = max(2.0 * rho, gb / cpn)
            trace.append((it, rho, gn, nrm(c), "expand", float(x.min())))
            if rho > rho_max:
                status, detail = INCONCLUSIVE, f"radius budget {rho_max:.3e} exhausted"
                it += 1
                break
        it += 1
    fr = b - mv(a, x)
    return dict(status=status, detail=detail, x=x, iterations=it, trace=trace, rho=rho,
                lower_bound=lb, min_x_entry=float(x.min()) if n else 0.0,
                residual_norm=nrm(fr), normal_residual_norm=nrm(rmv(a, fr)))


# --------------------------------------------------------------------------
# next rows: min-norm bisection (triangle.py:254-330) and hybrid (hybrid.py)
# --------------------------------------------------------------------------
def min_norm_solve(a, b, eps, x_eps, inner_cap=250_000, max_iters=4_000_000):
    """min_norm_solve (triangle.py:254-330); the outer trace rows carry the
    bracket events 'shrink' / 'expand'."""
    b = np.asarray(b, dtype=np.float64)
    if nrm(b) == 0.0:
        raise ValueError("b must be nonzero")
    x_eps = np.asarray(x_eps, dtype=np.float64)
    start_gap = nrm(b - mv(a, x_eps))
    if start_gap > eps * (1.0 + 1e-9):
        raise ValueError("x_eps is not an eps-approximate solution")
    floor = 1e-14 * fro(a) * nrm(b)
    hi, lo = nrm(x_eps), 0.0
    best = x_eps.copy()
    warm = None
    trace, it, status, detail = [], 0, MIN_NORM, ""
    budget = max(8, int(math.ceil(math.log2(max(hi / eps, 2.0)))) + 8)
    for _ in range(budget):
        if hi - lo <= eps or it >= max_iters:
            break
        rho = 0.5 * (hi + lo)
        if rho <= 0.0:
            break
        inner = ta_in_ball(a, b, rho, 0.25 * eps, eps_prime=floor,
                           max_iters=min(inner_cap, max_iters - it), x0=warm)
        for row in inner["trace"]:
            trace.append((it + row[0],) + tuple(row[1:]))
        it += inner["iterations"]
        gap = nrm(b - inner["b_prime"])
        if inner["status"] == APPROX:
            best = inner["x"]
            hi = min(rho, nrm(inner["x"]))
            warm = inner["x"]
            trace.append((it, hi, gap, 0.0, "shrink"))
        elif inner["status"] == WITNESS:
            lo = min(max(lo, inner["lower_bound"]), hi)
            warm = inner["x"]
            trace.append((it, lo, gap, 0.0, "expand"))
        elif inner["status"] == NORMAL_EQ:
            out = dict(status=NORMAL_EQ, iterations=it, trace=trace, rho=rho,
                       rho_interval=(lo, hi), detail="pivot direction vanished during bisection")
            return _finish(out, a, b, inner["x"])
        else:
            status = inner["status"]
            detail = ("inner membership test exhausted its budget" if status == CAP
                      else "non-finite iterate")
            break
    if status == MIN_NORM and hi - lo > eps:
        status, detail = CAP, "bisection budget exhausted"
    out = dict(status=status, iterations=it, trace=trace, rho=hi, rho_interval=(lo, hi),
               detail=detail)
    return _finish(out, a, b, best)


def hybrid_solve(a, b, eps_cta=1e-8, eps_ta=1e-15, want_min_norm=False, t_max=5, h_mode="aat",
                 max_iters_stage1=100_000, max_iters_stage2=400_000, min_norm_inner_cap=250_000):
    """hybrid_solve (hybrid.py:59-111)."""
    b = np.asarray(b, dtype=np.float64)
    bn = nrm(b)
    n = a.shape[1]
    if bn == 0.0:
        return dict(status=APPROX, x=np.zeros(n), residual_norm=0.0, normal_residual_norm=0.0,
                    iterations=0, trace=[], detail="")
    s1 = cta_solve(a, b, epsilon=eps_cta, t_max=t_max, h_mode=h_mode, max_iters=max_iters_stage1)
    if s1["status"] == APPROX and want_min_norm:
        eps2 = max(eps_ta * bn, 1.01 * s1["residual_norm"])
        s2 = min_norm_solve(a, b, eps2, s1["x"], inner_cap=min_norm_inner_cap,
                            max_iters=max_iters_stage2)
        status, x = s2["status"], s2["x"]
    elif s1["status"] == APPROX:
        s2 = ta_adaptive(a, b, eps=eps_ta * bn, max_iters=max_iters_stage2, x0=s1["x"])
        status = s2["status"]
        x = s2["x"] if s2["residual_norm"] <= s1["residual_norm"] else s1["x"]
    else:
        g = rmv(a, b)
        s2 = ta_adaptive(Gram(a), g, eps=eps_ta * nrm(g), max_iters=max_iters_stage2, x0=s1["x"])
        x = s2["x"] if s2["normal_residual_norm"] <= s1["normal_residual_norm"] else s1["x"]
        status = NORMAL_EQ if s2["status"] == APPROX else s2["status"]
    fr = b - mv(a, x)
    return dict(status=status, x=x, residual_norm=nrm(fr), normal_residual_norm=nrm(rmv(a, fr)),
                iterations=s1["iterations"] + s2["iterations"], detail=s2.get("detail", ""),
                trace=[], stage_status=(s1["status"], s2["status"]),
                stage_iterations=(s1["iterations"], s2["iterations"]))
