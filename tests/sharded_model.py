"""Host model of the column-sharded TA / CTA / TA-LP iterations (TEST-ONLY).

Each rank holds A[:, c0:c1] and its slice of x; m-vectors are replicated;
every A v is an all-reduce of the ranks' partial m-vectors and every n-space
reduction is an all-reduce of scalars — exactly the decomposition the device
path implements (csrc/ts_comm.cuh).  Used by tests/test_sharding_cpu.py with a
world-size-2 gloo group to check that the decomposition reproduces the
unsharded reference (oracle/port.py) — the host-side logic of the N > 1 path.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from oracle import port


def _ar(v):
    t = torch.as_tensor(np.atleast_1d(np.asarray(v, dtype=np.float64))).clone()
    dist.all_reduce(t)
    return t.numpy()


def _ar_min(v):
    t = torch.as_tensor(np.atleast_1d(np.asarray(v, dtype=np.float64))).clone()
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.numpy()[0])


def _mv(a_loc, v_loc):  # A v = sum_p A_p v_p
    return _ar(a_loc @ v_loc)


def _rmv(a_loc, r):  # local block of A^T r
    return np.asarray(r @ a_loc) if hasattr(a_loc, "tocsr") else a_loc.T @ r


def _nrm2_sharded(v_loc):
    return math.sqrt(float(_ar(float(np.dot(v_loc, v_loc)))[0]))


def ta_adaptive_sharded(a_loc, b, eps, max_iters, lp=False):
    """solve_adaptive (triangle.py:170-251) / nonnegative_feasibility
    (feasibility.py:59-140) with column-sharded A."""
    m = b.shape[0]
    n_loc = a_loc.shape[1]
    x = np.zeros(n_loc)
    bp = np.zeros(m)
    rho = 0.0
    events = []
    status = "inconclusive" if lp else "iteration_cap"
    it = 0
    while it < max_iters:
        gap = b - bp
        gn = float(np.linalg.norm(gap))
        if gn <= eps:
            status = "feasible" if lp else "approx_solution"
            break
        c = _rmv(a_loc, gap)
        cp = np.maximum(c, 0.0) if lp else c
        s = _ar([float(np.dot(c, c)), float(np.dot(cp, cp))])
        cn, cpn = math.sqrt(s[0]), math.sqrt(s[1])
        if lp and cpn == 0.0:
            status = "witness"
            events.append("witness")
            it += 1
            break
        if not lp and cn <= eps:
            status = "normal_eq_solution"
            break
        gb = float(np.dot(gap, b))
        piv_norm = cpn if lp else cn
        if rho > 0.0 and rho * piv_norm >= gb:
            pre = (rho / piv_norm) * cp
            v = _mv(a_loc, pre)
            d = v - bp
            al = min(1.0, max(0.0, float(np.dot(gap, d)) / float(np.dot(d, d))))
            bp = bp + al * d
            x = (1.0 - al) * x + al * pre
            if lp and _ar_min(x.min()) < -1e-12:
                status = "numerical_failure"
                break
            events.append("pivot")
        else:
            rho = max(2.0 * rho, gb / piv_norm)
            events.append("expand")
        it += 1
    fr = b - _mv(a_loc, x)
    return dict(status=status, iterations=it, x=x, events=events,
                residual_norm=float(np.linalg.norm(fr)),
                normal_residual_norm=_nrm2_sharded(_rmv(a_loc, fr)))


def cta_sharded(a_loc, b, epsilon, max_iters, t_max=5):
    """centering_solve (centering.py:263-358, Gram mode, no probe / accelerate)
    with column-sharded A: q_i local, p_i = all-reduce, phi replicated."""
    m = b.shape[0]
    x = np.zeros(a_loc.shape[1])
    r = b.copy()
    bn = float(np.linalg.norm(b))
    eps_abs = epsilon * bn
    sched = port.schedule(min(t_max, m))
    status, it = "iteration_cap", 0
    while it < max_iters:
        rn = float(np.linalg.norm(r))
        if rn <= eps_abs:
            status = "approx_solution"
            break
        t = next(sched)
        p, q = [r], []
        for _ in range(t):
            q.append(_rmv(a_loc, p[-1]))
            p.append(_mv(a_loc, q[-1]))
        phi = np.array([float(np.dot(p[k // 2], p[k - k // 2])) for k in range(1, 2 * t + 1)])
        if phi[1] == 0.0:
            status = "normal_eq_solution"
            break
        atr = _nrm2_sharded(q[0])
        pick = None
        for order in range(t, 0, -1):
            al = port.hankel_coeffs(phi, order)
            cand = r.copy()
            for i in range(order):
                cand -= al[i] * p[i + 1]
            cn = float(np.linalg.norm(cand))
            if pick is None or cn < pick[0]:
                pick = (cn, order, al, cand)
            if cn <= rn * (1.0 + 1e-13):
                pick = (cn, order, al, cand)
                break
        if atr * atr <= eps_abs * eps_abs:
            status = "normal_eq_solution"
            break
        _, order, al, r = pick
        for i in range(order):
            x = x + al[i] * q[i]
        it += 1
    fr = b - _mv(a_loc, x)
    return dict(status=status, iterations=it, x=x, residual_norm=float(np.linalg.norm(fr)),
                normal_residual_norm=_nrm2_sharded(_rmv(a_loc, fr)))


# ----------------------------------------------------------- row blocks ----
# Row-block sharding of a square matrix (RowShardedMatrix, k_halo): every
# vector is split like the rows; a pass reads its input through a halo of the
# band's half-width obtained from the neighbours; every dot / norm is a local
# sum all-reduced over ranks.

def _halo(v_loc, hw):
    """[left neighbour's tail | own block | right neighbour's head] (k_halo)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    parts = [None] * world
    dist.all_gather_object(parts, (v_loc[:hw].copy(), v_loc[len(v_loc) - hw:].copy()))
    left = parts[rank - 1][1] if rank > 0 else np.zeros(hw)
    right = parts[rank + 1][0] if rank + 1 < world else np.zeros(hw)
    return np.concatenate([left, v_loc, right])


def shifted_blocks(rows, cols, r0, hw):
    """Local CSR blocks whose indices address the halo-extended vector
    (global index j -> j - r0 + hw): the device's (j - r0) plus the offset of
    its halo padding."""
    import scipy.sparse as sp

    n_p = rows.shape[0]
    ext = n_p + 2 * hw
    shift = lambda blk: sp.csr_array((blk.data, blk.indices - r0 + hw, blk.indptr),  # noqa: E731
                                     shape=(n_p, ext))
    return shift(rows), shift(cols)


def _dot_rows(u, v):
    return float(_ar(float(np.dot(u, v)))[0])


def cta_row_sharded(rows_ext, cols_ext, hw, b_loc, epsilon, max_iters, t_max=5):
    """centering_solve (centering.py:263-358, Gram mode) on row blocks."""
    x = np.zeros(rows_ext.shape[0])
    r = b_loc.copy()
    bn = math.sqrt(_dot_rows(b_loc, b_loc))
    eps_abs = epsilon * bn
    m_glob = int(_ar(float(len(b_loc)))[0])
    sched = port.schedule(min(t_max, m_glob))
    status, it = "iteration_cap", 0
    while it < max_iters:
        rn = math.sqrt(_dot_rows(r, r))
        if rn <= eps_abs:
            status = "approx_solution"
            break
        t = next(sched)
        p, q = [r], []
        for _ in range(t):
            q.append(cols_ext @ _halo(p[-1], hw))   # A^T p: own columns, rows ascending
            p.append(rows_ext @ _halo(q[-1], hw))   # A q: own rows
        phi = np.array([_dot_rows(p[k // 2], p[k - k // 2]) for k in range(1, 2 * t + 1)])
        if phi[1] == 0.0:
            status = "normal_eq_solution"
            break
        atr = math.sqrt(_dot_rows(q[0], q[0]))
        pick = None
        for order in range(t, 0, -1):
            al = port.hankel_coeffs(phi, order)
            cand = r.copy()
            for i in range(order):
                cand -= al[i] * p[i + 1]
            cn = math.sqrt(_dot_rows(cand, cand))
            if pick is None or cn < pick[0]:
                pick = (cn, order, al, cand)
            if cn <= rn * (1.0 + 1e-13):
                pick = (cn, order, al, cand)
                break
        if atr * atr <= eps_abs * eps_abs:
            status = "normal_eq_solution"
            break
        _, order, al, r = pick
        for i in range(order):
            x = x + al[i] * q[i]
        it += 1
    fr = b_loc - rows_ext @ _halo(x, hw)
    atf = cols_ext @ _halo(fr, hw)
    return dict(status=status, iterations=it, x=x, residual_norm=math.sqrt(_dot_rows(fr, fr)),
                normal_residual_norm=math.sqrt(_dot_rows(atf, atf)))


# ------------------------------------------------------- tall row blocks ----
# Row-block sharding of a tall matrix (TallShardedMatrix): each rank holds
# A[r0:r1, :]; x-space vectors are replicated, b-space vectors split; A v is
# local, A^T r = sum_p A_p^T r_p is an all-reduce of n-vectors, every b-space
# dot / norm a scalar all-reduce, every x-space one local (replicated).

def _rmv_tall(a_loc, r_loc):
    return _ar(_rmv(a_loc, r_loc))


def cta_tall_sharded(a_loc, b_loc, epsilon, max_iters, t_max=5):
    """centering_solve (centering.py:263-358, Gram mode) on tall row blocks."""
    x = np.zeros(a_loc.shape[1])
    r = b_loc.copy()
    bn = math.sqrt(_dot_rows(b_loc, b_loc))
    eps_abs = epsilon * bn
    m_glob = int(_ar(float(len(b_loc)))[0])
    sched = port.schedule(min(t_max, m_glob))
    status, it = "iteration_cap", 0
    while it < max_iters:
        rn = math.sqrt(_dot_rows(r, r))
        if rn <= eps_abs:
            status = "approx_solution"
            break
        t = next(sched)
        p, q = [r], []
        for _ in range(t):
            q.append(_rmv_tall(a_loc, p[-1]))  # replicated n-vector
            p.append(a_loc @ q[-1])            # local rows
        phi = np.array([_dot_rows(p[k // 2], p[k - k // 2]) for k in range(1, 2 * t + 1)])
        if phi[1] == 0.0:
            status = "normal_eq_solution"
            break
        atr = float(np.linalg.norm(q[0]))
        pick = None
        for order in range(t, 0, -1):
            al = port.hankel_coeffs(phi, order)
            cand = r.copy()
            for i in range(order):
                cand -= al[i] * p[i + 1]
            cn = math.sqrt(_dot_rows(cand, cand))
            if pick is None or cn < pick[0]:
                pick = (cn, order, al, cand)
            if cn <= rn * (1.0 + 1e-13):
                pick = (cn, order, al, cand)
                break
        if atr * atr <= eps_abs * eps_abs:
            status = "normal_eq_solution"
            break
        _, order, al, r = pick
        for i in range(order):
            x = x + al[i] * q[i]
        it += 1
    fr = b_loc - a_loc @ x
    return dict(status=status, iterations=it, x=x, residual_norm=math.sqrt(_dot_rows(fr, fr)),
                normal_residual_norm=float(np.linalg.norm(_rmv_tall(a_loc, fr))))


def ta_tall_sharded(a_loc, b_loc, eps, max_iters):
    """solve_adaptive (triangle.py:170-251) on tall row blocks."""
    x = np.zeros(a_loc.shape[1])
    bp = np.zeros(len(b_loc))
    rho = 0.0
    events = []
    status, it = "iteration_cap", 0
    while it < max_iters:
        gap = b_loc - bp
        if math.sqrt(_dot_rows(gap, gap)) <= eps:
            status = "approx_solution"
            break
        c = _rmv_tall(a_loc, gap)
        cn = float(np.linalg.norm(c))
        if cn <= eps:
            status = "normal_eq_solution"
            break
        gb = _dot_rows(gap, b_loc)
        if rho > 0.0 and rho * cn >= gb:
            pre = (rho / cn) * c
            d = a_loc @ pre - bp
            al = min(1.0, max(0.0, _dot_rows(gap, d) / _dot_rows(d, d)))
            bp = bp + al * d
            x = (1.0 - al) * x + al * pre
            events.append("pivot")
        else:
            rho = max(2.0 * rho, gb / cn)
            events.append("expand")
        it += 1
    fr = b_loc - a_loc @ x
    return dict(status=status, iterations=it, x=x, events=events,
                residual_norm=math.sqrt(_dot_rows(fr, fr)))
