"""Golden parity cases: inputs + call recipes shared by the fixture generator
(``make_golden.py``, runs the real reference here) and the tests (which read
the recorded inputs back from the fixture, so nothing is regenerated on the
GPU box).

Each case is ``(name, builder, solver, kwargs)``; ``builder()`` returns
``(a, b)`` where ``a`` is a dense C-order ndarray or a ``csr_array``.
Solver names: ``cta`` (centering_solve), ``ta`` (solve_adaptive),
``ball`` (solve_in_ball), ``lp`` (nonnegative_feasibility),
``ta_gram`` (solve_adaptive on GramProduct(a) with rhs A^T b).
Tolerances that the reference CLI scales by ||b|| (cli.py:207-210) are
given as ``eps_rel`` and converted with the reference's own norm.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sparse

from paper_2304_12168_b200 import workloads as W


def _diag(d):
    return np.diag(np.asarray(d, dtype=np.float64))


def _poisson2d(k):
    t = sparse.diags_array([-np.ones(k - 1), 2 * np.ones(k), -np.ones(k - 1)], offsets=[-1, 0, 1])
    i = sparse.eye_array(k)
    return (sparse.kron(t, i) + sparse.kron(i, t)).toarray()


def _rand_feasible_lp(seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((5, 14))
    return a, a @ rng.uniform(0.2, 1.0, 14)


def _inball(seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((5, 11))
    b = a @ rng.standard_normal(11)
    return a, b


def _probe_case(seed):
    # inconsistent systems on which the enhanced first-order probe triggers
    rng = np.random.default_rng(seed)
    m = int(rng.integers(10, 40))
    n = int(rng.integers(3, m))
    return rng.standard_normal((m, n)), rng.standard_normal(m)


def _mn_under(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(2, 6))
    n = int(rng.integers(m + 1, 12))
    a = rng.standard_normal((m, n))
    x0 = rng.standard_normal(n)
    return a, a @ x0, x0


def _c(w):
    return (w.a, w.b)


def _gram_operand(seed, m, n, mn=False):
    """A (m x n) and b = (A^T A) x* in n-space, for solves on the implicit
    normal matrix GramProduct(A) (the reference's operator plug-in); with `mn`
    also x* (an exact solution, the min-norm bisection's start)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    xs = rng.standard_normal(n)
    b = a.T @ (a @ xs)
    return (a, b, xs) if mn else (a, b)


CASES = [
    # --- CTA (centering_solve) ------------------------------------------------
    ("cta_c1_window", lambda: _c(W.dense_gaussian(64, 64, seed=1)), "cta",
     dict(epsilon=1e-8, max_iters=40)),
    ("cta_c1_cap", lambda: _c(W.dense_gaussian(64, 64, seed=1)), "cta",
     dict(epsilon=1e-8, max_iters=600)),
    ("cta_c2_lowrank", lambda: _c(W.dense_lowrank(120, 480, 48, seed=2)), "cta",
     dict(epsilon=1e-8)),
    ("cta_c3_clement", lambda: _c(W.clement_variant(301, seed=3)), "cta",
     dict(epsilon=1e-8, max_iters=800)),
    ("cta_c4_convdiff", lambda: _c(W.convdiff_upwind(12, seed=4)), "cta",
     dict(epsilon=1e-8, max_iters=700)),
    ("cta_sym_diag", lambda: (_diag(np.arange(1.0, 101.0)), np.arange(1.0, 101.0)), "cta",
     dict(epsilon=1e-10 / float(np.linalg.norm(np.arange(1.0, 101.0))), h_mode="a")),
    ("cta_random_start", lambda: (_diag(np.linspace(1.0, 4.0, 20)), np.linspace(1.0, 4.0, 20)),
     "cta", dict(epsilon=1e-10, start="random", start_seed=9, h_mode="a")),
    ("cta_accelerate", lambda: (_diag([1.0, 1000.0]),
                                np.array([np.sqrt(1000.0 / 1001.0), np.sqrt(1.0 / 1001.0)])),
     "cta", dict(epsilon=1e-10, h_mode="a", t_max=1, max_iters=20000, accelerate=True)),
    ("cta_enhanced", lambda: (lambda r: (r.standard_normal((8, 3)), r.standard_normal(8)))(
        np.random.default_rng(12)), "cta", dict(epsilon=1e-9, enhanced=True)),
    ("cta_enhanced_probe31", lambda: _probe_case(31), "cta", dict(epsilon=1e-9, enhanced=True)),
    ("cta_enhanced_probe38", lambda: _probe_case(38), "cta", dict(epsilon=1e-9, enhanced=True)),
    ("cta_known_solvable", lambda: (_poisson2d(8), _poisson2d(8).sum(axis=1)), "cta",
     dict(epsilon=1e-13, h_mode="a", known_solvable=True)),
    ("cta_rank1_ne", lambda: (np.outer([1.0, 0.0], [1.0, 1.0]), np.array([0.0, 1.0])), "cta",
     dict(epsilon=1e-12)),
    ("cta_sparse_rect", lambda: (sparse.csr_array(sparse.random_array(
        (40, 90), density=0.1, rng=np.random.default_rng(5))), np.random.default_rng(6).standard_normal(40)),
     "cta", dict(epsilon=1e-9, max_iters=2000)),
    # CTA on the implicit normal matrix (centering.py:278 over linalg.py:93-114)
    ("cta_gram_operand", lambda: _gram_operand(21, 30, 12), "cta_gramop",
     dict(epsilon=1e-8, max_iters=40)),
    ("cta_gram_operand_sym", lambda: _gram_operand(22, 25, 9), "cta_gramop",
     dict(epsilon=1e-10, h_mode="a", max_iters=60)),
    # --- TA (solve_adaptive) --------------------------------------------------
    ("ta_c1_window", lambda: _c(W.dense_gaussian(64, 64, seed=1)), "ta",
     dict(eps_rel=1e-8, max_iters=50)),
    ("ta_c1_500", lambda: _c(W.dense_gaussian(64, 64, seed=1)), "ta",
     dict(eps_rel=1e-8, max_iters=500)),
    ("ta_c1_revalidate", lambda: _c(W.dense_gaussian(24, 24, seed=7)), "ta",
     dict(eps_rel=1e-10, max_iters=1300)),
    ("ta_c5_lp_matrix", lambda: _c(W.lp_columns(60, 3000, 10, seed=5)), "ta",
     dict(eps_rel=1e-6)),
    ("ta_diag", lambda: (_diag([1.0, 2.0]), np.array([1.0, 2.0])), "ta", dict(eps=1e-10)),
    ("ta_inconsistent", lambda: (np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([1.0, 1.0])), "ta",
     dict(eps=1e-12, eps_prime=1e-10)),
    ("ta_exact_zero", lambda: (np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([0.0, 1.0])), "ta",
     dict(eps=1e-12)),
    ("ta_restart", lambda: (lambda r: (lambda a: (a, a @ r.standard_normal(9)))(r.standard_normal((4, 9))))(
        np.random.default_rng(9)), "ta", dict(eps=1e-10, eps_prime=1e-2, restart_halvings=60)),
    ("ta_rho_cap", lambda: (np.array([[1.0, 0.0], [0.0, 1e-3]]), np.array([1.0, 1.0])), "ta",
     dict(eps=1e-12, rho_cap=50.0)),
    ("ta_sparse_c3", lambda: _c(W.clement_variant(101, seed=8)), "ta",
     dict(eps_rel=1e-8, max_iters=400)),
    ("ta_gram", lambda: (lambda r: (r.standard_normal((3, 6)), r.standard_normal(3)))(
        np.random.default_rng(5)), "ta_gram", dict(eps_rel=1e-9, max_iters=100000)),
    # --- in-ball (solve_in_ball) ----------------------------------------------
    ("ball_inside", lambda: (np.eye(2), np.array([1.0, 0.0])), "ball", dict(rho=1.0, eps=1e-12)),
    ("ball_witness", lambda: (np.eye(2), np.array([2.0, 0.0])), "ball", dict(rho=1.0, eps=1e-12)),
    ("ball_random_witness", lambda: _inball(3), "ball", dict(rho_frac=0.5, eps=1e-10, max_iters=20000)),
    ("ball_random_inside", lambda: _inball(4), "ball", dict(rho_frac=1.5, eps=1e-8, max_iters=3000)),
    # --- LP (nonnegative_feasibility) -----------------------------------------
    ("lp_c5_stall", lambda: _c(W.lp_columns(60, 3000, 10, seed=5)), "lp", dict(eps_rel=1e-6)),
    ("lp_identity", lambda: (np.eye(2), np.array([1.0, 1.0])), "lp", dict(eps=1e-8)),
    ("lp_obstructed", lambda: (np.array([[1.0, 1.0]]), np.array([-1.0])), "lp",
     dict(eps=1e-8, max_iters=10000)),
    ("lp_random_feasible", lambda: _rand_feasible_lp(1), "lp", dict(eps=1e-8, max_iters=400000)),
    ("lp_sparse_feasible", lambda: (lambda w: (w.a, w.b))(W.lp_columns(8, 40, 3, seed=11)), "lp",
     dict(eps_rel=1e-6, max_iters=200000)),
    # --- min-norm bisection (min_norm_solve) -------------------------------------
    ("mn_identity", lambda: (np.eye(2), np.array([1.0, 0.0]), np.array([1.0, 0.0])), "mn",
     dict(eps=1e-6)),
    ("mn_wide_row", lambda: (np.array([[1.0, 1.0]]), np.array([2.0]), np.array([2.0, 0.0])), "mn",
     dict(eps=1e-6)),
    ("mn_underdetermined", lambda: _mn_under(6), "mn", dict(eps=1e-6)),
    ("mn_bisection", lambda: (lambda r: (lambda a, x0: (a, a @ x0, x0))(
        r.standard_normal((3, 7)), r.standard_normal(7)))(np.random.default_rng(7)), "mn",
     dict(eps=1e-7)),
    ("mn_ne_branch", lambda: (np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([1.0, 0.5]),
                              np.array([1.0, 0.0])), "mn", dict(eps=0.6)),
    ("mn_gram_operand", lambda: _gram_operand(23, 6, 10, mn=True), "mn_gramop", dict(eps=1e-6)),
    # --- hybrid CTA -> TA (hybrid_solve) --------------------------------------
    ("hy_min_norm", lambda: (lambda r: (lambda a: (a, a @ r.standard_normal(5)))(
        r.standard_normal((2, 5))))(np.random.default_rng(0)), "hybrid",
     dict(eps_cta=1e-8, eps_ta=1e-8, want_min_norm=True)),
    ("hy_overdetermined", lambda: (lambda r: (r.standard_normal((5, 2)), r.standard_normal(5)))(
        np.random.default_rng(1)), "hybrid", dict(eps_cta=1e-8, eps_ta=1e-9)),
    ("hy_consistent", lambda: (lambda r: (lambda a: (a, a @ r.standard_normal(6)))(
        r.standard_normal((3, 6))))(np.random.default_rng(2)), "hybrid",
     dict(eps_cta=1e-6, eps_ta=1e-12)),
    ("hy_c2_lowrank", lambda: _c(W.dense_lowrank(60, 200, 20, seed=9)), "hybrid",
     dict(eps_cta=1e-8, eps_ta=1e-10)),
    ("hy_gram_operand", lambda: _gram_operand(24, 20, 8), "hybrid_gramop",
     dict(eps_cta=1e-6, eps_ta=1e-12, max_iters_stage2=40)),
]


def case_by_name(name):
    for c in CASES:
        if c[0] == name:
            return c
    raise KeyError(name)
