// CTA (centering family) device pieces: moments epilogues, the equilibrated
// min-norm Hankel solve, the monotone-retry candidate pass and the fused
// residual / solution update (centering.py:67-213, driver 263-358).
#pragma once

#include "ts_state.cuh"

namespace ts {

// ---- equilibrated min-norm Hankel solve (centering.py:87-110) -------------
// numpy: hankel[i,j] = phi[i+j+1]; rhs = phi[:t]; s = sqrt|diag| (0 -> 1);
// beta = lstsq(hankel / outer(s,s), rhs / s, rcond) ; alpha = beta / s.
// lstsq (LAPACK gelsd) is the SVD pseudo-inverse with singular values
// <= rcond * s_max dropped.  The balanced matrix is exactly symmetric, so its
// SVD is |eigen-decomposition|: cyclic Jacobi in fp64 gives the eigenpairs.
// Returns false on non-finite input (numpy raises LinAlgError there).
// Register-resident version: every index is a compile-time constant after
// unrolling, so B, V stay in registers (T <= kTMax).
// Fast path of the same solve: Cholesky of the balanced matrix B (symmetric
// positive semi-definite: a Gram matrix of Krylov vectors).  When
// lambda_min(B) >= 1 / trace(B^-1) exceeds 10 * rcond * trace(B) >= 10 * rcond *
// lambda_max(B), gelsd would keep every singular value, so its answer is the
// unique solution B^-1 c, which the Cholesky solve delivers (both are
// backward stable).  T square roots and reciprocals in sequence instead of
// Jacobi sweeps (measured 15-25 us per CTA step on C1/C3/C4).  Returns false
// (caller falls back to Jacobi) when B is not numerically positive definite
// or too ill-conditioned for that guarantee.
template <int T>
__device__ __forceinline__ bool chol_solve_T(const double (&B)[T][T], const double (&c)[T], double rcond,
                                             double (&beta)[T]) {
  double L[T][T], W[T][T];
  double trB = 0.0;
#pragma unroll
  for (int j = 0; j < T; ++j) {
    trB += B[j][j];
    double d = B[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d);
    const double inv = 1.0 / ljj;
    L[j][j] = ljj;
    W[j][j] = inv;
#pragma unroll
    for (int i = j + 1; i < T; ++i) {
      double v = B[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[i][k] * L[j][k];
      L[i][j] = v * inv;
    }
  }
  // W = L^-1 (lower triangular); trace(B^-1) = ||W||_F^2
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < T; ++i) {
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double v = 0.0;
#pragma unroll
      for (int k = j; k < i; ++k) v += L[i][k] * W[k][j];
      W[i][j] = -v * W[i][i];
      tr += W[i][j] * W[i][j];
    }
    tr += W[i][i] * W[i][i];
  }
  if (!(tr * trB * rcond * 10.0 < 1.0)) return false;
  double y[T];
#pragma unroll
  for (int i = 0; i < T; ++i) {
    double v = 0.0;
#pragma unroll
    for (int j = 0; j <= i; ++j) v += W[i][j] * c[j];
    y[i] = v;
  }
#pragma unroll
  for (int j = 0; j < T; ++j) {
    double v = 0.0;
#pragma unroll
    for (int i = j; i < T; ++i) v += W[i][j] * y[i];
    beta[j] = v;
  }
  return true;
}

template <int T>
__device__ __forceinline__ bool hankel_T(const double* phi, double rcond, double* alpha) {
  double B[T][T], V[T][T], s[T], c[T];
  bool finite = true;
#pragma unroll
  for (int i = 0; i < T; ++i) {
    s[i] = sqrt(fabs(phi[2 * i + 1]));
    if (s[i] == 0.0) s[i] = 1.0;
  }
#pragma unroll
  for (int i = 0; i < T; ++i) {
#pragma unroll
    for (int j = 0; j < T; ++j) {
      B[i][j] = phi[i + j + 1] / (s[i] * s[j]);  // hankel / outer(s, s)
      V[i][j] = (i == j) ? 1.0 : 0.0;
      finite = finite && isfinite(B[i][j]);
    }
    c[i] = phi[i] / s[i];
    finite = finite && isfinite(c[i]);
  }
  if (!finite) return false;
  {
    double bc[T];
    if (chol_solve_T<T>(B, c, rcond, bc)) {
      bool ok = true;
#pragma unroll
      for (int i = 0; i < T; ++i) {
        alpha[i] = bc[i] / s[i];
        ok = ok && isfinite(alpha[i]);
      }
      if (ok) return true;
    }
  }
  // cyclic Jacobi: rotate while some |b_pq| > eps * sqrt|b_pp b_qq|
  for (int sweep = 0; sweep < 32; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < T - 1; ++p) {
#pragma unroll
      for (int q = p + 1; q < T; ++q) {
        const double apq = B[p][q], app = B[p][p], aqq = B[q][q];
        if (apq != 0.0 && fabs(apq) > 1e-16 * sqrt(fabs(app * aqq))) {
          rotated = true;
          const double tau = (aqq - app) / (2.0 * apq);
          const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          const double cs = 1.0 / sqrt(1.0 + tt * tt);
          const double sn = tt * cs;
#pragma unroll
          for (int k = 0; k < T; ++k) {  // B <- B J
            const double bkp = B[k][p], bkq = B[k][q];
            B[k][p] = cs * bkp - sn * bkq;
            B[k][q] = sn * bkp + cs * bkq;
          }
#pragma unroll
          for (int k = 0; k < T; ++k) {  // B <- J^T B
            const double bpk = B[p][k], bqk = B[q][k];
            B[p][k] = cs * bpk - sn * bqk;
            B[q][k] = sn * bpk + cs * bqk;
          }
#pragma unroll
          for (int k = 0; k < T; ++k) {  // V <- V J
            const double vkp = V[k][p], vkq = V[k][q];
            V[k][p] = cs * vkp - sn * vkq;
            V[k][q] = sn * vkp + cs * vkq;
          }
        }
      }
    }
    if (!rotated) break;
  }
  double smax = 0.0;
#pragma unroll
  for (int k = 0; k < T; ++k) smax = fmax(smax, fabs(B[k][k]));
  const double cut = rcond * smax;  // gelsd: s_i <= rcond * s_max treated as zero
  double beta[T];
#pragma unroll
  for (int i = 0; i < T; ++i) beta[i] = 0.0;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const double lam = B[k][k];
    if (fabs(lam) > cut) {
      double proj = 0.0;
#pragma unroll
      for (int i = 0; i < T; ++i) proj += V[i][k] * c[i];
      const double wk = proj / lam;
#pragma unroll
      for (int i = 0; i < T; ++i) beta[i] += wk * V[i][k];
    }
  }
  bool ok = true;
#pragma unroll
  for (int i = 0; i < T; ++i) {
    alpha[i] = beta[i] / s[i];
    ok = ok && isfinite(alpha[i]);
  }
  return ok;
}

__device__ __noinline__ bool hankel_min_norm(const double* phi, int order, double rcond,
                                             double* alpha) {
  switch (order) {
    case 1: return hankel_T<1>(phi, rcond, alpha);
    case 2: return hankel_T<2>(phi, rcond, alpha);
    case 3: return hankel_T<3>(phi, rcond, alpha);
    case 4: return hankel_T<4>(phi, rcond, alpha);
    case 5: return hankel_T<5>(phi, rcond, alpha);
    case 6: return hankel_T<6>(phi, rcond, alpha);
    case 7: return hankel_T<7>(phi, rcond, alpha);
    case 8: return hankel_T<8>(phi, rcond, alpha);
    default: return false;
  }
}

// triangle-wave order schedule (centering.py:254-260)
__device__ __forceinline__ int sched_order(int t_max, int pos) {
  if (t_max == 1) return 1;
  const int len = 2 * t_max - 2;
  const int k = pos % len;
  return k < t_max ? k + 1 : 2 * t_max - 1 - k;
}

// loop top: `while iterations < max_iters`, residual checks, next order
// (centering.py:296-304)
__device__ inline void cta_head(SolveState* s) {
  if (s->status != TS_RUNNING) return;
  if (s->iterations >= s->max_iters) {
    s->status = TS_ITERATION_CAP;
    return;
  }
  if (!isfinite(s->r_norm)) {
    s->status = TS_NUMERICAL_FAILURE;
    s->detail = TS_DETAIL_NONFINITE_RESIDUAL;
    return;
  }
  if (s->r_norm <= s->eps_abs) {
    s->status = TS_APPROX_SOLUTION;
    return;
  }
  s->t = sched_order(s->t_max, s->sched_pos);
  s->slot = s->t_max == 1 ? 0 : s->sched_pos % (2 * s->t_max - 2);
  s->sched_pos += 1;
}

// init (start = "zero"): r = b.  sums: b.b, r.r ; x = 0
struct EpiCtaInit : EpiBase {
  static constexpr int K = 2;
  const double* b;
  double *r, *x;
  int64_t m, n;
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t i, double (&acc)[K]) const {
    if (i < m) {
      const double bi = b[i];
      r[i] = bi;
      acc[0] = fma(bi, bi, acc[0]);
      acc[1] = fma(bi, bi, acc[1]);
    }
    if (i < n) x[i] = 0.0;
  }
  __device__ void finish(double (&red)[K]) const;
};
// init (start = "random"): r = b - A x.  sums: b.b, r.r
struct EpiCtaInitR : EpiBase {
  static constexpr int K = 2;
  const double* b;
  double* r;
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    const double bi = b[i];
    const double ri = __dsub_rn(bi, y);
    r[i] = ri;
    acc[0] = fma(bi, bi, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  __device__ void finish(double (&red)[K]) const;
};

__device__ inline void cta_init_finish(SolveState* s, double bb, double rr) {
  s->t0 = globaltimer();
  s->b_norm = sqrt(bb);
  if (s->b_norm == 0.0) {
    s->trivial = 1;
    s->status = TS_APPROX_SOLUTION;
    return;
  }
  s->eps_abs = s->epsilon * s->b_norm;
  s->quad = s->eps_abs * s->eps_abs;
  s->r_norm = sqrt(rr);
  cta_head(s);
}
__device__ inline void EpiCtaInit::finish(double (&red)[K]) const { cta_init_finish(st, red[0], red[1]); }
__device__ inline void EpiCtaInitR::finish(double (&red)[K]) const { cta_init_finish(st, red[0], red[1]); }

__device__ __forceinline__ bool cta_pair_active(const SolveState* s, int i) {
  return s->status == TS_RUNNING && s->maint == MAINT_NONE && s->t >= i;
}

// q_i = A^T p_{i-1}.  sums: q.q (kept for i == 1: ||A^T r||)
struct EpiCtaQ : EpiBase {
  static constexpr int K = 1;
  double* q;
  int i;
  __device__ bool active() const { return cta_pair_active(st, i) && slot_ok(st, slot); }
  __device__ void elem(int64_t j, double y, double (&acc)[K]) const {
    q[j] = y;
    acc[0] = fma(y, y, acc[0]);
  }
  __device__ void finish(double (&red)[K]) const {
    if (i == 1) st->atr2 = red[0];
  }
};

// p_i = A q_i (Gram) or A p_{i-1} (symmetric).  sums: p_{i-1}.p_i, p_i.p_i
// -> phi_{2i-1}, phi_{2i} (centering.py:80-83)
struct EpiCtaP : EpiBase {
  static constexpr int K = 2;
  const double* pprev;
  double* p;
  int i;
  __device__ bool active() const { return cta_pair_active(st, i) && slot_ok(st, slot); }
  __device__ void elem(int64_t r, double y, double (&acc)[K]) const {
    p[r] = y;
    acc[0] = fma(pprev[r], y, acc[0]);
    acc[1] = fma(y, y, acc[1]);
  }
  __device__ void finish(double (&red)[K]) const {
    st->phi[2 * i - 2] = red[0];
    st->phi[2 * i - 1] = red[1];
    if (i == st->t && with_solve) {
      if (st->phi[1] == 0.0) {  // H r == 0: NormalEquationReached (centering.py:183-184)
        st->status = TS_NORMAL_EQ_SOLUTION;
        return;
      }
      st->atr_norm = st->gram ? sqrt(st->atr2) : sqrt(st->phi[1]);
      // enhanced probe: first step uses phi_1 = r.Hr, phi_2 = Hr.Hr (centering.py:241-245)
      st->probe_hit = 0;
      st->probe_done = !(st->enhanced && st->t >= 2);
      if (!st->probe_done) st->probe_alpha = st->phi[0] / st->phi[1];
    }
  }
  // the last pass of the moments runs the order-1..t Hankel solves, one
  // thread per order, in its finishing block (no separate launch)
  __device__ void finish_block() const {
    __shared__ int bad;
    if (!(with_solve && i == st->t && st->status == TS_RUNNING)) return;
    __shared__ unsigned long long t0;
    if (threadIdx.x == 0) {
      bad = 0;
      t0 = globaltimer();
    }
    __syncthreads();
    // one WARP per order: the orders run different code (hankel_T<o>), so lanes
    // of one warp would run them one after another
    const int o = (threadIdx.x >> 5) + 1;
    if ((threadIdx.x & 31) == 0 && o <= st->t) {
      if (!hankel_min_norm(st->phi, o, st->rcond, st->alpha_o[o - 1])) atomicExch(&bad, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (bad) {
        st->status = TS_NUMERICAL_FAILURE;
        st->detail = TS_DETAIL_MOMENT_SOLVE;
      }
      KTimer* kt = &st->kt[3];  // live accounting class 3: the Hankel solves
      kt->total_ns += globaltimer() - t0;
      kt->count += 1;
    }
  }
  int with_solve = 1;
};

// Graph head (once per launch, before the WHILE node): select the order-t case
// of the first trip's SWITCH node (t - 1); later trips are selected by the
// update's finisher.  Not running: no case and no trip.
__global__ void k_cta_head(SolveState* s, cudaGraphConditionalHandle sw, cudaGraphConditionalHandle hw,
                           int nocase) {
  if (threadIdx.x == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&s->launches), 1ull);
    const bool run = s->status == TS_RUNNING && s->maint == MAINT_NONE;
    cudaGraphSetConditional(sw, run ? (unsigned)(s->t - 1) : (unsigned)nocase);
    if (!run) cudaGraphSetConditional(hw, 0u);  // nothing to do: skip the loop
  }
}

struct KrylovPtrs {
  double* p[kTMax + 1];  // p[0] = r
  double* q[kTMax];      // Gram directions
};

// candidate residuals for every order o <= t (r - sum_{i<=o} alpha^o_i p_i,
// centering.py:189-199).  sums: ||cand_o||^2, o = 1..kTMax
struct EpiCtaCand : EpiBase {
  static constexpr int K = kTMax;
  KrylovPtrs kp;
  int64_t m;
  int t_c = 0;
  const double* al_s = nullptr;  // block copy of alpha_o (shared memory)
  __device__ bool active() const { return running(st) && slot_ok(st, slot); }
  __device__ void prepare(double* smem) {
    t_c = st->t;
    for (int k = threadIdx.x; k < kTMax * kTMax; k += kNT) smem[k] = (&st->alpha_o[0][0])[k];
    al_s = smem;
  }
  __device__ void elem(int64_t j, double (&acc)[K]) const {
    const int t = t_c;
    const double rj = kp.p[0][j];
    double pv[kTMax];
#pragma unroll
    for (int i = 0; i < kTMax; ++i) pv[i] = (i < t) ? kp.p[i + 1][j] : 0.0;
#pragma unroll
    for (int o = 1; o <= kTMax; ++o) {
      if (o > t) break;
      double cv = rj;
#pragma unroll
      for (int i = 0; i < kTMax; ++i)
        if (i < o) cv = __dsub_rn(cv, __dmul_rn(al_s[(o - 1) * kTMax + i], pv[i]));
      acc[o - 1] = fma(cv, cv, acc[o - 1]);
    }
  }
  // pair version: the same per-element arithmetic for j, j+1 (128-bit loads),
  // order-t specialised so the t direction loads are independent registers
  static constexpr bool kPair = true;
  static constexpr int kVecBlocks = 2;  // 128 registers: the order-8 pair paths spilled at 64
  template <int T>
  __device__ __forceinline__ void cand2(int64_t j, double (&acc)[K]) const {
    double2 r, pv[T];
    if (j + 1 < m) {
      r = ld_pair(kp.p[0] + j);
#pragma unroll
      for (int i = 0; i < T; ++i) pv[i] = ld_pair(kp.p[i + 1] + j);
    } else {
      r = make_double2(kp.p[0][j], 0.0);
#pragma unroll
      for (int i = 0; i < T; ++i) pv[i] = make_double2(kp.p[i + 1][j], 0.0);
    }
    const bool two = j + 1 < m;
#pragma unroll
    for (int o = 1; o <= T; ++o) {
      double cx = r.x, cy = r.y;
#pragma unroll
      for (int i = 0; i < o; ++i) {
        const double a = al_s[(o - 1) * kTMax + i];
        cx = __dsub_rn(cx, __dmul_rn(a, pv[i].x));
        cy = __dsub_rn(cy, __dmul_rn(a, pv[i].y));
      }
      acc[o - 1] = fma(cx, cx, acc[o - 1]);
      if (two) acc[o - 1] = fma(cy, cy, acc[o - 1]);
    }
  }
  // orders above the default t_max = 5 take the scalar path twice (the same
  // arithmetic and accumulation order; the order-8 pair code spilled)
  __device__ void elem2(int64_t j, double (&acc)[K]) const {
    switch (t_c) {
      case 1: cand2<1>(j, acc); break;
      case 2: cand2<2>(j, acc); break;
      case 3: cand2<3>(j, acc); break;
      case 4: cand2<4>(j, acc); break;
      case 5: cand2<5>(j, acc); break;
      default:
        elem(j, acc);
        if (j + 1 < m) elem(j + 1, acc);
        break;
    }
  }
  __device__ void finish(double (&red)[K]) const {
    SolveState* s = st;
    const int t = s->t;
    int best = -1;
    double best_n = 0.0;
    for (int o = t; o >= 1; --o) {
      const double cn = sqrt(red[o - 1]);
      s->cand[o - 1] = cn;
      if (best < 0 || cn < best_n) {
        best = o;
        best_n = cn;
      }
      if (cn <= s->r_norm * (1.0 + 1e-13)) {  // _MONOTONE_SLACK
        best = o;
        best_n = cn;
        break;
      }
    }
    s->sel_order = best;
    trace_row(s, s->iterations, t, s->r_norm, s->atr_norm, 0.0, 0.0, globaltimer());
    if (!s->known_solvable && s->atr_norm * s->atr_norm <= s->quad) {
      s->status = TS_NORMAL_EQ_SOLUTION;  // x_new discarded (centering.py:318-323)
      s->detail = TS_DETAIL_NE_CERTIFIED_CTA;
      s->detail_value = s->eps_abs;
      return;
    }
    s->blend = 0;
    if (s->accelerate) {  // centering.py:324-332
      const double ratio = s->r_norm > 0.0 ? best_n / s->r_norm : 0.0;
      s->slow_steps = ratio > s->accel_ratio ? s->slow_steps + 1 : 0;
      if (s->slow_steps >= s->accel_patience) {
        s->w_blend = ratio / (1.0 + ratio);
        s->blend = 1;
        s->slow_steps = 0;
      }
    }
  }
};

// r <- chosen candidate; x <- x + sum alpha_i dir_i (centering.py:200-204,
// 333), optional acceleration blend.  sums: ||r||^2
struct EpiCtaUpd : EpiBase {
  static constexpr int K = 1;
  KrylovPtrs kp;
  double* x;
  int64_t m, n;
  int gram;
  int o_c = 0, blend_c = 0;
  double w_c = 0.0;
  const double* al_s = nullptr;
  __device__ bool active() const { return running(st) && slot_ok(st, slot); }
  __device__ void prepare(double* smem) {
    o_c = st->sel_order;
    blend_c = st->blend;
    w_c = st->w_blend;
    if (o_c >= 1)
      for (int k = threadIdx.x; k < kTMax; k += kNT) smem[k] = st->alpha_o[o_c - 1][k];
    al_s = smem;
  }
  __device__ void elem(int64_t j, double (&acc)[K]) const {
    const int o = o_c;
    const double* al = al_s;
    const int blend = blend_c;
    const double w = w_c;
    double rold = 0.0, rnew = 0.0;
    if (j < m) {
      rold = kp.p[0][j];
      double cv = rold;
      for (int i = 0; i < o; ++i) cv = __dsub_rn(cv, __dmul_rn(al[i], kp.p[i + 1][j]));
      rnew = cv;
    }
    if (j < n) {
      const double xo = x[j];
      double xn = xo;
      for (int i = 0; i < o; ++i) {
        const double dv = gram ? kp.q[i][j] : (i == 0 ? rold : kp.p[i][j]);
        xn = __dadd_rn(xn, __dmul_rn(al[i], dv));
      }
      if (blend) xn = __dadd_rn(__dmul_rn(w, xo), __dmul_rn(1.0 - w, xn));
      x[j] = xn;
    }
    if (j < m) {
      if (blend) rnew = __dadd_rn(__dmul_rn(w, rold), __dmul_rn(1.0 - w, rnew));
      kp.p[0][j] = rnew;
      acc[0] = fma(rnew, rnew, acc[0]);
    }
  }
  // pair version (elements j, j+1; 128-bit loads), specialised on the chosen
  // order so every direction load is issued before the arithmetic
  static constexpr bool kPair = true;
  static constexpr int kVecBlocks = 2;  // 128 registers: the order-8 pair paths spilled at 64
  template <int O>
  __device__ __forceinline__ void upd2(int64_t j, double (&acc)[K]) const {
    const double* al = al_s;
    const int blend = blend_c;
    const double w = w_c;
    const bool hm = j < m, hn = j < n, pm = j + 1 < m, pn = j + 1 < n;
    double2 rold = make_double2(0.0, 0.0), pv[O > 0 ? O : 1], dv[O > 0 ? O : 1], xo;
    if (hm) {
      rold = pm ? ld_pair(kp.p[0] + j) : make_double2(kp.p[0][j], 0.0);
#pragma unroll
      for (int i = 0; i < O; ++i) pv[i] = pm ? ld_pair(kp.p[i + 1] + j) : make_double2(kp.p[i + 1][j], 0.0);
    }
    if (hn) {
      xo = pn ? ld_pair(x + j) : make_double2(x[j], 0.0);
#pragma unroll
      for (int i = 0; i < O; ++i) {
        if (gram) dv[i] = pn ? ld_pair(kp.q[i] + j) : make_double2(kp.q[i][j], 0.0);
        else dv[i] = i == 0 ? rold : pv[i - 1];  // symmetric: dir_i = p_i (p_0 = r)
      }
      double xnx = xo.x, xny = xo.y;
#pragma unroll
      for (int i = 0; i < O; ++i) {
        xnx = __dadd_rn(xnx, __dmul_rn(al[i], dv[i].x));
        xny = __dadd_rn(xny, __dmul_rn(al[i], dv[i].y));
      }
      if (blend) {
        xnx = __dadd_rn(__dmul_rn(w, xo.x), __dmul_rn(1.0 - w, xnx));
        xny = __dadd_rn(__dmul_rn(w, xo.y), __dmul_rn(1.0 - w, xny));
      }
      if (pn) st_pair(x + j, make_double2(xnx, xny));
      else x[j] = xnx;
    }
    if (hm) {
      double rx = rold.x, ry = rold.y;
#pragma unroll
      for (int i = 0; i < O; ++i) {
        rx = __dsub_rn(rx, __dmul_rn(al[i], pv[i].x));
        ry = __dsub_rn(ry, __dmul_rn(al[i], pv[i].y));
      }
      if (blend) {
        rx = __dadd_rn(__dmul_rn(w, rold.x), __dmul_rn(1.0 - w, rx));
        ry = __dadd_rn(__dmul_rn(w, rold.y), __dmul_rn(1.0 - w, ry));
      }
      if (pm) st_pair(kp.p[0] + j, make_double2(rx, ry));
      else kp.p[0][j] = rx;
      acc[0] = fma(rx, rx, acc[0]);
      if (pm) acc[0] = fma(ry, ry, acc[0]);
    }
  }
  __device__ void elem2(int64_t j, double (&acc)[K]) const {
    switch (o_c) {
      case 0: upd2<0>(j, acc); break;
      case 1: upd2<1>(j, acc); break;
      case 2: upd2<2>(j, acc); break;
      case 3: upd2<3>(j, acc); break;
      case 4: upd2<4>(j, acc); break;
      case 5: upd2<5>(j, acc); break;
      default:  // orders above t_max = 5: the scalar path (same arithmetic)
        elem(j, acc);
        if (j + 1 < (m > n ? m : n)) elem(j + 1, acc);
        break;
    }
  }
  __device__ void finish(double (&red)[K]) const {
    SolveState* s = st;
    s->iterations += 1;
    s->r_norm = sqrt(red[0]);
    if (s->enhanced && s->probe_hit) {
      s->maint = MAINT_PROBE;  // centering.py:335-343, finished by the host-driven passes
    } else if (s->recheck_every > 0 && (s->iterations % s->recheck_every) == 0) {
      s->maint = MAINT_RECHECK;
    } else {
      cta_head(s);
    }
    tail();
    // the next trip's SWITCH case (graph mode): the order cta_head just took,
    // the recheck case (index ncases) when it is due, none (ncases + 1) otherwise
    if (use_sw)
      cudaGraphSetConditional(sw, running(s) ? (unsigned)(s->t - 1)
                                  : (s->status == TS_RUNNING && s->maint == MAINT_RECHECK) ? (unsigned)ncases
                                                                                           : (unsigned)(ncases + 1));
  }
  int ncases = 0;
};

// ---- enhanced probe (first_order_probe, centering.py:227-251) ------------
struct ProbePtrs {
  double *y, *hy, *aty, *xh, *fr2;
};
__device__ __forceinline__ bool probe_on(const SolveState* s, int j) {
  return s->status == TS_RUNNING && s->maint == MAINT_NONE && !s->probe_done && j < s->t;
}
// x_hat += alpha (A^T y | y);  y = y - alpha H y     (step j)
struct EpiProbeUpd : EpiBase {
  static constexpr int K = 1;
  KrylovPtrs kp;
  ProbePtrs pp;
  const double* x;
  int64_t m, n;
  int gram, j;
  double pal_c = 0.0;
  __device__ bool active() const { return probe_on(st, j); }
  __device__ void prepare(double*) { pal_c = st->probe_alpha; }
  __device__ void elem(int64_t i, double (&)[K]) const {
    const double al = pal_c;
    double yo = 0.0;
    if (i < m) yo = (j == 1) ? kp.p[0][i] : pp.y[i];
    if (i < n) {
      const double xo = (j == 1) ? x[i] : pp.xh[i];
      const double dir = gram ? ((j == 1) ? kp.q[0][i] : pp.aty[i]) : yo;
      pp.xh[i] = __dadd_rn(xo, __dmul_rn(al, dir));
    }
    if (i < m) {
      const double hr = (j == 1) ? kp.p[1][i] : pp.hy[i];
      pp.y[i] = __dsub_rn(yo, __dmul_rn(al, hr));
    }
  }
  __device__ void finish(double (&)[K]) const {}
};
// Gram mode: aty = A^T y
struct EpiProbeT : EpiBase {
  static constexpr int K = 1;
  double* aty;
  int j;
  __device__ bool active() const { return probe_on(st, j); }
  __device__ void elem(int64_t i, double v, double (&)[K]) const { aty[i] = v; }
  __device__ void finish(double (&)[K]) const {}
};
// hy = H y; hit test |y.Hy| <= eps_abs^2, else next alpha = y.Hy / Hy.Hy
struct EpiProbeN : EpiBase {
  static constexpr int K = 2;
  const double* y;
  double* hy;
  int j;
  __device__ bool active() const { return probe_on(st, j); }
  __device__ void elem(int64_t r, double v, double (&acc)[K]) const {
    hy[r] = v;
    acc[0] = fma(y[r], v, acc[0]);
    acc[1] = fma(v, v, acc[1]);
  }
  __device__ void finish(double (&red)[K]) const {
    SolveState* s = st;
    if (fabs(red[0]) <= s->quad) {
      s->probe_hit = j;
      s->probe_done = 1;
    } else if (j + 1 >= s->t || red[1] == 0.0) {
      s->probe_done = 1;  // orbit exhausted / terminated without triggering
    } else {
      s->probe_alpha = red[0] / red[1];
    }
  }
};
// post-step comparison: ||A^T (b - A x)|| vs ||A^T (b - A x_hat)||
struct EpiProbeR : EpiBase {  // fr = b - A v
  static constexpr int K = 1;
  const double* b;
  double* fr;
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t i, double y, double (&)[K]) const { fr[i] = __dsub_rn(b[i], y); }
  __device__ void finish(double (&)[K]) const {}
};
struct EpiProbeNR : EpiBase {  // ||A^T fr||
  static constexpr int K = 1;
  int which;  // 0 stepped, 1 refined
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t, double y, double (&acc)[K]) const { acc[0] = fma(y, y, acc[0]); }
  __device__ void finish(double (&red)[K]) const {
    if (which == 0) {
      st->probe_stepped = sqrt(red[0]);
    } else {
      st->probe_refined = sqrt(red[0]);
      st->probe_take = st->probe_refined < st->probe_stepped;
    }
  }
};
struct EpiProbeTake : EpiBase {  // x = x_hat; r = b - A x_hat (when refined wins)
  static constexpr int K = 1;
  const double *xh, *fr2;
  double *x, *r;
  int64_t m, n;
  int take_c = 0;
  __device__ bool active() const { return true; }
  __device__ void prepare(double*) { take_c = st->probe_take; }
  __device__ void elem(int64_t i, double (&)[K]) const {
    if (!take_c) return;
    if (i < n) x[i] = xh[i];
    if (i < m) r[i] = fr2[i];
  }
  __device__ void finish(double (&)[K]) const {
    st->maint = MAINT_NONE;
    st->status = TS_NORMAL_EQ_SOLUTION;
  }
};

// recheck (centering.py:344-352): fresh = b - A x; drift = ||fresh - r||;
// r = fresh.  sums: ||fresh - r||^2, ||fresh||^2
struct EpiCtaRecheck : EpiBase {
  static constexpr int K = 2;
  const double* b;
  double* r;
  int need_maint = 0;  // in-graph recheck: runs only when that maintenance is due
  __device__ bool active() const {
    return st->status == TS_RUNNING && (!need_maint || st->maint == need_maint);
  }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    const double f = __dsub_rn(b[i], y);
    const double d = __dsub_rn(f, r[i]);
    r[i] = f;
    acc[0] = fma(d, d, acc[0]);
    acc[1] = fma(f, f, acc[1]);
  }
  __device__ void finish(double (&red)[K]) const {
    SolveState* s = st;
    s->maint = MAINT_NONE;
    const double drift = sqrt(red[0]);
    const double scale = s->b_norm + s->a_fro * s->x_norm;
    if (drift > 1e-10 * scale) {
      s->status = TS_NUMERICAL_FAILURE;
      s->detail = TS_DETAIL_DRIFT;
      graph_tail();
      return;
    }
    s->r_norm = sqrt(red[1]);
    cta_head(s);
    graph_tail();
  }
  // in-graph recheck (the SWITCH case after the orders): loop condition and the next case
  __device__ void graph_tail() const {
    tail();
    if (use_sw) cudaGraphSetConditional(sw, running(st) ? (unsigned)(st->t - 1) : (unsigned)nocase);
  }
  int nocase = 0;
};

// ---------------------------------------------------------- k_chain_wdense ----
// ALL moment pairs of one CTA iteration in one cooperative kernel, for a small
// L2-resident dense matrix (C1).  Between the pairs only vectors flow — the
// sums phi_k and ||A^T r||^2 are first needed after the last pair (the Hankel
// solve) — so the 2 t products run back to back with a grid barrier after
// each, every pair's three block sums are parked per block as they complete,
// and ONE arrival / last-block reduction at the end runs the t pairs' finishers
// in order and then the Hankel solves.  Against t pair kernels this removes
// t - 1 reduction chains, kernel boundaries and state reads.  Each product
// keeps k_rows_wdense's row arithmetic and row -> (block, warp) split, every sum
// its block / thread composition, the finishers are the epilogues' own: the
// bits of the separate passes.  Up to 5 pairs (15 sums in the two partial rows).
constexpr int kChainMaxT = 5;

// kTail: systems of <= 1024 unknowns — the last block, once it has run the pairs'
// finishers and the Hankel solves, goes straight on with the candidate and the
// update pass (single-block passes: no other block is needed), so a whole CTA
// iteration is ONE kernel.
struct ChainTail {
  EpiCtaCand cand;
  EpiCtaUpd upd;
  int64_t len_cand, len_upd;
};

template <int XN, bool kTail>
__global__ void __launch_bounds__(kNT, 2) k_chain_wdense(const __grid_constant__ DenseRows AT,
                                                        const __grid_constant__ DenseRows A,
                                                        const __grid_constant__ KrylovPtrs kp, SolveState* st,
                                                        int npairs, int slot, const __grid_constant__ Work wk,
                                                        int PT, int PN, const __grid_constant__ ChainTail tail) {
  constexpr int C = kWdChunks;
  __shared__ double sm[kWarps * kKMax];
  __shared__ __align__(16) double xsl[kWdMaxN + 64];
  __shared__ int sflag;
  EpiCtaP ep0;  // activity, accounting and the launch counter are the first pair's
  ep0.st = st; ep0.i = 1; ep0.slot = slot; ep0.tclass = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ep0.count_launch();
  unsigned long long t_in = 0;  // entry time (thread 0): hoisted work stays inside the accounted interval
  if (threadIdx.x == 0) t_in = globaltimer();
  const int64_t P = gridDim.x, b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double2 v[C];
  auto load = [&](const DenseRows& D, int64_t r, int64_t c0) {
    const double* row = D.a + r * D.lda + 2 * lane;
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int64_t c = c0 + 64 * k + 2 * lane;
      v[k] = c < D.lda ? ld_stream2(row + c0 + 64 * k) : make_double2(0.0, 0.0);
    }
  };
  auto rows = [&](const DenseRows& D, int64_t r, int64_t r1, auto&& sink) {
    const int64_t n = D.n;
    bool first = true;
    for (; r < r1; r += kWarps) {
      double a0 = 0.0, a1 = 0.0;
      for (int64_t c0 = 0; c0 < n; c0 += 64 * C) {
        if (!(first && c0 == 0)) load(D, r, c0);
#pragma unroll
        for (int k = 0; k < C; k += 2) {
          const int64_t ca = c0 + 64 * k + 2 * lane, cb = ca + 64;
          if (ca < n) {
            const double2 xa = *reinterpret_cast<const double2*>(xsl + ca);
            a0 = fma(v[k].x, xa.x, a0);
            if (ca + 1 < n) a0 = fma(v[k].y, xa.y, a0);
          }
          if (cb < n) {
            const double2 xb = *reinterpret_cast<const double2*>(xsl + cb);
            a1 = fma(v[k + 1].x, xb.x, a1);
            if (cb + 1 < n) a1 = fma(v[k + 1].y, xb.y, a1);
          }
        }
      }
      first = false;
      const double y = warp_reduce(a0 + a1, RED_SUM);
      if (lane == 0) sink(r, y);
    }
  };
  // stage a vector of length n into xsl; kCoh: written inside this kernel (L2-coherent loads)
  auto stage = [&](const double* x, int64_t n, bool coh) {
    double xr[XN];
#pragma unroll
    for (int u = 0; u < XN; ++u) {
      const int k = threadIdx.x + u * kNT;
      xr[u] = k < n ? (coh ? __ldcg(x + k) : __ldg(x + k)) : 0.0;
    }
    const int npad = (int)((n + 63) & ~(int64_t)63);
#pragma unroll
    for (int u = 0; u < XN; ++u) {
      const int k = threadIdx.x + u * kNT;
      if (k < npad) xsl[k] = k < n ? xr[u] : 0.0;
    }
  };
  const int64_t t0 = b < PT ? AT.m * b / PT : 0, t1 = b < PT ? AT.m * (b + 1) / PT : 0;
  const int64_t r0 = b < PN ? A.m * b / PN : 0, r1 = b < PN ? A.m * (b + 1) / PN : 0;
  int64_t r = t0 + wid;
  if (r < t1) load(AT, r, 0);  // the matrix is immutable: in flight with the state word
  if (!ep0.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ep0.idle();
      if constexpr (kTail) {  // the passes that would have followed: inactive too, the update owns the loop condition
        tail.cand.idle();
        tail.upd.idle();
      }
    }
    return;
  }
  ktimer_begin_at(ep0.timer(), t_in);
  const int t = st->t < npairs ? st->t : npairs;  // the state's order (the slot's, in graph mode)
  const OpsSum ops;
  unsigned nbar = 0;  // barriers passed so far
  for (int i = 1; i <= t; ++i) {
    EpiCtaQ eq;
    eq.st = st; eq.q = kp.q[i - 1]; eq.i = i;
    EpiCtaP ep;
    ep.st = st; ep.pprev = kp.p[i - 1]; ep.p = kp.p[i]; ep.i = i;
    double acc[3] = {0.0, 0.0, 0.0};
    double (&aq)[1] = *reinterpret_cast<double (*)[1]>(&acc[0]);
    double (&ap)[2] = *reinterpret_cast<double (*)[2]>(&acc[1]);
    // q_i = A^T p_{i-1} (p_0 = r comes from an earlier kernel, later p's from this one)
    stage(kp.p[i - 1], AT.n, i > 1);
    __syncthreads();
    rows(AT, r, t1, [&](int64_t row, double y) { eq.elem(row, y, aq); });
    r = r0 + wid;
    if (r < r1) load(A, r, 0);  // A's first rows in flight across the barrier
    grid_barrier(wk.done + 2, ++nbar * (unsigned)P);
    // p_i = A q_i
    stage(kp.q[i - 1], A.n, true);
    __syncthreads();
    rows(A, r, r1, [&](int64_t row, double y) { ep.elem(row, y, ap); });
    block_reduce<3>(acc, sm, ops);
    if (threadIdx.x == 0) {  // pair i's block sums: slots 3 (i - 1) .. 3 (i - 1) + 2 of the two partial rows
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int sl = 3 * (i - 1) + k;
        (sl < kKMax ? wk.bacc : wk.facc)[b * kKMax + (sl < kKMax ? sl : sl - kKMax)] = acc[k];
      }
    }
    if (i < t) {
      r = t0 + wid;
      if (r < t1) load(AT, r, 0);
      grid_barrier(wk.done + 2, ++nbar * (unsigned)P);
    }
  }
  if (arrive_last(wk.done, (unsigned)P, &sflag)) {
    if (threadIdx.x == 0) wk.done[2] = 0u;  // the barrier counter, for the next launch
    // the separate passes' reduction, slot by slot: 256 threads stride the blocks, then the block tree
    for (int i = 1; i <= t; ++i) {
      double red[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) red[k] = 0.0;
      for (int bb = threadIdx.x; bb < (int)P; bb += kNT) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int sl = 3 * (i - 1) + k;
          red[k] += __ldcg((sl < kKMax ? wk.bacc : wk.facc) + (size_t)bb * kKMax + (sl < kKMax ? sl : sl - kKMax));
        }
      }
      block_reduce<3>(red, sm, ops);
      if (threadIdx.x == 0) {
        EpiCtaQ eq;
        eq.st = st; eq.i = i;
        double rq[1] = {red[0]};
        eq.finish(rq);
        EpiCtaP ep;
        ep.st = st; ep.i = i; ep.with_solve = 1;
        double rp[2] = {red[1], red[2]};
        if (i == t) ktimer_end(ep0.timer(), 2 * t);
        ep.finish(rp);
      }
      __syncthreads();
    }
    EpiCtaP ep;
    ep.st = st; ep.i = t; ep.with_solve = 1;
    ep.finish_block();
    if constexpr (kTail) {
      __syncthreads();  // the finishers' state, visible to the whole block
      EpiCtaCand ec = tail.cand;
      EpiCtaUpd eu = tail.upd;
      if (!ec.active()) {
        if (threadIdx.x == 0) ec.idle();
      } else {
        body_vec<EpiCtaCand, false>(tail.len_cand, ec, wk, 0, 1);
      }
      __syncthreads();
      if (!eu.active()) {
        if (threadIdx.x == 0) eu.idle();
      } else {
        body_vec<EpiCtaUpd, false>(tail.len_upd, eu, wk, 0, 1);
      }
    }
  }
}

inline bool dense_chain_ok(const Mat& M, int npairs) {
  static const bool off = [] {
    const char* e = getenv("TS_DENSE_CHAIN");
    return e && e[0] == '0';
  }();
  return !off && npairs >= 1 && npairs <= kChainMaxT && dense_pair_ok(M);
}
inline int launch_chain_wdense(const Mat& M, const KrylovPtrs& kp, SolveState* st, int npairs, int slot,
                               const Work& wk, cudaStream_t s, const ChainTail* tail = nullptr) {
  const int PT = std::min(M.planT.P, 2 * M.sms), PN = std::min(M.planN.P, 2 * M.sms);
  const int P = std::max(PT, PN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(kNT);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const DenseRows dT{M.aT, M.ldaT, M.n, M.m};
  const int64_t len = std::max(M.m, M.n);
  if (!coop_fits(k_chain_wdense<16, false>, P, M)) return kNoCoop;
  if (tail) {  // (<= 1024 unknowns: the 4-entry staging variant)
    if (!coop_fits(k_chain_wdense<4, true>, P, M)) return kNoCoop;
    TS_CUDA(cudaLaunchKernelEx(&cfg, k_chain_wdense<4, true>, dT, M.dense(), kp, st, npairs, slot, wk, PT, PN, *tail));
    return 0;
  }
  const ChainTail none{};
  if (len <= 4 * kNT) TS_CUDA(cudaLaunchKernelEx(&cfg, k_chain_wdense<4, false>, dT, M.dense(), kp, st, npairs, slot, wk, PT, PN, none));
  else if (len <= 8 * kNT) TS_CUDA(cudaLaunchKernelEx(&cfg, k_chain_wdense<8, false>, dT, M.dense(), kp, st, npairs, slot, wk, PT, PN, none));
  else TS_CUDA(cudaLaunchKernelEx(&cfg, k_chain_wdense<16, false>, dT, M.dense(), kp, st, npairs, slot, wk, PT, PN, none));
  return 0;
}

// ------------------------------------------------------------ k_chain_csr ----
// The same chain for an L2-resident short-row CSR matrix that is not banded: thread per row in
// scipy's order (k_rows_short's arithmetic and row -> thread mapping), q and p'
// exchanged through L2 between the phases, so no bandwidth condition and no
// halo recomputation (k_pair_band needs a banded square matrix).
__device__ __forceinline__ double row_serial_cg(const CsrRows& A, int k0, int k1, const double* xq) {
  double s = 0.0;
  int k = k0;
  for (; k + 4 <= k1; k += 4) {
    double v[4], xv[4];
    int j[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = ld_stream(A.val + k + u);
      j[u] = ld_stream_i(A.ci + k + u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = __ldcg(xq + j[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
  }
  const int rem = k1 - k;
  double v[3], xv[3];
  int j[3];
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (u < rem) {
      v[u] = ld_stream(A.val + k + u);
      j[u] = ld_stream_i(A.ci + k + u);
    }
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (u < rem) xv[u] = __ldcg(xq + j[u]);
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (u < rem) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
  return s;
}

__global__ void __launch_bounds__(kNT, kMinBlocks) k_chain_csr(const __grid_constant__ CsrRows AT,
                                                             const __grid_constant__ CsrRows A,
                                                             const __grid_constant__ KrylovPtrs kp, SolveState* st,
                                                             int npairs, int slot, const __grid_constant__ Work wk,
                                                             int PT, int PN) {
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  EpiCtaP ep0;
  ep0.st = st; ep0.i = 1; ep0.slot = slot; ep0.tclass = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ep0.count_launch();
  const int64_t P = gridDim.x, b = blockIdx.x;
  const int64_t t0 = b < PT ? AT.m * b / PT : 0, t1 = b < PT ? AT.m * (b + 1) / PT : 0;
  const int64_t r0 = b < PN ? A.m * b / PN : 0, r1 = b < PN ? A.m * (b + 1) / PN : 0;
  if (!ep0.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ep0.idle();
    return;
  }
  ktimer_begin(ep0.timer());
  const int t = st->t < npairs ? st->t : npairs;
  const OpsSum ops;
  unsigned nbar = 0;
  for (int i = 1; i <= t; ++i) {
    EpiCtaQ eq;
    eq.st = st; eq.q = kp.q[i - 1]; eq.i = i;
    EpiCtaP ep;
    ep.st = st; ep.pprev = kp.p[i - 1]; ep.p = kp.p[i]; ep.i = i;
    double acc[3] = {0.0, 0.0, 0.0};
    double (&aq)[1] = *reinterpret_cast<double (*)[1]>(&acc[0]);
    double (&ap)[2] = *reinterpret_cast<double (*)[2]>(&acc[1]);
    for (int64_t j = t0 + threadIdx.x; j < t1; j += kNT)
      eq.elem(j, row_serial_cg(AT, __ldg(AT.rp + j), __ldg(AT.rp + j + 1), kp.p[i - 1]), aq);
    grid_barrier(wk.done + 2, ++nbar * (unsigned)P);
    for (int64_t r = r0 + threadIdx.x; r < r1; r += kNT)
      ep.elem(r, row_serial_cg(A, __ldg(A.rp + r), __ldg(A.rp + r + 1), kp.q[i - 1]), ap);
    block_reduce<3>(acc, sm, ops);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int sl = 3 * (i - 1) + k;
        (sl < kKMax ? wk.bacc : wk.facc)[b * kKMax + (sl < kKMax ? sl : sl - kKMax)] = acc[k];
      }
    }
    if (i < t) grid_barrier(wk.done + 2, ++nbar * (unsigned)P);
  }
  if (arrive_last(wk.done, (unsigned)P, &sflag)) {
    if (threadIdx.x == 0) wk.done[2] = 0u;  // the barrier counter, for the next launch
    for (int i = 1; i <= t; ++i) {
      double red[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) red[k] = 0.0;
      for (int bb = threadIdx.x; bb < (int)P; bb += kNT) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int sl = 3 * (i - 1) + k;
          red[k] += __ldcg((sl < kKMax ? wk.bacc : wk.facc) + (size_t)bb * kKMax + (sl < kKMax ? sl : sl - kKMax));
        }
      }
      block_reduce<3>(red, sm, ops);
      if (threadIdx.x == 0) {
        EpiCtaQ eq;
        eq.st = st; eq.i = i;
        double rq[1] = {red[0]};
        eq.finish(rq);
        EpiCtaP ep;
        ep.st = st; ep.i = i; ep.with_solve = 1;
        double rp[2] = {red[1], red[2]};
        if (i == t) ktimer_end(ep0.timer(), 2 * t);
        ep.finish(rp);
      }
      __syncthreads();
    }
    EpiCtaP ep;
    ep.st = st; ep.i = t; ep.with_solve = 1;
    ep.finish_block();
  }
}

inline bool csr_chain_ok(const Mat& M, int npairs) {
  static const bool off = [] {
    const char* e = getenv("TS_CSR_CHAIN");
    return e && e[0] == '0';
  }();
  // a banded square matrix keeps one kernel per pair (k_pair_band, halo recomputation
  // instead of barriers): on C3, 391 blocks, 7.4 us per pair against the chain's 8.3
  return !off && npairs >= 1 && npairs <= kChainMaxT && M.kind == 1 && !M.comm && !band_pair_ok(M) &&
         M.planN.kind == PLAN_SHORT && M.planT.kind == PLAN_SHORT &&
         std::max(M.planN.P, M.planT.P) <= M.sms * kMinBlocks;
}
inline int launch_chain_csr(const Mat& M, const KrylovPtrs& kp, SolveState* st, int npairs, int slot,
                            const Work& wk, cudaStream_t s) {
  const int PT = M.planT.P, PN = M.planN.P;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::max(PT, PN));
  cfg.blockDim = dim3(kNT);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (!coop_fits(k_chain_csr, std::max(PT, PN), M)) return kNoCoop;
  TS_CUDA(cudaLaunchKernelEx(&cfg, k_chain_csr, M.csrT(), M.csr(), kp, st, npairs, slot, wk, PT, PN));
  return 0;
}

}  // namespace ts
