// Device-resident solver state and the fused epilogues / finishers.
//
// The reference drivers are host `while` loops with data-dependent branches
// (centering.py:296-352, triangle.py:141-167 / 210-250, feasibility.py:85-133).
// Here every scalar decision is taken ON THE DEVICE by the finisher of the
// pass that produces its inputs (thread 0 of the last block to arrive), and
// every kernel reads the resulting state at entry to decide whether it has
// work.  The host never reads a scalar inside an iteration, so one iteration
// is a static kernel sequence that is captured once into the body of a CUDA
// graph WHILE node; the tail kernel of the body sets the loop condition.
//
// Elementwise updates mirror numpy's rounding exactly (separate multiply and
// add, no FMA contraction: __dmul_rn / __dadd_rn / __dsub_rn), so given the
// same scalars an update is bit-identical to the reference's numpy statement.
#pragma once

#include "ts_matrix.cuh"

namespace ts {

enum Mode : int { MODE_ADAPTIVE = 0, MODE_BALL = 1, MODE_LP = 2, MODE_CTA = 3 };
enum Event : int { EV_NONE = 0, EV_PIVOT = 1, EV_EXPAND = 2 };
enum Maint : int { MAINT_NONE = 0, MAINT_REVALIDATE = 1, MAINT_RECHECK = 2, MAINT_PROBE = 3 };

struct alignas(16) SolveState {
  // control
  int status, detail, maint, event;
  int error, trivial, mode, gram;
  int halvings_left, since_reval, has_lb, warm;
  int t, sched_pos, t_max, sel_order;
  int slow_steps, blend, known_solvable, accelerate;
  int accel_patience, enhanced, seg_cap, slot;  // slot: position in the order schedule's period
  long long iterations, max_iters, recheck_every;
  long long m_rows, n_cols;
  long long trace_count, trace_flushed, body_runs, launches;
  unsigned long long t0, wall_pending;
  // TA / ball / LP
  double eps, eps_prime, rho, rho_cap, rho_max;
  double b_norm, gap_norm, gap_dot_b, c_norm, cp_norm;
  double scale, alpha, x_min, lower_bound, detail_value;
  // CTA
  double epsilon, eps_abs, quad, r_norm, atr_norm, atr2;
  double a_fro, x_norm, ratio, w_blend, accel_ratio, rcond;
  // enhanced probe (first_order_probe, centering.py:227-251)
  int probe_hit, probe_done, probe_take, pad1;
  double probe_alpha, probe_stepped, probe_refined;
  double phi[2 * kTMax];
  double alpha_o[kTMax][kTMax];
  double cand[kTMax];
  // final report
  double residual_norm, normal_residual_norm;
  ts_trace_row* trace;  // device ring of seg_cap rows
  KTimer kt[4];         // [0] A v, [1] A^T v, [2] vector passes, [3] scalar kernels
};

__device__ __forceinline__ void set_cond(cudaGraphConditionalHandle h, int use, const SolveState* s) {
  if (!use) return;
  // the b' = A x revalidation and the CTA residual recheck are cases of the
  // graph's SWITCH node: the loop keeps running through them
  const unsigned keep = (s->status == TS_RUNNING && s->maint != MAINT_PROBE &&
                         (s->trace_count - s->trace_flushed) < (long long)s->seg_cap)
                            ? 1u
                            : 0u;
  cudaGraphSetConditional(h, keep);
}

__device__ __forceinline__ void trace_row(SolveState* s, long long it, int tag, double v0, double v1,
                                          double v2, double v3, unsigned long long wall) {
  ts_trace_row* row = s->trace + (s->trace_count % s->seg_cap);
  row->iter = it;
  row->wall_ns = (long long)(wall - s->t0);
  row->tag = tag;
  row->reserved = 0;
  row->v[0] = v0;
  row->v[1] = v1;
  row->v[2] = v2;
  row->v[3] = v3;
  s->trace_count += 1;
}

__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }  // max(a, b)
__device__ __forceinline__ double py_min(double a, double b) { return b < a ? b : a; }  // min(a, b)

// ===================================================================== TA ====
// head of a TA / ball / LP iteration: the `while` guard and the gap checks
// (triangle.py:141-147, 210-218; feasibility.py:85-92)
__device__ inline void ta_head(SolveState* s) {
  if (s->status != TS_RUNNING) return;
  if (s->iterations >= s->max_iters) {
    if (s->mode == MODE_LP) {
      s->status = TS_INCONCLUSIVE;
      s->detail = TS_DETAIL_ITER_BUDGET;
    } else {
      s->status = TS_ITERATION_CAP;
    }
    return;
  }
  if (!isfinite(s->gap_norm)) {
    s->status = TS_NUMERICAL_FAILURE;
    s->detail = (s->mode == MODE_BALL) ? TS_DETAIL_NONE : TS_DETAIL_NONFINITE_ITERATE;
    return;
  }
  if (s->gap_norm <= s->eps) {
    s->status = (s->mode == MODE_LP) ? TS_FEASIBLE : TS_APPROX_SOLUTION;
    s->detail = TS_DETAIL_NONE;
  }
}

// decision after c = A^T (b - b') (triangle.py:148-167, 219-249;
// feasibility.py:94-132).  sums: ||c||^2, ||c+||^2
__device__ inline void ta_decide(SolveState* s, double c2, double cp2) {
  const double c_norm = sqrt(c2);
  s->c_norm = c_norm;
  s->event = EV_NONE;
  const unsigned long long wall = globaltimer();
  s->wall_pending = wall;
  const double gb = s->gap_dot_b;
  if (s->mode == MODE_LP) {
    const double cpn = sqrt(cp2);
    s->cp_norm = cpn;
    if (cpn == 0.0) {  // constrained stall (feasibility.py:98-107)
      s->status = TS_WITNESS;
      s->lower_bound = c_norm > 0.0 ? gb / c_norm : INFINITY;
      s->has_lb = 1;
      s->detail = TS_DETAIL_CONE_STALL;
      trace_row(s, s->iterations, TS_EVENT_WITNESS, s->rho, s->gap_norm, c_norm, s->x_min, wall);
      s->iterations += 1;
      return;
    }
    if (s->rho > 0.0 && s->rho * cpn >= gb) {
      s->scale = s->rho / cpn;
      s->event = EV_PIVOT;
      return;
    }
    s->rho = py_max(2.0 * s->rho, gb / cpn);
    trace_row(s, s->iterations, TS_EVENT_EXPAND, s->rho, s->gap_norm, c_norm, s->x_min, wall);
    s->event = EV_EXPAND;
    if (s->rho > s->rho_max) {
      s->status = TS_INCONCLUSIVE;
      s->detail = TS_DETAIL_RADIUS_BUDGET;
      s->detail_value = s->rho_max;
      s->iterations += 1;
      return;
    }
    s->iterations += 1;
    ta_head(s);
    return;
  }
  if (c_norm <= s->eps_prime) {
    if (s->mode == MODE_ADAPTIVE) {
      while (c_norm <= s->eps_prime && c_norm > 0.0 && s->halvings_left > 0) {
        s->halvings_left -= 1;  // restart heuristic (triangle.py:222-227)
        s->eps_prime *= 0.5;
      }
      if (c_norm <= s->eps_prime) {
        s->status = TS_NORMAL_EQ_SOLUTION;
        s->detail = c_norm == 0.0 ? TS_DETAIL_PIVOT_VANISHED : TS_DETAIL_NE_CERTIFIED_TA;
        s->detail_value = s->eps_prime;
        return;
      }
    } else {
      s->status = TS_NORMAL_EQ_SOLUTION;
      return;
    }
  }
  if (s->mode == MODE_BALL) {
    if (s->rho * c_norm >= gb) {
      s->scale = s->rho / c_norm;
      s->event = EV_PIVOT;
      return;
    }
    s->lower_bound = gb / c_norm;
    s->has_lb = 1;
    trace_row(s, s->iterations, TS_EVENT_WITNESS, s->rho, s->gap_norm, c_norm, 0.0, wall);
    s->status = TS_WITNESS;
    s->iterations += 1;
    return;
  }
  // adaptive
  if (s->rho > 0.0 && s->rho * c_norm >= gb) {
    s->scale = s->rho / c_norm;
    s->event = EV_PIVOT;
    return;
  }
  s->rho = py_max(2.0 * s->rho, gb / c_norm);
  trace_row(s, s->iterations, TS_EVENT_EXPAND, s->rho, s->gap_norm, c_norm, 0.0, wall);
  s->event = EV_EXPAND;
  if (s->rho > s->rho_cap) {
    s->status = TS_ITERATION_CAP;
    s->detail = TS_DETAIL_RADIUS_CAP;
    s->detail_value = s->rho_cap;
    s->iterations += 1;
    return;
  }
  s->iterations += 1;
  ta_head(s);
}

// ------------------------------------------------------------ epilogues ----
struct EpiBase {
  SolveState* st = nullptr;
  cudaGraphConditionalHandle cond = 0;  // WHILE loop condition (tail kernels)
  cudaGraphConditionalHandle sw = 0;    // SWITCH selector set by a finisher
  int use_cond = 0;
  int use_sw = 0;
  int tclass = -1;  // live accounting class (set by the launch helper)
  int slot = -1;    // CTA period graph: the schedule slot this kernel belongs to (-1: any)
  // vector passes: reduction slots that sum over n-space (column-sharded)
  static constexpr unsigned kShardMask = 0;
  // vector passes: true -> the epilogue provides elem2(i, acc) for elements
  // i, i+1 (i even) and k_vec walks pairs
  static constexpr bool kPair = false;
  __device__ __forceinline__ void count_launch() const {
    if (st) atomicAdd(reinterpret_cast<unsigned long long*>(&st->launches), 1ull);
  }
  __device__ __forceinline__ int op(int) const { return RED_SUM; }
  __device__ __forceinline__ KTimer* timer() const {
    return (st && tclass >= 0) ? &st->kt[tclass] : nullptr;
  }
  __device__ __forceinline__ void idle() const {
    if (use_cond) {
      st->body_runs += 1;
      set_cond(cond, 1, st);
    }
  }
  __device__ __forceinline__ void tail() const {
    if (use_cond) {
      st->body_runs += 1;
      set_cond(cond, 1, st);
    }
  }
  __device__ __forceinline__ void finish_block() const {}
  __device__ __forceinline__ void prepare(double*) {}
};

__device__ __forceinline__ bool running(const SolveState* s) {
  return s->status == TS_RUNNING && s->maint == MAINT_NONE;
}
// CTA period graph (one WHILE trip = one period of the order schedule, every
// iteration's kernels baked in with their slot): a kernel runs when the state
// stands at its slot and the trace ring has room for the iteration's row
__device__ __forceinline__ bool slot_ok(const SolveState* s, int slot) {
  return slot < 0 || (s->slot == slot && (s->trace_count - s->trace_flushed) < (long long)s->seg_cap);
}

// TA init without warm start: b' = 0, gap = b.  sums: gap.gap, gap.b, b.b
struct EpiTaInitZero : EpiBase {
  static constexpr int K = 3;
  const double* b;
  double *bp, *gap, *x;
  int64_t m, n;
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t i, double (&acc)[K]) const {
    if (i < m) {
      const double bi = b[i];
      const double g = __dsub_rn(bi, 0.0);
      bp[i] = 0.0;
      gap[i] = g;
      acc[0] = fma(g, g, acc[0]);
      acc[1] = fma(g, bi, acc[1]);
      acc[2] = fma(bi, bi, acc[2]);
    }
    if (i < n) x[i] = 0.0;
  }
  __device__ void finish(double (&r)[K]) const;
};

// b' = A x (warm start / revalidation), gap = b - b'. sums: gap.gap, gap.b, b.b
struct EpiTaBp : EpiBase {
  static constexpr int K = 3;
  const double* b;
  double *bp, *gap;
  int kind;  // 0: init, 1: revalidate
  __device__ bool active() const { return st->status == TS_RUNNING; }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    const double bi = b[i];
    const double g = __dsub_rn(bi, y);
    bp[i] = y;
    gap[i] = g;
    acc[0] = fma(g, g, acc[0]);
    acc[1] = fma(g, bi, acc[1]);
    acc[2] = fma(bi, bi, acc[2]);
  }
  __device__ void finish(double (&r)[K]) const;
};

// norm of a vector into the state (x0 warm start): sums v.v
struct EpiNormTo : EpiBase {
  static constexpr int K = 1;
  static constexpr unsigned kShardMask = 1u;  // ||v||^2 over n-space
  const double* v;
  int64_t len;
  int what;  // 0: ta x0 (rho / warm flag), 1: cta x norm (recheck)
  int need_maint = 0;  // in-graph recheck: runs only when that maintenance is due
  __device__ bool active() const {
    return st->status == TS_RUNNING && (!need_maint || st->maint == need_maint);
  }
  __device__ void elem(int64_t i, double (&acc)[K]) const {
    const double a = v[i];
    acc[0] = fma(a, a, acc[0]);
  }
  __device__ void finish(double (&r)[K]) const {
    const double nv = sqrt(r[0]);
    if (what == 0) {
      if (st->mode == MODE_BALL) {
        st->warm = nv <= st->rho * (1.0 + 1e-9);
      } else {
        st->rho = nv;  // solve_adaptive: rho = ||x0|| (triangle.py:200)
        st->warm = 1;
      }
    } else {
      st->x_norm = nv;
    }
  }
};

// ||x|| of the final iterate (always active; after the loop)
struct EpiXNorm : EpiBase {
  static constexpr int K = 1;
  static constexpr unsigned kShardMask = 1u;
  const double* v;
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t i, double (&acc)[K]) const { acc[0] = fma(v[i], v[i], acc[0]); }
  __device__ void finish(double (&r)[K]) const { st->x_norm = sqrt(r[0]); }
};

// x = warm ? x0 : 0
struct EpiCopyWarm : EpiBase {
  static constexpr int K = 1;
  const double* src;
  double* dst;
  __device__ bool active() const { return st->status == TS_RUNNING; }
  int warm_c = 0;
  __device__ void prepare(double*) { warm_c = st->warm; }
  __device__ void elem(int64_t i, double (&acc)[K]) const { dst[i] = warm_c ? src[i] : 0.0; }
  __device__ void finish(double (&)[K]) const {}
};

// c = A^T gap.  sums: c.c, c+.c+
struct EpiTaC : EpiBase {
  static constexpr int K = 2;
  double* c;
  __device__ bool active() const { return running(st); }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    c[i] = y;
    acc[0] = fma(y, y, acc[0]);
    const double cp = (y >= 0.0 || y != y) ? y : 0.0;
    acc[1] = fma(cp, cp, acc[1]);
  }
  // graph SWITCH cases: 0 pivot, 1 revalidate (b' = A x, every 512 pivots), 2 none
  __device__ void idle() const {
    if (use_sw)
      cudaGraphSetConditional(sw, (st->status == TS_RUNNING && st->maint == MAINT_REVALIDATE) ? 1u : 2u);
    EpiBase::idle();
  }
  __device__ void finish(double (&r)[K]) const {
    ta_decide(st, r[0], r[1]);
    if (use_sw) cudaGraphSetConditional(sw, st->event == EV_PIVOT ? 0u : 2u);
    if (use_cond) {
      if (st->event != EV_PIVOT) st->body_runs += 1;
      set_cond(cond, 1, st);
    }
  }
};

// v = A pre, d = v - b'.  sums: d.d, gap.d  (move_to_pivot, triangle.py:69-81)
struct EpiTaV : EpiBase {
  static constexpr int K = 2;
  const double *bp, *gap;
  double* d;
  __device__ bool active() const { return st->status == TS_RUNNING && st->event == EV_PIVOT; }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    const double di = __dsub_rn(y, bp[i]);
    d[i] = di;
    acc[0] = fma(di, di, acc[0]);
    acc[1] = fma(gap[i], di, acc[1]);
  }
  __device__ void finish(double (&r)[K]) const {
    if (r[0] == 0.0) {  // "degenerate pivot: v coincides with the iterate"
      st->error = TS_EDEGENERATE;
      st->status = TS_NUMERICAL_FAILURE;
      return;
    }
    st->alpha = py_min(1.0, py_max(0.0, r[1] / r[0]));
  }
};

// b' += alpha d; gap = b - b'; x = (1-alpha) x + alpha pre.
// sums: gap.gap, gap.b, min(x)
struct EpiTaUpd : EpiBase {
  static constexpr int K = 3;
  static constexpr unsigned kShardMask = 1u << 2;  // min(x) over n-space
  const double *b, *d, *c;
  double *bp, *gap, *x;
  int64_t m, n;
  int relu;
  double al_c = 0.0, scale_c = 0.0;
  __device__ int op(int k) const { return k == 2 ? RED_MIN : RED_SUM; }
  __device__ bool active() const { return st->status == TS_RUNNING && st->event == EV_PIVOT; }
  __device__ void prepare(double*) {
    al_c = st->alpha;
    scale_c = st->scale;
  }
  __device__ void elem(int64_t i, double (&acc)[K]) const {
    const double al = al_c;
    if (i < m) {
      const double nb = __dadd_rn(bp[i], __dmul_rn(al, d[i]));
      const double bi = b[i];
      const double g = __dsub_rn(bi, nb);
      bp[i] = nb;
      gap[i] = g;
      acc[0] = fma(g, g, acc[0]);
      acc[1] = fma(g, bi, acc[1]);
    }
    if (i < n) {
      double cv = c[i];
      if (relu) cv = (cv >= 0.0 || cv != cv) ? cv : 0.0;
      const double pre = __dmul_rn(scale_c, cv);
      const double nx = __dadd_rn(__dmul_rn(1.0 - al, x[i]), __dmul_rn(al, pre));
      x[i] = nx;
      acc[2] = py_min(acc[2], nx);
    }
  }
  __device__ void finish(double (&r)[K]) const {
    SolveState* s = st;
    if (s->mode == MODE_LP) {
      const double xm = r[2];
      s->x_min = xm;
      if (xm < -1e-12) {  // feasibility.py:113-118
        s->status = TS_NUMERICAL_FAILURE;
        s->detail = TS_DETAIL_LEFT_CONE;
        tail();
        return;
      }
      trace_row(s, s->iterations, TS_EVENT_PIVOT, s->rho, s->gap_norm, s->c_norm, xm,
                s->wall_pending);
    } else {
      trace_row(s, s->iterations, TS_EVENT_PIVOT, s->rho, s->gap_norm, s->c_norm, 0.0,
                s->wall_pending);
    }
    s->gap_norm = sqrt(r[0]);
    s->gap_dot_b = r[1];
    s->since_reval += 1;
    s->iterations += 1;
    if (s->since_reval >= 512) {
      s->maint = MAINT_REVALIDATE;  // b' = A x (triangle.py:239-242)
    } else {
      ta_head(s);
    }
    tail();
  }
};

// final honest residual: fr = b - A x (sums fr.fr), then ||A^T fr||
struct EpiFinalR : EpiBase {
  static constexpr int K = 1;
  const double* b;
  double* fr;
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    const double f = __dsub_rn(b[i], y);
    fr[i] = f;
    acc[0] = fma(f, f, acc[0]);
  }
  __device__ void finish(double (&r)[K]) const { st->residual_norm = sqrt(r[0]); }
};
struct EpiFinalNR : EpiBase {
  static constexpr int K = 1;
  double* out;  // optional
  __device__ bool active() const { return true; }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    if (out) out[i] = y;
    acc[0] = fma(y, y, acc[0]);
  }
  __device__ void finish(double (&r)[K]) const { st->normal_residual_norm = sqrt(r[0]); }
};

// plain y = M v with an optional sum of squares into a scalar slot.
// pred: 0 always; 1 while running (TA c pass); 2 on pivot iterations.
struct EpiStore : EpiBase {
  static constexpr int K = 1;
  double* y = nullptr;
  double* sq = nullptr;  // optional: ||y||^2
  int pred = 0;
  __device__ bool active() const {
    if (pred == 0) return true;
    if (pred == 1) return running(st);
    return st->status == TS_RUNNING && st->event == EV_PIVOT;
  }
  __device__ void idle() const {}
  __device__ void elem(int64_t i, double v, double (&acc)[K]) const {
    y[i] = v;
    acc[0] = fma(v, v, acc[0]);
  }
  __device__ void finish(double (&r)[K]) const {
    if (sq) *sq = r[0];
  }
};

struct EpiDot {
  static constexpr int K = 1;
  const double *u, *v;
  double* out;
  int sqrt_out;
  __device__ int op(int) const { return RED_SUM; }
  __device__ bool active() const { return true; }
  __device__ void idle() const {}
  __device__ KTimer* timer() const { return nullptr; }
  __device__ void finish_block() const {}
  __device__ void count_launch() const {}
  __device__ void prepare(double*) {}
  __device__ void elem(int64_t i, double (&acc)[K]) const { acc[0] = fma(u[i], v[i], acc[0]); }
  __device__ void finish(double (&r)[K]) const { *out = sqrt_out ? sqrt(r[0]) : r[0]; }
};

// --- finishers that need the full definitions ---------------------------------
__device__ inline void EpiTaInitZero::finish(double (&r)[K]) const {
  SolveState* s = st;
  s->t0 = globaltimer();
  s->b_norm = sqrt(r[2]);
  s->gap_norm = sqrt(r[0]);
  s->gap_dot_b = r[1];
  s->x_min = 0.0;
  if (s->b_norm == 0.0) {
    s->trivial = 1;
    s->status = TS_APPROX_SOLUTION;
    return;
  }
  if (s->eps_prime < 0.0) s->eps_prime = s->eps;
  if (s->rho_cap < 0.0) s->rho_cap = 4.0 * (s->b_norm * s->b_norm) / s->eps_prime;
  if (s->mode == MODE_LP && s->rho_max < 0.0) {
    // default_rho_max (feasibility.py:49-56), sigma = ||A||_F / sqrt(m)
    double sigma = s->a_fro / sqrt((double)s->m_rows);
    if (sigma == 0.0) sigma = 1.0;
    s->rho_max = 10.0 * (double)s->n_cols * py_max(1.0, s->b_norm / sigma);
  }
  ta_head(s);
}

__device__ inline void EpiTaBp::finish(double (&r)[K]) const {
  SolveState* s = st;
  s->gap_norm = sqrt(r[0]);
  s->gap_dot_b = r[1];
  if (kind == 0) {
    s->t0 = globaltimer();
    s->b_norm = sqrt(r[2]);
    s->x_min = 0.0;
    if (s->b_norm == 0.0) {
      s->trivial = 1;
      s->status = TS_APPROX_SOLUTION;
      return;
    }
    if (s->eps_prime < 0.0) s->eps_prime = s->eps;
    if (s->rho_cap < 0.0) s->rho_cap = 4.0 * (s->b_norm * s->b_norm) / s->eps_prime;
  } else {
    s->since_reval = 0;
    s->maint = MAINT_NONE;
  }
  ta_head(s);
  tail();  // in-graph revalidation (SWITCH case 1): the loop condition
}

}  // namespace ts
