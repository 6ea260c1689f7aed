/*
 * mirror.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * A plain-C restatement of the DEVICE arithmetic of the dense TA path
 * (solve_adaptive, reference pkg/src/trisolve/triangle.py:170-251) exactly as
 * the CUDA library executes it: the same launch geometry (grids derived from
 * the SM count), the same per-thread FMA chains, the same xor-butterfly warp
 * reductions, fixed block orders and split-tile merges, and numpy-exact
 * elementwise updates.  It exists so that a long run of the device path can be
 * checked BIT FOR BIT on the CPU (BASELINE configs[0]: "TA at fixed 500
 * iterations for the bitwise-path check (runs on CPU)"), something the numpy
 * oracle cannot do: past ~50 iterations the reference disagrees with itself
 * once only the BLAS reduction order changes.
 *
 * Device code it restates (paper_2304_12168_b200/csrc/):
 *   k_cols_tile<Epi,2>          ts_passes.cuh  dense A^T v (512-column tiles; large A)
 *   k_rows_tile_fused on A^T    ts_passes.cuh  dense A^T v of small A (PLAN_TRANS)
 *   k_rows_tile_fused           ts_passes.cuh  dense A v
 *   k_vec                       ts_passes.cuh  fused vector passes
 *   block_reduce, warp_reduce,  ts_common.cuh  fixed-order reductions
 *   reduce_partials
 *   EpiTaInitZero, EpiTaC, EpiTaV, EpiTaUpd, EpiTaBp, EpiFinalR,
 *   EpiFinalNR, EpiXNorm, ta_head, ta_decide   ts_state.cuh
 * Compile with -ffp-contract=off: every fused multiply-add here is an explicit
 * fma(), as on the device (the device code contracts nothing on this path).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NT 256
#define WARPS 8
#define MINBLK 4
#define TW 512 /* 2 columns per thread */
#define RU 12 /* kTileTRows: rows in flight per thread in k_cols_tile */
#define TBLK_T 3 /* kTileTBlocks */
#define TBLK_N 2 /* kTileNBlocks */

enum { RED_SUM = 0, RED_MIN = 1 };

static double red_combine(int op, double a, double b) { return op == RED_MIN ? (b < a ? b : a) : a + b; }
static double red_identity(int op) { return op == RED_MIN ? INFINITY : 0.0; }
static double py_max(double a, double b) { return b > a ? b : a; }
static double py_min(double a, double b) { return b < a ? b : a; }

/* xor-butterfly over 32 lanes; returns lane 0's value (every lane ends equal) */
static double warp_reduce(const double* v, int op) {
  double a[32], t[32];
  memcpy(a, v, sizeof(a));
  for (int o = 16; o > 0; o >>= 1) {
    for (int l = 0; l < 32; ++l) t[l] = red_combine(op, a[l], a[l ^ o]);
    memcpy(a, t, sizeof(a));
  }
  return a[0];
}

/* block_reduce of NT thread values (slot k): result of thread 0 */
static double block_reduce1(const double* v, int op) {
  double w[WARPS];
  for (int j = 0; j < WARPS; ++j) w[j] = warp_reduce(v + 32 * j, op);
  double s = w[0];
  for (int j = 1; j < WARPS; ++j) s = red_combine(op, s, w[j]);
  return s;
}

#define KMAX 3
typedef struct {
  int K;
  int op[KMAX];
} Ops;

/* reduce_partials over nb blocks (+ optional fix partials) */
static void reduce_partials(const double* bacc, const double* facc, int nb, const Ops* ops, double* out) {
  double* tv = (double*)malloc(sizeof(double) * NT);
  for (int k = 0; k < ops->K; ++k) {
    for (int t = 0; t < NT; ++t) {
      double o = red_identity(ops->op[k]);
      for (int b = t; b < nb; b += NT) {
        double v = bacc[(size_t)b * KMAX + k];
        if (facc) v = red_combine(ops->op[k], v, facc[(size_t)b * KMAX + k]);
        o = red_combine(ops->op[k], o, v);
      }
      tv[t] = o;
    }
    out[k] = block_reduce1(tv, ops->op[k]);
  }
  free(tv);
}

static int64_t blk_of(int64_t p, int64_t E, int64_t P) { return ((p + 1) * P + E - 1) / E - 1; }

/* ------------------------------------------------------------ geometry -- */
typedef struct {
  int sms;
  int64_t m, n;
} Geo;
static int64_t resident(const Geo* g) { return (int64_t)g->sms * MINBLK; }
static int tile_grid(const Geo* g, int per_sm, int min_rows) {
  const int64_t nct = (g->n + TW - 1) / TW, U = nct * g->m;
  int64_t p = U / min_rows; /* kTileMinRowsN = 8 (A v), kTileMinRowsT = 32 (A^T v) */
  if (p > (int64_t)g->sms * per_sm) p = (int64_t)g->sms * per_sm;
  if (p < 1) p = 1;
  return (int)p;
}
static int combine_grid(const Geo* g) {
  int64_t p = (g->m + WARPS - 1) / WARPS;
  if (p > resident(g)) p = resident(g);
  if (p < 1) p = 1;
  return (int)p;
}
static int vec_grid(const Geo* g, int64_t len) {
  int64_t p = (len + NT * 4 - 1) / (NT * 4);
  if (p > resident(g)) p = resident(g);
  if (p < 1) p = 1;
  return (int)p;
}

/* ------------------------------------------------------------ state ----- */
enum { RUNNING = 0, APPROX = 1, NORMAL_EQ = 2, ITER_CAP = 7, NUMFAIL = 8 };
enum { EV_NONE = 0, EV_PIVOT = 1, EV_EXPAND = 2 };
typedef struct {
  int status, event, maint, since_reval;
  int64_t iterations, max_iters;
  double eps, eps_prime, rho, rho_cap, b_norm, gap_norm, gap_dot_b, c_norm, scale, alpha, x_min;
  double residual_norm, normal_residual_norm, x_norm;
  double* trace; /* rows of 5: iter, tag, rho, gap_norm, c_norm */
  int64_t trace_rows, trace_cap;
} St;

static void trace_row(St* s, int tag) {
  if (s->trace_rows < s->trace_cap) {
    double* r = s->trace + 5 * s->trace_rows;
    r[0] = (double)s->iterations;
    r[1] = tag;
    r[2] = s->rho;
    r[3] = s->gap_norm;
    r[4] = s->c_norm;
  }
  s->trace_rows += 1;
}

static void ta_head(St* s) { /* triangle.py:210-218 */
  if (s->status != RUNNING) return;
  if (s->iterations >= s->max_iters) {
    s->status = ITER_CAP;
    return;
  }
  if (!isfinite(s->gap_norm)) {
    s->status = NUMFAIL;
    return;
  }
  if (s->gap_norm <= s->eps) s->status = APPROX;
}

static void ta_decide(St* s, double c2) { /* adaptive branch of ta_decide */
  const double c_norm = sqrt(c2);
  s->c_norm = c_norm;
  s->event = EV_NONE;
  const double gb = s->gap_dot_b;
  if (c_norm <= s->eps_prime) {
    s->status = NORMAL_EQ;
    return;
  }
  if (s->rho > 0.0 && s->rho * c_norm >= gb) {
    s->scale = s->rho / c_norm;
    s->event = EV_PIVOT;
    return;
  }
  s->rho = py_max(2.0 * s->rho, gb / c_norm);
  trace_row(s, 1);
  s->event = EV_EXPAND;
  if (s->rho > s->rho_cap) {
    s->status = ITER_CAP;
    s->iterations += 1;
    return;
  }
  s->iterations += 1;
  ta_head(s);
}

/* ------------------------------------------------------------ passes ---- */
/* epilogue callbacks: elem(ctx, i, y, acc[KMAX]) */
typedef void (*ElemFn)(void* ctx, int64_t i, double y, double* acc);

typedef struct {
  const double* a;
  int64_t lda;
  double* aT; /* PLAN_TRANS (small matrices): n x m transposed copy, else NULL */
  Geo g;
  int P_t, P_n, P_c;
  int64_t nct;
  double* part;  /* nct * m */
  double* tpart; /* P_t * 2 * TW */
  double* bacc;  /* P * KMAX */
  double* facc;
} Dev;

/* one (tile, row-range) segment of k_cols_tile for thread t: column sums */
static int64_t cols_seg(const Dev* D, const double* x, double xs, int use_xs, int64_t ct, int64_t r0,
                        int64_t r1, int t, double sv[2]) {
  const int64_t n = D->g.n, lda = D->lda;
  const int64_t c = ct * TW + 2 * t;
  const int64_t nv = n - c < 2 ? (n - c > 0 ? n - c : 0) : 2;
  double ac[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  int64_t r = r0;
  if (nv == 2) {
    for (; r + RU <= r1; r += RU) {
      for (int i = 0; i < RU; ++i) {
        const double xr = use_xs ? xs * x[r + i] : x[r + i];
        const double* row = D->a + (r + i) * lda + c;
        ac[i & 1][0] = fma(row[0], xr, ac[i & 1][0]);
        ac[i & 1][1] = fma(row[1], xr, ac[i & 1][1]);
      }
    }
    for (; r < r1; ++r) {
      const double xr = use_xs ? xs * x[r] : x[r];
      const double* row = D->a + r * lda + c;
      ac[0][0] = fma(row[0], xr, ac[0][0]);
      ac[0][1] = fma(row[1], xr, ac[0][1]);
    }
  } else if (nv > 0) {
    for (; r < r1; ++r) {
      const double xr = use_xs ? xs * x[r] : x[r];
      const double* row = D->a + r * lda + c;
      for (int j = 0; j < nv; ++j) ac[0][j] = fma(row[j], xr, ac[0][j]);
    }
  }
  sv[0] = ac[0][0] + ac[1][0];
  sv[1] = ac[0][1] + ac[1][1];
  return nv;
}

/* k_cols_tile<Epi, 2>: y = A^T x (x on the m side), epilogue per column */
static void rows_pass(Dev* D, const double* a, int64_t lda, int64_t m, int64_t n, const double* x,
                      double xs, int use_xs, const Ops* ops, ElemFn elem, void* ctx, double* red);
static void pass_T(Dev* D, const double* x, double xs, int use_xs, const Ops* ops, ElemFn elem, void* ctx,
                   double* red) {
  if (D->aT) { /* PLAN_TRANS: the fused row-tile pass over the transposed copy */
    rows_pass(D, D->aT, D->g.m, D->g.n, D->g.m, x, xs, use_xs, ops, elem, ctx, red);
    return;
  }
  const int64_t m = D->g.m, n = D->g.n;
  const int64_t nct = (n + TW - 1) / TW, U = nct * m;
  const int P = D->P_t;
  const int K = ops->K;
  double* acc = (double*)malloc(sizeof(double) * NT * KMAX);
  double tv[NT];
  for (int b = 0; b < P; ++b) {
    const int64_t U0 = U * b / P, U1 = U * (b + 1) / P;
    for (int t = 0; t < NT; ++t)
      for (int k = 0; k < K; ++k) acc[t * KMAX + k] = red_identity(ops->op[k]);
    int64_t ct_first = -1;
    for (int64_t u = U0; u < U1;) {
      const int64_t ct = u / m, r0 = u - ct * m;
      const int64_t r1 = (m < r0 + (U1 - u)) ? m : r0 + (U1 - u);
      const int full_tile = (r0 == 0 && r1 == m);
      const int which = (r0 > 0) ? 0 : 1;  /* 0: the tile began in an earlier block */
      for (int t = 0; t < NT; ++t) {
        double sv[2];
        const int64_t nv = cols_seg(D, x, xs, use_xs, ct, r0, r1, t, sv);
        const int64_t c = ct * TW + 2 * t;
        if (full_tile) {
          for (int j = 0; j < 2; ++j)
            if (j < nv) elem(ctx, c + j, sv[j], acc + t * KMAX);
        } else {
          double* dst = D->tpart + ((size_t)b * 2 + which) * TW + 2 * t;
          dst[0] = sv[0];
          dst[1] = sv[1];
        }
      }
      if (!full_tile && which == 0) ct_first = ct;
      u += r1 - r0;
    }
    const int end_block = (ct_first >= 0 && ct_first * m + m <= U1);
    for (int k = 0; k < K; ++k) {
      for (int t = 0; t < NT; ++t) tv[t] = acc[t * KMAX + k];
      D->bacc[(size_t)b * KMAX + k] = block_reduce1(tv, ops->op[k]);
      if (!end_block) D->facc[(size_t)b * KMAX + k] = red_identity(ops->op[k]);
    }
  }
  /* split-tile merges (whichever block arrives last, the pieces are added in
     block order): result into facc[bb] */
  for (int64_t ct = 0; ct < nct; ++ct) {
    const int64_t ba = blk_of(ct * m, U, P), bb = blk_of(ct * m + m - 1, U, P);
    if (ba == bb) continue; /* the whole tile inside one block */
    for (int t = 0; t < NT; ++t) {
      const int64_t c = ct * TW + 2 * t;
      double y[2];
      for (int j = 0; j < 2; ++j) y[j] = D->tpart[((size_t)ba * 2 + 1) * TW + 2 * t + j];
      for (int64_t q = ba + 1; q <= bb; ++q)
        for (int j = 0; j < 2; ++j) y[j] += D->tpart[((size_t)q * 2) * TW + 2 * t + j];
      for (int k = 0; k < K; ++k) acc[t * KMAX + k] = red_identity(ops->op[k]);
      for (int j = 0; j < 2; ++j)
        if (c + j < n) elem(ctx, c + j, y[j], acc + t * KMAX);
    }
    for (int k = 0; k < K; ++k) {
      for (int t = 0; t < NT; ++t) tv[t] = acc[t * KMAX + k];
      D->facc[(size_t)bb * KMAX + k] = block_reduce1(tv, ops->op[k]);
    }
  }
  free(acc);
  reduce_partials(D->bacc, D->facc, P, ops, red);
}

/* k_rows_wdense (small, L2-resident dense; ts_passes.cuh wdense_fits): one warp
 * per row; lane l owns columns 64 k + 2 l, 64 k + 2 l + 1, chunk k feeds FMA
 * chain k & 1, lanes are added by the xor butterfly; lane 0 of the warp runs
 * the epilogue; rows of block b are [m b / P, m (b + 1) / P), warp w takes
 * every 8th of them; block partials are reduced in block order. */
static int wdense_fits(int64_t m, int64_t n) {
  return n >= 128 && n <= 4096 && m >= 1 && 8 * m * n <= (32ll << 20);
}
static void rows_pass_warp(Dev* D, const double* a, int64_t lda, int64_t m, int64_t n, const double* x,
                           double xs, int use_xs, const Ops* ops, ElemFn elem, void* ctx, double* red) {
  const int K = ops->K;
  Geo g = D->g;
  g.m = m;
  g.n = n;
  int64_t P = (m + WARPS - 1) / WARPS;
  if (P > resident(&g)) P = resident(&g);
  if (P < 1) P = 1;
  double* xv = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t c = 0; c < n; ++c) xv[c] = use_xs ? xs * x[c] : x[c];
  for (int64_t b = 0; b < P; ++b) {
    const int64_t r0 = m * b / P, r1 = m * (b + 1) / P;
    double tv[KMAX][NT];
    for (int k = 0; k < K; ++k)
      for (int t = 0; t < NT; ++t) tv[k][t] = red_identity(ops->op[k]);
    for (int w = 0; w < WARPS; ++w) {
      double acc[KMAX];
      for (int k = 0; k < K; ++k) acc[k] = red_identity(ops->op[k]);
      for (int64_t r = r0 + w; r < r1; r += WARPS) {
        const double* row = a + r * lda;
        double lane[32];
        for (int l = 0; l < 32; ++l) {
          double a0 = 0.0, a1 = 0.0;
          for (int64_t c0 = 0; c0 < n; c0 += 64 * 16)
            for (int k = 0; k < 16; k += 2) {
              const int64_t ca = c0 + 64 * k + 2 * l, cb = ca + 64;
              if (ca < n) a0 = fma(row[ca], xv[ca], a0);
              if (ca + 1 < n) a0 = fma(row[ca + 1], xv[ca + 1], a0);
              if (cb < n) a1 = fma(row[cb], xv[cb], a1);
              if (cb + 1 < n) a1 = fma(row[cb + 1], xv[cb + 1], a1);
            }
          lane[l] = a0 + a1;
        }
        elem(ctx, r, warp_reduce(lane, RED_SUM), acc);
      }
      for (int k = 0; k < K; ++k) tv[k][w * 32] = acc[k];
    }
    for (int k = 0; k < K; ++k) D->bacc[b * KMAX + k] = block_reduce1(tv[k], ops->op[k]);
  }
  free(xv);
  reduce_partials(D->bacc, NULL, (int)P, ops, red);
}

/* k_rows_tile_fused: y = A x (x on the n side, optional scale).  The
 * (row, tile) partials do not depend on which block computes them; the
 * combine runs per 256-row group: one thread per row sums its tile partials
 * in tile order, the group's block_reduce lands in slot g, and the slots are
 * reduced in group order. */
static void rows_pass(Dev* D, const double* a, int64_t lda, int64_t m, int64_t n, const double* x,
                      double xs, int use_xs, const Ops* ops, ElemFn elem, void* ctx, double* red) {
  if (wdense_fits(m, n)) {
    rows_pass_warp(D, a, lda, m, n, x, xs, use_xs, ops, elem, ctx, red);
    return;
  }
  const int64_t nct = (n + TW - 1) / TW;
  for (int64_t ct = 0; ct < nct; ++ct) {
    const int64_t cb = ct * TW;
    const int full = cb + TW <= n;
    double xv[32][8][2];
    for (int l = 0; l < 32; ++l)
      for (int k = 0; k < 8; ++k) {
        const int64_t c = cb + 64 * k + 2 * l;
        xv[l][k][0] = (c < n) ? (use_xs ? xs * x[c] : x[c]) : 0.0;
        xv[l][k][1] = (c + 1 < n) ? (use_xs ? xs * x[c + 1] : x[c + 1]) : 0.0;
      }
    for (int64_t r = 0; r < m; ++r) {
      const double* row = a + r * lda + cb;
      double lane[32];
      for (int l = 0; l < 32; ++l) {
        double a0 = 0.0, a1 = 0.0;
        if (full) {
          for (int k = 0; k < 8; k += 2) {
            a0 = fma(row[64 * k + 2 * l], xv[l][k][0], a0);
            a0 = fma(row[64 * k + 2 * l + 1], xv[l][k][1], a0);
            a1 = fma(row[64 * (k + 1) + 2 * l], xv[l][k + 1][0], a1);
            a1 = fma(row[64 * (k + 1) + 2 * l + 1], xv[l][k + 1][1], a1);
          }
        } else {
          for (int k = 0; k < 8; ++k) {
            const int64_t c = cb + 64 * k + 2 * l;
            if (c < n) a0 = fma(row[64 * k + 2 * l], xv[l][k][0], a0);
            if (c + 1 < n) a1 = fma(row[64 * k + 2 * l + 1], xv[l][k][1], a1);
          }
        }
        lane[l] = a0 + a1;
      }
      D->part[r * nct + ct] = warp_reduce(lane, RED_SUM);
    }
  }
  const int K = ops->K;
  const int64_t ng = (m + NT - 1) / NT;
  double* gacc = (double*)malloc(sizeof(double) * (size_t)ng * KMAX);
  for (int64_t g = 0; g < ng; ++g) {
    double tv[KMAX][NT];
    for (int t = 0; t < NT; ++t) {
      double acc[KMAX];
      for (int k = 0; k < K; ++k) acc[k] = red_identity(ops->op[k]);
      const int64_t r = g * NT + t;
      if (r < m) {
        const double* pr = D->part + r * nct;
        double y = pr[0];
        for (int64_t c = 1; c < nct; ++c) y += pr[c];
        elem(ctx, r, y, acc);
      }
      for (int k = 0; k < K; ++k) tv[k][t] = acc[k];
    }
    for (int k = 0; k < K; ++k) gacc[g * KMAX + k] = block_reduce1(tv[k], ops->op[k]);
  }
  reduce_partials(gacc, NULL, (int)ng, ops, red);
  free(gacc);
}

static void pass_N(Dev* D, const double* x, double xs, int use_xs, const Ops* ops, ElemFn elem, void* ctx,
                   double* red) {
  rows_pass(D, D->a, D->lda, D->g.m, D->g.n, x, xs, use_xs, ops, elem, ctx, red);
}

/* k_vec: elem(ctx, i, 0, acc) over [0, len) */
static void pass_vec(Dev* D, int64_t len, const Ops* ops, ElemFn elem, void* ctx, double* red) {
  const int P = vec_grid(&D->g, len);
  const int64_t stride = (int64_t)P * NT;
  const int K = ops->K;
  double tv[NT];
  double* acc = (double*)malloc(sizeof(double) * NT * KMAX);
  for (int b = 0; b < P; ++b) {
    for (int t = 0; t < NT; ++t) {
      for (int k = 0; k < K; ++k) acc[t * KMAX + k] = red_identity(ops->op[k]);
      for (int64_t i = (int64_t)b * NT + t; i < len; i += stride) elem(ctx, i, 0.0, acc + t * KMAX);
    }
    for (int k = 0; k < K; ++k) {
      for (int t = 0; t < NT; ++t) tv[t] = acc[t * KMAX + k];
      D->bacc[(size_t)b * KMAX + k] = block_reduce1(tv, ops->op[k]);
    }
  }
  free(acc);
  reduce_partials(D->bacc, NULL, P, ops, red);
}

/* ------------------------------------------------------------ epilogues -- */
typedef struct {
  int64_t m, n;
  const double* b;
  double *bp, *gap, *d, *x, *c, *fr;
  double al, scale;
} Ctx;

static void e_init(void* p, int64_t i, double y, double* acc) { /* EpiTaInitZero */
  Ctx* C = (Ctx*)p;
  (void)y;
  if (i < C->m) {
    const double bi = C->b[i];
    const double g = bi - 0.0;
    C->bp[i] = 0.0;
    C->gap[i] = g;
    acc[0] = fma(g, g, acc[0]);
    acc[1] = fma(g, bi, acc[1]);
    acc[2] = fma(bi, bi, acc[2]);
  }
  if (i < C->n) C->x[i] = 0.0;
}
static void e_c(void* p, int64_t i, double y, double* acc) { /* EpiTaC */
  Ctx* C = (Ctx*)p;
  C->c[i] = y;
  acc[0] = fma(y, y, acc[0]);
  const double cp = (y >= 0.0 || y != y) ? y : 0.0;
  acc[1] = fma(cp, cp, acc[1]);
}
static void e_v(void* p, int64_t i, double y, double* acc) { /* EpiTaV */
  Ctx* C = (Ctx*)p;
  const double di = y - C->bp[i];
  C->d[i] = di;
  acc[0] = fma(di, di, acc[0]);
  acc[1] = fma(C->gap[i], di, acc[1]);
}
static void e_upd(void* p, int64_t i, double y, double* acc) { /* EpiTaUpd (adaptive) */
  Ctx* C = (Ctx*)p;
  (void)y;
  const double al = C->al;
  if (i < C->m) {
    const double nb = C->bp[i] + al * C->d[i];
    const double bi = C->b[i];
    const double g = bi - nb;
    C->bp[i] = nb;
    C->gap[i] = g;
    acc[0] = fma(g, g, acc[0]);
    acc[1] = fma(g, bi, acc[1]);
  }
  if (i < C->n) {
    const double pre = C->scale * C->c[i];
    const double nx = (1.0 - al) * C->x[i] + al * pre;
    C->x[i] = nx;
    acc[2] = py_min(acc[2], nx);
  }
}
static void e_bp(void* p, int64_t i, double y, double* acc) { /* EpiTaBp */
  Ctx* C = (Ctx*)p;
  const double bi = C->b[i];
  const double g = bi - y;
  C->bp[i] = y;
  C->gap[i] = g;
  acc[0] = fma(g, g, acc[0]);
  acc[1] = fma(g, bi, acc[1]);
  acc[2] = fma(bi, bi, acc[2]);
}
static void e_fr(void* p, int64_t i, double y, double* acc) { /* EpiFinalR */
  Ctx* C = (Ctx*)p;
  const double f = C->b[i] - y;
  C->fr[i] = f;
  acc[0] = fma(f, f, acc[0]);
}
static void e_sq(void* p, int64_t i, double y, double* acc) { /* EpiFinalNR */
  (void)p;
  (void)i;
  acc[0] = fma(y, y, acc[0]);
}
static void e_xn(void* p, int64_t i, double y, double* acc) { /* EpiXNorm */
  Ctx* C = (Ctx*)p;
  (void)y;
  acc[0] = fma(C->x[i], C->x[i], acc[0]);
}

/* ------------------------------------------------------------ driver ---- */
/* out[0..7]: status, iterations, residual_norm, normal_residual_norm, rho,
   x_norm, gap_norm, c_norm.  trace: trace_cap rows of (iter, tag, rho,
   gap_norm, c_norm), tag 0 pivot / 1 expand.  Returns trace rows produced. */
int64_t ts_mirror_ta_dense(const double* a, int64_t m, int64_t n, const double* b, double eps,
                           int64_t max_iters, int sms, double* x_out, double* trace, int64_t trace_cap,
                           double* out) {
  Dev D;
  memset(&D, 0, sizeof(D));
  D.g.sms = sms;
  D.g.m = m;
  D.g.n = n;
  D.a = a;
  D.lda = n;
  D.P_t = tile_grid(&D.g, TBLK_T, 32);
  D.P_n = tile_grid(&D.g, TBLK_N, 8);
  D.P_c = combine_grid(&D.g);
  D.nct = (n + TW - 1) / TW;
  const int64_t pmax = (int64_t)sms * 8 + 8;
  /* the library's PLAN_TRANS rule (ts_lib.cu, kTransBytes in ts_matrix.cuh) */
  if (m >= 128 && n >= 128 && 8 * m * n <= (32ll << 20)) {
    D.aT = (double*)malloc(sizeof(double) * (size_t)(m * n));
    for (int64_t r = 0; r < m; ++r)
      for (int64_t c = 0; c < n; ++c) D.aT[c * m + r] = a[r * n + c];
  }
  const int64_t nctT = (m + TW - 1) / TW;
  D.part = (double*)calloc((size_t)(D.nct * m > nctT * n ? D.nct * m : nctT * n), sizeof(double));
  D.tpart = (double*)calloc((size_t)pmax * 2 * TW, sizeof(double));
  D.bacc = (double*)calloc((size_t)pmax * KMAX, sizeof(double));
  D.facc = (double*)calloc((size_t)pmax * KMAX, sizeof(double));
  Ctx C;
  memset(&C, 0, sizeof(C));
  C.m = m;
  C.n = n;
  C.b = b;
  C.bp = (double*)calloc((size_t)m, sizeof(double));
  C.gap = (double*)calloc((size_t)m, sizeof(double));
  C.d = (double*)calloc((size_t)m, sizeof(double));
  C.fr = (double*)calloc((size_t)m, sizeof(double));
  C.x = (double*)calloc((size_t)n, sizeof(double));
  C.c = (double*)calloc((size_t)n, sizeof(double));
  St s;
  memset(&s, 0, sizeof(s));
  s.status = RUNNING;
  s.max_iters = max_iters;
  s.eps = eps;
  s.eps_prime = -1.0;
  s.rho_cap = -1.0;
  s.trace = trace;
  s.trace_cap = trace_cap;
  double red[KMAX];
  const Ops o3 = {3, {RED_SUM, RED_SUM, RED_SUM}};
  const Ops o2 = {2, {RED_SUM, RED_SUM}};
  const Ops ou = {3, {RED_SUM, RED_SUM, RED_MIN}};
  const Ops o1 = {1, {RED_SUM}};
  const int64_t mx = m > n ? m : n;
  /* init (triangle.py:197-204) */
  pass_vec(&D, mx, &o3, e_init, &C, red);
  s.b_norm = sqrt(red[2]);
  s.gap_norm = sqrt(red[0]);
  s.gap_dot_b = red[1];
  s.x_min = 0.0;
  int trivial = 0;
  if (s.b_norm == 0.0) {
    trivial = 1;
    s.status = APPROX;
  } else {
    if (s.eps_prime < 0.0) s.eps_prime = s.eps;
    if (s.rho_cap < 0.0) s.rho_cap = 4.0 * (s.b_norm * s.b_norm) / s.eps_prime;
    ta_head(&s);
  }
  while (s.status == RUNNING) {
    if (s.since_reval >= 512) { /* b' = A x (triangle.py:239-242) */
      pass_N(&D, C.x, 0.0, 0, &o3, e_bp, &C, red);
      s.gap_norm = sqrt(red[0]);
      s.gap_dot_b = red[1];
      s.since_reval = 0;
      ta_head(&s);
      continue;
    }
    pass_T(&D, C.gap, 0.0, 0, &o2, e_c, &C, red);
    ta_decide(&s, red[0]);
    if (s.event != EV_PIVOT) continue;
    C.scale = s.scale;
    pass_N(&D, C.c, s.scale, 1, &o2, e_v, &C, red);
    if (red[0] == 0.0) {
      s.status = NUMFAIL;
      break;
    }
    s.alpha = py_min(1.0, py_max(0.0, red[1] / red[0]));
    C.al = s.alpha;
    pass_vec(&D, mx, &ou, e_upd, &C, red);
    trace_row(&s, 0);
    s.gap_norm = sqrt(red[0]);
    s.gap_dot_b = red[1];
    s.since_reval += 1;
    s.iterations += 1;
    if (s.since_reval < 512) ta_head(&s);
  }
  if (trivial) {
    memset(C.x, 0, sizeof(double) * (size_t)n);
  } else {
    pass_N(&D, C.x, 0.0, 0, &o1, e_fr, &C, red);
    s.residual_norm = sqrt(red[0]);
    pass_T(&D, C.fr, 0.0, 0, &o1, e_sq, &C, red);
    s.normal_residual_norm = sqrt(red[0]);
    pass_vec(&D, n, &o1, e_xn, &C, red);
    s.x_norm = sqrt(red[0]);
  }
  memcpy(x_out, C.x, sizeof(double) * (size_t)n);
  out[0] = s.status;
  out[1] = (double)s.iterations;
  out[2] = s.residual_norm;
  out[3] = s.normal_residual_norm;
  out[4] = s.rho;
  out[5] = s.x_norm;
  out[6] = s.gap_norm;
  out[7] = s.c_norm;
  free(D.part);
  free(D.aT);
  free(D.tpart);
  free(D.bacc);
  free(D.facc);
  free(C.bp);
  free(C.gap);
  free(C.d);
  free(C.fr);
  free(C.x);
  free(C.c);
  return s.trace_rows;
}
