/*
 * trisolve_b200 — C ABI of the B200-native TA / CTA / TA-LP iteration path.
 *
 * Plain pointers and sizes only; no torch types.  Every vector argument may
 * be a host pointer (pageable or pinned) or a device pointer on the
 * matrix's device: inputs are staged into library-owned device buffers and
 * outputs copied back with cudaMemcpyDefault (unified addressing), so the
 * caller never needs to say which it passed.  `stream` is a
 * cudaStream_t (NULL = legacy default stream).
 *
 * Return codes: 0 = OK; < 0 = invalid argument (the Python layer raises
 * ValueError with ts_last_error()); > 0 = CUDA / resource failure (raises
 * RuntimeError).  Numerical outcomes are never errors: they are the
 * `status` field of ts_result (1:1 with the reference's status strings,
 * reference pkg/src/trisolve/results.py:11-18).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/trisolve/):
 *   ts_matrix_create_dense / _csr   matrix storage for linalg.py:34-56 (ndarray / csr_array)
 *   ts_matvec                        linalg.matvec            linalg.py:34-42
 *   ts_rmatvec                       linalg.matvec_transpose  linalg.py:45-56
 *   ts_norm2 / ts_dot                linalg.norm2 / np.dot    linalg.py:59-61
 *   ts_matrix_info (frobenius)       linalg.frobenius_norm    linalg.py:64-69
 *   ts_gram_matvec                   GramProduct.matvec       linalg.py:93-114
 *   ts_moments                       centering.moments        centering.py:67-84
 *   ts_hankel_min_norm               centering.min_norm_coefficients centering.py:87-110
 *   ts_cta_solve                     centering.centering_solve centering.py:263-358
 *                                    (ts_cta_step_only => centering_step centering.py:216-224)
 *   ts_ta_adaptive                   triangle.solve_adaptive  triangle.py:170-251
 *   ts_ta_in_ball                    triangle.solve_in_ball   triangle.py:92-113 (+ _membership_loop 136-167)
 *   ts_lp_feasibility                feasibility.nonnegative_feasibility feasibility.py:59-140
 *   ts_mm_parse / _coo / _dense      mmio.read_matrix_market_with_info mmio.py:100-156
 *   ts_mm_to_device                  mmio coordinate read + csr_array(coo), assembled on the device
 */
#ifndef TRISOLVE_B200_H
#define TRISOLVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TS_API __attribute__((visibility("default")))
#else
#define TS_API
#endif

#define TS_ABI_VERSION 2

typedef struct ts_matrix ts_matrix; /* opaque; immutable after creation */
typedef struct ts_comm ts_comm;     /* column-sharding communicator (one per rank) */

/* ---- return codes -------------------------------------------------------- */
enum {
  TS_OK = 0,
  TS_EINVAL = -1,      /* contract violation (shape, option, b = 0, ...) */
  TS_EDEGENERATE = -2, /* "degenerate pivot" (triangle.py:77-78) */
  TS_ECUDA = 1,        /* CUDA runtime failure */
  TS_ENOMEM = 2
};

/* ---- terminal statuses (results.py:11-18) --------------------------------- */
enum {
  TS_RUNNING = 0,
  TS_APPROX_SOLUTION = 1,
  TS_NORMAL_EQ_SOLUTION = 2,
  TS_MIN_NORM_SOLUTION = 3,
  TS_WITNESS = 4,
  TS_FEASIBLE = 5,
  TS_INCONCLUSIVE = 6,
  TS_ITERATION_CAP = 7,
  TS_NUMERICAL_FAILURE = 8
};

/* ---- detail codes (the reference's `detail` strings) ---------------------- */
enum {
  TS_DETAIL_NONE = 0,
  TS_DETAIL_NONFINITE_RESIDUAL = 1, /* "non-finite residual"                       centering.py:299 */
  TS_DETAIL_MOMENT_SOLVE = 2,       /* "moment solve failed: ..."                  centering.py:315 */
  TS_DETAIL_NE_CERTIFIED_CTA = 3,   /* "certified ||A^T A x - A^T b|| <= %.3e"     centering.py:322 */
  TS_DETAIL_DRIFT = 4,              /* "residual drift exceeded budget"            centering.py:349 */
  TS_DETAIL_NONFINITE_ITERATE = 5,  /* "non-finite iterate"                        triangle.py:214 */
  TS_DETAIL_PIVOT_VANISHED = 6,     /* "pivot direction vanished"                  triangle.py:229 */
  TS_DETAIL_NE_CERTIFIED_TA = 7,    /* "certified ||A^T(b - Ax)|| <= %.3e"         triangle.py:230 */
  TS_DETAIL_RADIUS_CAP = 8,         /* "radius exceeded cap %.3e"                  triangle.py:247 */
  TS_DETAIL_CONE_STALL = 9,         /* "no ascent direction in the nonnegative cone section" feasibility.py:433 */
  TS_DETAIL_LEFT_CONE = 10,         /* "iterate left the nonnegative cone"         feasibility.py:447 */
  TS_DETAIL_RADIUS_BUDGET = 11,     /* "radius budget %.3e exhausted"              feasibility.py:460 */
  TS_DETAIL_ITER_BUDGET = 12,       /* "iteration budget exhausted"                feasibility.py:411 */
  TS_DETAIL_DEVICE_WATCHDOG = 13    /* device loop barrier watchdog (library-side; never expected) */
};

/* trace events (TA / LP `event` column) */
enum { TS_EVENT_PIVOT = 0, TS_EVENT_EXPAND = 1, TS_EVENT_WITNESS = 2 };

/* One trace row.  Column meaning per solver (results.py:97-101):
 *   CTA: tag = t;     v = {residual_norm, normal_residual_norm, 0, 0}
 *   TA : tag = event; v = {rho, gap_norm, normal_gap_norm, 0}
 *   LP : tag = event; v = {rho, gap_norm, normal_gap_norm, min_x_entry}
 * wall_ns is %globaltimer minus the solve's start stamp. */
typedef struct {
  int64_t iter;
  int64_t wall_ns;
  int32_t tag;
  int32_t reserved;
  double v[4];
} ts_trace_row;

typedef struct {
  int32_t status;
  int32_t detail;
  int64_t iterations;
  double residual_norm;        /* ||b - A x|| of the returned x */
  double normal_residual_norm; /* ||A^T (b - A x)|| */
  double rho;
  double lower_bound;          /* witness bound (in-ball / LP) */
  double min_x_entry;          /* LP */
  double detail_value;         /* number formatted into the detail string */
  int64_t trace_rows;          /* rows produced (may exceed the caller's capacity) */
  int32_t has_lower_bound;
  int32_t trivial;             /* 1: the b == 0 early return (no residual recompute) */
  double elapsed_ms;           /* device time of the solve loop (CUDA events) */
  int64_t kernel_launches;     /* kernels launched by the solve (incl. graph nodes) */
  /* live per-class kernel accounting inside the solve (%globaltimer, earliest
   * block start to last block's finisher): [0] A v passes, [1] A^T v passes,
   * [2] fused vector passes, [3] the CTA Hankel solves
   * (run by the finishing block of the last moments pass) */
  double kernel_ms[4];
  int64_t kernel_count[4];
  double gap_norm;             /* TA family: ||b - b'|| of the final iterate pair */
  double x_norm;               /* ||x|| of the returned iterate */
} ts_result;

typedef struct {
  double epsilon;      /* relative to ||b|| (centering.py:128-131) */
  int32_t t_max;
  int32_t h_mode;      /* 0 = "aat" (Gram), 1 = "a" (symmetric) */
  int64_t max_iters;
  int32_t enhanced;
  int32_t known_solvable;
  int64_t recheck_every;
  double rcond;
  int32_t accelerate;
  int32_t accel_patience;
  double accel_ratio;
  const double* x_start; /* NULL: start = "zero"; else the random start vector (n) */
  /* 1: the operator is the implicit normal matrix A^T A (n x n) of the handle
   * (the reference's GramProduct, linalg.py:93-114): every operator apply is
   * the pass pair A^T (A v); b, x and the Krylov vectors live in n-space. */
  int32_t normal_operand;
  int32_t reserved;
} ts_cta_options;

typedef struct {
  double eps;
  double eps_prime;    /* < 0: default = eps */
  double rho_cap;      /* < 0: default = 4 ||b||^2 / eps_prime */
  int64_t max_iters;
  int32_t restart_halvings;
  int32_t gram;        /* 1: operate on the implicit pair (A^T A, b) (GramProduct, linalg.py:93-114) */
  const double* x0;    /* optional warm start (n) */
} ts_ta_options;

typedef struct {
  double rho;
  double eps;
  double eps_prime;    /* < 0: default = eps */
  int64_t max_iters;
  const double* x0;    /* optional warm start, used only if ||x0|| <= rho (1 + 1e-9) */
  int32_t gram;
  int32_t reserved;
} ts_ball_options;

typedef struct {
  double eps;
  double rho_max;      /* < 0: default_rho_max (feasibility.py:49-56) */
  int64_t max_iters;
  int32_t gram;
  int32_t reserved;
} ts_lp_options;

/* ---- library ------------------------------------------------------------- */
TS_API int ts_abi_version(void);
TS_API const char* ts_last_error(void); /* thread-local message of the last failing call */
TS_API int ts_device_count(int* count);

/* ---- matrices ------------------------------------------------------------ */
/* Row-major dense m x n with leading dimension lda (>= n), fp64. */
TS_API int ts_matrix_create_dense(const double* a, int64_t m, int64_t n, int64_t lda, int device,
                           void* stream, ts_matrix** out);
/* CSR (int32 indptr/indices, fp64 data); duplicates must already be summed.
 * A transposed CSR copy (= CSC of A) is built on the device so that A^T v is a
 * deterministic gather with no atomics. */
TS_API int ts_matrix_create_csr(const int32_t* indptr, const int32_t* indices, const double* data,
                         int64_t m, int64_t n, int64_t nnz, int device, void* stream,
                         ts_matrix** out);
TS_API int ts_matrix_destroy(ts_matrix* a);
/* kind: 0 dense, 1 csr.  frobenius: ||A||_F computed once at creation. */
TS_API int ts_matrix_info(const ts_matrix* a, int64_t* m, int64_t* n, int64_t* nnz, int32_t* kind,
                   double* frobenius);
/* The launch plans chosen for the handle's two passes (diagnostics / tests):
 * 0 flat split, 1 thread per row, 2 dense tiles, 7 warp per row, 9 dense
 * transposed copy, 10 sliced ELL, 11 column slabs. */
TS_API int ts_matrix_plans(const ts_matrix* a, int32_t* plan_av, int32_t* plan_atv);

/* ---- storage pools --------------------------------------------------------
 * ts_matrix_destroy retires an unsharded handle (device storage, launch plans,
 * cached solver instances and their instantiated graphs) into a small
 * per-process pool; creating a matrix of the same kind and shape on the same
 * device recycles it, uploading the new entries into the same buffers
 * (TS_MATRIX_POOL=0 disables).  ts_pool_trim releases retired storage on
 * `device` (< 0: every device) and the cached pinned host blocks. */
TS_API int ts_pool_trim(int device);
/* Page-locked host blocks for solver outputs, cached by size after ts_host_free. */
TS_API int ts_host_alloc(size_t bytes, void** out);
TS_API int ts_host_free(void* ptr);

/* ---- Matrix Market ingest (reference mmio.py:41-156) ------------------------
 * ts_mm_parse reads a file (is_path = 1: `data` is a NUL-terminated path) or an
 * in-memory image (`data`, `len`) with the reference's acceptance rules; a
 * malformed input returns TS_EINVAL with ts_last_error() = "line N: ..."
 * (the reference's MatrixMarketError text).  ts_mm_coo returns the
 * coordinate entries expanded as the reference stores them (each entry, then
 * its mirror for symmetric / skew-symmetric files; `stored` of them);
 * ts_mm_dense the m x n row-major array of an array file.  ts_mm_to_device
 * builds a CSR handle from a coordinate file with the assembly (mirroring,
 * sort, duplicate summation in file order, compression) on the device. */
typedef struct ts_mm ts_mm;
typedef struct {
  int32_t format;   /* 0 coordinate, 1 array */
  int32_t field;    /* 0 real, 1 integer, 2 pattern */
  int32_t symmetry; /* 0 general, 1 symmetric, 2 skew-symmetric */
  int32_t reserved;
  int64_t rows, cols;
  int64_t entries; /* as stated in the size line (array: rows * cols) */
  int64_t stored;  /* coordinate: expanded entries; array: values in the file */
} ts_mm_info;
TS_API int ts_mm_parse(const char* data, int64_t len, int32_t is_path, ts_mm** out, ts_mm_info* info);
TS_API int ts_mm_coo(const ts_mm* mm, int32_t* rows, int32_t* cols, double* vals);
TS_API int ts_mm_dense(const ts_mm* mm, double* rowmajor);
TS_API int ts_mm_to_device(const ts_mm* mm, int device, void* stream, ts_matrix** out,
                           int64_t* duplicates);
TS_API int ts_mm_free(ts_mm* mm);

/* ---- device gallery (reference gallery.py:64-71, 118-191) -------------------
 * The 5-point stencil families (poisson Dirichlet / Neumann, convdiff) and
 * Clement generated straight into a device CSR handle.  Stencil coefficients
 * are passed in (computed by the caller with the reference's expressions);
 * center_mode = 1 puts the neighbour count on the diagonal (Neumann). */
TS_API int ts_matrix_gen_stencil5(int64_t grid, double center, double west, double east, double south,
                                  double north, int32_t center_mode, int device, void* stream,
                                  ts_matrix** out);
TS_API int ts_matrix_gen_clement(int64_t n, int device, void* stream, ts_matrix** out);

/* ---- operator layer -------------------------------------------------------- */
TS_API int ts_matvec(const ts_matrix* a, const double* x, double* y, void* stream);   /* y = A x  */
TS_API int ts_rmatvec(const ts_matrix* a, const double* x, double* y, void* stream);  /* y = A^T x */
TS_API int ts_gram_matvec(const ts_matrix* a, const double* x, double* y, void* stream); /* y = A^T (A x) */
TS_API int ts_norm2(const double* v, int64_t len, double* out, void* stream);
/* r = b - A x (r_out optional), ||r||, and ||A^T r|| (atr_norm optional):
 * the honest-residual step of every driver (triangle.py:84-89, hybrid.py:102-104) */
TS_API int ts_residual(const ts_matrix* a, const double* x, const double* b, double* r_out,
                       double* r_norm, double* atr_norm, void* stream);
/* ts_residual for the implicit normal operator G = A^T A of the handle (the
 * reference's GramProduct): r = b - G x (n), ||r||, ||G r||. */
TS_API int ts_gram_residual(const ts_matrix* a, const double* x, const double* b, double* r_out,
                            double* r_norm, double* gr_norm, void* stream);
TS_API int ts_dot(const double* u, const double* v, int64_t len, double* out, void* stream);

/* ---- CTA pieces ------------------------------------------------------------ */
/* phi[0..2t) = r^T H^k r; krylov (optional, (t+1) x m) = p_0..p_t;
 * transposed (optional, t x n, Gram mode only) = q_1..q_t. */
TS_API int ts_moments(const ts_matrix* a, int32_t h_mode, const double* r, int32_t t, double* phi,
               double* krylov, double* transposed, void* stream);
/* Equilibrated min-norm Hankel solve of the given order from phi (2*t entries). */
TS_API int ts_hankel_min_norm(const double* phi, int32_t t, int32_t order, double rcond, double* alpha,
                       void* stream);
/* One order-t step (centering_step): x_out/r_out (may alias x/r).  *status_out
 * = TS_NORMAL_EQ_SOLUTION when H r == 0 (NormalEquationReached). */
TS_API int ts_cta_step(const ts_matrix* a, int32_t h_mode, const double* x, const double* r, int32_t t,
                double rcond, double* x_out, double* r_out, int32_t* order_out,
                double* atr_norm_out, int32_t* status_out, void* stream);

/* Events-timed back-to-back launches of one matvec pass (A v or A^T v) on
 * device-resident vectors: average milliseconds per launch (kernel tuning and
 * the bench's cross-check of the in-solve kernel timers). */
TS_API int ts_time_pass(const ts_matrix* a, int32_t trans, int32_t reps, double* avg_ms, void* stream);

/* ---- column sharding over NVLink (BASELINE north_star) ---------
 * One process per GPU.  Each rank creates a communicator, exports 128 bytes of
 * IPC handles, all-gathers them (e.g. torch.distributed), connects, and
 * attaches it to its column block A_p = A[:, off:off+n_p] (a normal matrix
 * handle).  Solves on the attached handle then exchange one fixed-rank-order
 * all-reduce of the m-vector A_p v_p per A-pass (fused into the pass
 * epilogue, deterministic, identical on every rank) and one scalar
 * all-reduce per n-space reduction.  b, b', r, gap, Krylov vectors are
 * replicated; x, x0, x_start, c are the rank's LOCAL column slice. */
TS_API int ts_comm_create(int device, int rank, int world, int64_t vec_capacity, ts_comm** out,
                          void* ipc_handles_out /* 128 bytes */);
TS_API int ts_comm_connect(ts_comm* comm, const void* all_handles /* world x 128 bytes */);
TS_API int ts_comm_destroy(ts_comm* comm);
TS_API int ts_matrix_set_shard(ts_matrix* a, ts_comm* comm, int64_t n_global, int64_t col_offset,
                               double frobenius_global);
/* Row-block sharding of a square matrix (C4-like banded operators): rank p
 * owns rows AND columns [off, off + m).  The handle holds the rank's rows of A
 * and its columns of A (as rows of A^T), indices local to the block (j - off),
 * reaching at most `halo` entries past either end.  Every vector of a solve on
 * it is the rank's block (b, x, r, ...); before each pass a halo exchange
 * copies the neighbours' boundary entries over NVLink, and every reduction is
 * summed over ranks in rank order.  Bitwise identical operator results to the
 * unsharded path (each row / column is still added in the reference's order). */
TS_API int ts_matrix_create_csr_pair(const int32_t* indptr, const int32_t* indices, const double* data,
                                     int64_t nnz, const int32_t* indptr_t, const int32_t* indices_t,
                                     const double* data_t, int64_t nnz_t, int64_t m, int64_t halo,
                                     int device, void* stream, ts_matrix** out);
TS_API int ts_matrix_set_row_shard(ts_matrix* a, ts_comm* comm, int64_t n_global, int64_t row_offset,
                                   double frobenius_global);
/* Row-block sharding of a tall matrix (m >> n; north_star "tall matrices are
 * row-sharded symmetrically"): rank p owns rows [off, off + m_p) of A with
 * all n columns (a normal matrix handle).  The mirror image of column
 * sharding: x, x0, c and the Krylov q-vectors are replicated; b, b', r, gap
 * and the p-vectors are the rank's row block; A v is local, A^T v sums an
 * n-vector over ranks in rank order (fused, deterministic), every m-space
 * reduction is summed over ranks.  Replaces the unsharded linalg.py:45-56
 * A^T r of every solver for this layout. */
TS_API int ts_matrix_set_tall_shard(ts_matrix* a, ts_comm* comm, int64_t m_global, int64_t row_offset,
                                    double frobenius_global);
/* In-process world: `world` communicators of ONE process (out receives
 * `world` handles, rank order), rank r on devices[r] (devices NULL: every rank
 * on `device`, an emulated world that runs the sharded device code at world
 * > 1 on a single GPU).  Ranks on different GPUs read each other's slots over
 * NVLink (peer access is enabled).  Each rank's solves run on their own host
 * thread; every exchange is ordered on the host between the producer and the
 * consumer kernels (events) instead of spinning on device flags, so ranks may
 * share a GPU.  Results are bit-identical to a world of the same size with one
 * process per GPU. */
TS_API int ts_comm_create_local(int device, int world, int64_t vec_capacity, const int32_t* devices,
                                ts_comm** out);

/* ---- solvers --------------------------------------------------------------- */
TS_API int ts_cta_solve(const ts_matrix* a, const double* b, const ts_cta_options* opts, double* x_out,
                 ts_trace_row* trace, int64_t trace_cap, ts_result* res, void* stream);
TS_API int ts_ta_adaptive(const ts_matrix* a, const double* b, const ts_ta_options* opts,
                   double* x_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                   void* stream);
TS_API int ts_ta_in_ball(const ts_matrix* a, const double* b, const ts_ball_options* opts, double* x_out,
                  double* b_prime_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                  void* stream);
TS_API int ts_lp_feasibility(const ts_matrix* a, const double* b, const ts_lp_options* opts,
                      double* x_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TRISOLVE_B200_H */
