// Matrix handles (ts_matrix) and launch plans.
//
// HBM layout:
//   dense  row-major fp64, leading dimension padded to a multiple of 16
//          doubles (128 B) for n >= 64 (even otherwise) so every row starts
//          on a 128-byte line and every double2 load is aligned.
//   CSR    int32 row pointers, int32 column indices, fp64 values (A v).
//   CSR^T  the transposed CSR (= CSC of A), built on the device once by a
//          stable radix sort on the column index, so A^T v is a per-column
//          gather in ascending row order (the reference's `v @ csr` scatter
//          order, linalg.py:55) with no atomics.
//
// Each orientation gets a RowPlan: which kernel (flat split or thread-per-row)
// and, for the flat split, the first row touched by every warp.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cstdlib>
#include <mutex>

#include "ts_passes.cuh"

namespace ts {

// PLAN_FLAT   CSR rows with >= 32 entries on average, irregular lengths (k_rows_flat)
// PLAN_SHORT  thread per row, L2-resident (k_rows_short; dense n < 128 too)
// PLAN_TILE   dense A v (k_rows_tile_fused) / dense A^T v (k_cols_tile)
// PLAN_WROW   long CSR rows of near-uniform length (k_rows_wrow)
// PLAN_TRANS  small dense A^T v over a transposed copy (k_rows_tile_fused)
// PLAN_SELL   short CSR rows, HBM-sized: sliced-ELL copy (k_rows_sell)
// PLAN_SLAB   long CSR rows of a wide matrix: column slabs (k_slab_av + k_slab_combine)
// PLAN_NCOLS  large dense A v as column tiles over a transposed copy (k_cols_tile)
enum PlanKind : int { PLAN_FLAT = 0, PLAN_SHORT = 1, PLAN_TILE = 2, PLAN_WROW = 7, PLAN_TRANS = 9,
                      PLAN_SELL = 10, PLAN_SLAB = 11, PLAN_NCOLS = 12 };


// elements of Work::npart a dense matrix needs (0 for CSR / non-tiled plans):
// tile partials, then the fused A v's group slots and counters (k_rows_tile_fused)
inline int64_t npart_elems(int64_t m, int64_t n) {
  const int64_t g = tile_groups(m);
  return ((n + 2 * kNT - 1) / (2 * kNT)) * m + g * kKMax + (g + 1) / 2;
}

struct RowPlan {
  int kind = PLAN_SHORT;
  int wdense = 0;  // dense, small and L2-resident: one warp per row (k_rows_wdense)
  int P = 1;            // blocks
  int* wrow = nullptr;  // device [P * kWarps] (PLAN_FLAT)
  // PLAN_SELL: the sliced-ELL copy of this orientation (see k_rows_sell)
  int64_t sell_slots = 0;  // padded entries
  int* sell_sp = nullptr;  // device [ceil(rows / 32) + 1]
  int* sell_ci = nullptr;  // device [sell_slots]
  double* sell_val = nullptr;
  int sell_borrowed = 0;   // tables refilled in place in a recycled handle's plan (not owned)
  // PLAN_SLAB: the column-slab copy (see k_slab_av); P = slabs
  int slab_nsl = 0, slab_maxw = 0;
  int64_t slab_slots = 0, slab_rows = 0;
  int *slab_cb = nullptr, *slab_sp = nullptr, *slab_pos = nullptr;
  int2* slab_wr = nullptr;  // [P * 33] (first slice, slot offset) of every warp run
  uint16_t* slab_col = nullptr;
  double* slab_val = nullptr;
  int slab_borrowed = 0;
};

struct Instance;  // cached solver instance (ts_drivers.cuh)
struct Comm;      // column-sharding communicator (ts_comm.cuh)

struct Mat {
  int dev = 0;
  int sms = 148;
  int64_t m = 0, n = 0, nnz = 0;
  int kind = 0;  // 0 dense, 1 csr
  // dense
  double* a = nullptr;
  int64_t lda = 0;
  // small (L2-sized) dense A: a transposed copy, so A^T v runs as the fused
  // row-tile A v over it (PLAN_TRANS) instead of column tiles with split merges
  double* aT = nullptr;
  int64_t ldaT = 0;
  // csr + transposed csr
  int *rp = nullptr, *ci = nullptr, *rpT = nullptr, *ciT = nullptr;
  double *val = nullptr, *valT = nullptr;
  double fro = 0.0;
  int64_t band = -1;  // csr: max |row - column| over the stored entries (-1: unknown)
  RowPlan planN, planT;
  int Pmax = 0;  // largest grid any pass of this matrix uses
  // per-(tile,row) partials a solve's Work needs (dense tile A v)
  int64_t npart = 0;
  // column shard of a matrix split over ranks (nullptr: unsharded)
  Comm* comm = nullptr;
  int64_t n_global = 0, col_off = 0;
  // row-block shard (square A): rows / columns [row_off, row_off + m) are this
  // rank's; column indices are local (j - row_off) and reach `halo` entries
  // past either end, served from neighbours before every pass (k_halo)
  int row_shard = 0;
  int64_t halo = 0, m_global = 0, row_off = 0;
  // tall row-block shard: rows [row_off, row_off + m) of A with all n columns;
  // x-space is replicated, b-space split; A^T v sums an n-vector over ranks
  int tall_shard = 0;
  // solver instances (buffers + instantiated graphs) cached per solver shape
  std::mutex cache_mu;
  std::vector<Instance*> cache;

  DenseRows dense() const { return DenseRows{a, lda, m, n}; }
  CsrRows csr() const { return CsrRows{rp, ci, val, m, nnz}; }
  CsrRows csrT() const { return CsrRows{rpT, ciT, valT, n, nnz}; }
};

// one full wave of pass blocks (occupancy is register-bound at kMinBlocks per
// SM); TS_BLOCKS_PER_SM overrides for experiments
inline int blocks_per_sm() {
  static int v = [] {
    const char* e = getenv("TS_BLOCKS_PER_SM");
    int b = e ? atoi(e) : kMinBlocks;
    return (b > 0 && b <= 8) ? b : kMinBlocks;
  }();
  return v;
}
inline int resident_blocks(int sms) { return sms * blocks_per_sm(); }
inline int work_blocks(int sms) { return sms * 8; }  // workspace sizing upper bound

// first row touched by the warp whose range starts at s (see k_rows_flat)
inline int64_t first_row_at(const int* rp, int64_t rows, int64_t s) {
  // q = largest r in [0, rows) with rp[r] <= s
  int64_t lo = 0, hi = rows - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (rp[mid] <= s) lo = mid; else hi = mid - 1;
  }
  int64_t q = lo;
  if (rp[q] < s) return q;  // s strictly inside row q (continuation)
  // rp[q] == s: first row of the run starting at s
  int64_t lo2 = 0, hi2 = q;
  while (lo2 < hi2) {
    int64_t mid = (lo2 + hi2) / 2;
    if (rp[mid] >= s) hi2 = mid; else lo2 = mid + 1;
  }
  return lo2;
}

int plan_rows_csr(const int* rp_host, int64_t rows, int64_t nnz, int sms, RowPlan* out,
                  cudaStream_t st);
int plan_rows_dense(int64_t m, int64_t n, int sms, RowPlan* out, cudaStream_t st);
void destroy_instances(Mat* M);

inline int vec_grid(int64_t len, int sms, int per_sm = 0) {
  int64_t g = (len + kNT * 4 - 1) / (kNT * 4);
  int64_t pmax = per_sm > 0 ? (int64_t)sms * per_sm : resident_blocks(sms);
  if (g > pmax) g = pmax;
  if (g < 1) g = 1;
  return (int)g;
}

// per_sm: resident blocks per SM of the tile kernel (one full wave);
// min_rows: rows of a tile per block at least.  Only small (L2-resident)
// matrices feel it: for A^T v the column pieces of a tile are merged in block
// order by one block, and C1 runs 9.5 us per A^T v with 32 rows per block vs
// 15.7 us with 8 (16 and 64 were worse); A v is best at 8 (7.2 vs 9.1 us).
// dense matrices up to this size keep a transposed copy for A^T v (PLAN_TRANS)
constexpr int64_t kTransBytes = 32ll << 20;
// HBM-sized dense matrices keep a transposed copy too, for A v: the column-tile
// kernel (each thread owns two columns, 12 rows in flight, no warp reductions,
// no per-(tile, row) partials) streams at 0.96 of the copy peak, the row-tile
// kernel at 0.86-0.90 (C2: 126 vs 135-142 us); 180 GB of HBM pay for the copy
constexpr int64_t kNcolsBytes = 256ll << 20;
constexpr int kTileMinRowsN = 8;
constexpr int kTileMinRowsT = 32;
inline int tile_grid(int64_t m, int64_t n, int sms, int per_sm = kMinBlocks, int min_rows = kTileMinRowsN) {
  const int64_t tw = 2 * kNT;
  const int64_t nct = (n + tw - 1) / tw;
  const int64_t U = nct * m;
  int64_t g = U / min_rows;
  const int64_t pmax = (int64_t)sms * per_sm;
  if (g > pmax) g = pmax;
  if (g < 1) g = 1;
  return (int)g;
}

// ------------------------------------------------------------ dispatch ----
// y = M v (trans = 0) or y = M^T v (trans = 1) with a fused epilogue.
// A square banded L2-resident CSR matrix runs a CTA moments pair as one kernel
// (k_pair_band); TS_BAND_PAIR=0 keeps the two passes
inline size_t band_pair_smem(const Mat& M) {
  const int64_t P = M.planN.P > 0 ? M.planN.P : 1;
  return (size_t)((M.m + P - 1) / P + 1 + 2 * M.band) * sizeof(double);
}
inline bool band_pair_ok(const Mat& M) {
  static const bool off = [] {
    const char* e = getenv("TS_BAND_PAIR");
    return e && e[0] == '0';
  }();
  return !off && M.kind == 1 && !M.comm && M.m == M.n && M.band >= 0 && M.band <= 512 &&
         M.planN.kind == PLAN_SHORT && M.planT.kind == PLAN_SHORT && M.planN.P == M.planT.P &&
         M.band * 8 <= (M.m + M.planN.P - 1) / M.planN.P && band_pair_smem(M) <= 40 * 1024;
}
template <class EpiQ, class EpiP>
int launch_pair_band(const Mat& M, const double* pprev, const EpiQ& eq, const EpiP& ep, const Work& wk,
                     cudaStream_t st) {
  k_pair_band<EpiQ, EpiP><<<M.planN.P, kNT, band_pair_smem(M), st>>>(M.csrT(), M.csr(), pprev, (int)M.band, eq, ep, wk);
  TS_CUDA(cudaGetLastError());
  return 0;
}

// Cooperative kernels (grid barriers) need their whole grid resident: the device
// must support cooperative launches and `grid` blocks of the kernel must fit
// (occupancy x multiprocessors; asked once per kernel and device).  false: the
// caller keeps the barrier-free kernels.
template <class Kern>
inline bool coop_fits(Kern kernel, int grid, const Mat& M) {
  static int per_sm[64] = {0};  // 0: not asked yet, -1: no
  const int d = (M.dev >= 0 && M.dev < 64) ? M.dev : 0;
  if (per_sm[d] == 0) {
    int coop = 0, nb = 0;
    if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, M.dev) != cudaSuccess || !coop ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kNT, 0) != cudaSuccess || nb < 1) {
      cudaGetLastError();
      nb = -1;
    }
    per_sm[d] = nb;
  }
  return per_sm[d] > 0 && grid <= per_sm[d] * M.sms;
}
constexpr int kNoCoop = -7001;  // launch helper: the grid would not be co-resident

// A small L2-resident dense matrix (both orientations on the warp-per-row
// kernel) runs a CTA moments pair as one cooperative kernel (k_pair_wdense);
// TS_DENSE_PAIR=0 keeps the two passes
inline bool dense_pair_ok(const Mat& M) {
  static const bool off = [] {
    const char* e = getenv("TS_DENSE_PAIR");
    return e && e[0] == '0';
  }();
  return !off && M.kind == 0 && !M.comm && M.aT && M.planN.wdense && M.planT.wdense &&
         M.planT.kind == PLAN_TRANS;
}
template <class EpiQ, class EpiP>
int launch_pair_wdense(const Mat& M, const double* pprev, const double* q, const EpiQ& eq, const EpiP& ep,
                       const Work& wk, cudaStream_t st) {
  // one grid for both phases, co-resident (2 blocks/SM by the launch bounds)
  const int PT = std::min(M.planT.P, 2 * M.sms), PN = std::min(M.planN.P, 2 * M.sms);
  const int P = std::max(PT, PN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(kNT);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const DenseRows dT{M.aT, M.ldaT, M.n, M.m};
  const int64_t len = std::max(M.m, M.n);  // the longer of the two staged vectors
  if (!coop_fits(k_pair_wdense<EpiQ, EpiP, 16>, P, M)) return kNoCoop;
  if (len <= 4 * kNT)
    TS_CUDA(cudaLaunchKernelEx(&cfg, k_pair_wdense<EpiQ, EpiP, 4>, dT, M.dense(), pprev, q, eq, ep, wk, PT, PN));
  else if (len <= 8 * kNT)
    TS_CUDA(cudaLaunchKernelEx(&cfg, k_pair_wdense<EpiQ, EpiP, 8>, dT, M.dense(), pprev, q, eq, ep, wk, PT, PN));
  else
    TS_CUDA(cudaLaunchKernelEx(&cfg, k_pair_wdense<EpiQ, EpiP, 16>, dT, M.dense(), pprev, q, eq, ep, wk, PT, PN));
  return 0;
}

template <class Epi>
int launch_pass(const Mat& M, int trans, const double* x, XS xs, const Epi& epi, const Work& wk,
                cudaStream_t st) {
  if (M.kind == 0) {
    if (!trans) {
      if (M.planN.wdense)
        k_rows_wdense<Epi><<<M.planN.P, kNT, 0, st>>>(M.dense(), x, xs, epi, wk);
      else if (M.planN.kind == PLAN_NCOLS)
        k_cols_tile<Epi, 2><<<M.planN.P, kNT, 0, st>>>(DenseRows{M.aT, M.ldaT, M.n, M.m}, x, xs, epi, wk);
      else if (M.planN.kind == PLAN_TILE)
        k_rows_tile_fused<Epi><<<M.planN.P, kNT, 0, st>>>(M.dense(), x, xs, epi, wk);
      else
        k_rows_short<DenseRows, Epi><<<M.planN.P, kNT, 0, st>>>(M.dense(), x, xs, epi, wk);
    } else if (M.planT.kind == PLAN_TRANS) {
      // its partials / group slots / counters live after the A v pass's: the
      // counters must stay zero between launches (self-resetting)
      Work wt = wk;
      wt.npart = wk.npart + npart_elems(M.m, M.n);
      if (M.planT.wdense)
        k_rows_wdense<Epi><<<M.planT.P, kNT, 0, st>>>(DenseRows{M.aT, M.ldaT, M.n, M.m}, x, xs, epi, wt);
      else
        k_rows_tile_fused<Epi><<<M.planT.P, kNT, 0, st>>>(DenseRows{M.aT, M.ldaT, M.n, M.m}, x, xs, epi, wt);
    } else {
      k_cols_tile<Epi, 2><<<M.planT.P, kNT, 0, st>>>(M.dense(), x, xs, epi, wk);
    }
  } else {
    const RowPlan& pl = trans ? M.planT : M.planN;
    const CsrRows acc = trans ? M.csrT() : M.csr();
    if (pl.kind == PLAN_SLAB) {
      static bool attr_done[64] = {false};  // per device: the attribute is per function and device
      if (M.dev >= 0 && M.dev < 64 && !attr_done[M.dev]) {
        TS_CUDA(cudaFuncSetAttribute(k_slab_av<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlabSmemMax));
        attr_done[M.dev] = true;
      }
      const SlabRows sr{(int)acc.m, pl.P, pl.slab_nsl, (pl.slab_maxw + 15) & ~15, pl.slab_cb, pl.slab_sp,
                        pl.slab_wr, pl.slab_pos, pl.slab_col, pl.slab_val};
      k_slab_av<Epi><<<pl.P, kSlabT, slab_smem(pl.slab_maxw, pl.slab_nsl), st>>>(sr, x, xs, epi, wk.npart);
      const int ng = (int)((acc.m + 31) / 32);
      k_slab_combine<Epi><<<std::max(1, std::min(ng, wk.pmax)), kNT, 0, st>>>((int)acc.m, pl.P, wk.npart, epi,
                                                                             wk);
    } else if (pl.kind == PLAN_SELL)
      k_rows_sell<Epi><<<pl.P, kNT, 0, st>>>(SellRows{pl.sell_sp, pl.sell_ci, pl.sell_val, acc.m}, x, xs,
                                             epi, wk);
    else if (pl.kind == PLAN_FLAT)
      k_rows_flat<CsrRows, Epi><<<pl.P, kNT, 0, st>>>(acc, x, xs, epi, wk, pl.wrow);
    else if (pl.kind == PLAN_WROW)
      k_rows_wrow<Epi><<<pl.P, kNT, 0, st>>>(acc, x, xs, epi, wk);
    else
      k_rows_short<CsrRows, Epi><<<pl.P, kNT, 0, st>>>(acc, x, xs, epi, wk);
  }
  TS_CUDA(cudaGetLastError());
  return 0;
}

template <class Epi>
int launch_vec(int64_t len, int sms, const Epi& epi, const Work& wk, cudaStream_t st) {
  k_vec<Epi><<<vec_grid(len, sms, kVecBlocksOf<Epi>), kNT, 0, st>>>(len, epi, wk);
  TS_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace ts
