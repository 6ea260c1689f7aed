// Streaming "pass" kernels: one read of the matrix per launch, a per-output
// epilogue fused in, and a deterministic multi-slot reduction whose last
// arriving block runs a scalar finisher (the solver state machine).
//
//   k_rows_flat       y = M v, CSR with long irregular rows.  The flat entry
//                     range [0, E) is split into equal contiguous ranges per
//                     block and per warp, so every launch is load balanced for
//                     any row-length distribution; rows cut by a warp boundary
//                     are merged inside the block, rows cut by a block boundary
//                     by the last block to arrive on that row.
//   k_rows_wrow       long CSR rows of near-uniform length: warp per row with
//                     the next chunks' loads in flight.
//   k_slab_av         long CSR rows of a wide matrix (C5's A v): column slabs
//   + k_slab_combine  with x staged in shared memory, SELL-32-sigma inside.
//   k_rows_short      one thread per row, sequential left-to-right sum without
//                     FMA: bitwise scipy csr_matvec; L2-resident matrices (C3).
//   k_rows_sell       one thread per row over a sliced-ELL copy, bitwise
//                     scipy; HBM-sized short rows (C4, C5's A^T v).
//   k_rows_tile_fused dense A v: 512-column tiles, group-major (tile, row)
//                     units, groups combined by the block that completes them.
//   k_cols_tile       y = A^T v for dense row-major A without materialising
//                     A^T: 512-column tiles, the (tile, row) unit space split
//                     evenly over blocks, partial tiles at block boundaries
//                     merged by the last arriving block.
//   k_vec             fused elementwise vector pass (+ reductions, + finisher).
// Every reduction has a fixed order; no atomics on values.
//
// Epilogue contract (class Epi):
//   static constexpr int K;               reduction slots (<= kKMax)
//   __device__ int  op(int k) const;       RED_SUM / RED_MIN
//   __device__ bool active() const;        read once at kernel entry
//   __device__ void elem(int64 i, double y, double (&acc)[K]) const;   passes
//   __device__ void elem(int64 i, double (&acc)[K]) const;             k_vec
//   __device__ void finish(double (&red)[K]) const;  thread 0, last block
//   __device__ void idle() const;           block 0 / thread 0 when inactive
//   __device__ KTimer* timer() const;       live accounting slot or nullptr
//   __device__ void finish_block() const;   whole last block, after finish()
//   __device__ void count_launch() const;   block 0 / thread 0 at entry
//   __device__ void prepare(double* smem);   all threads at entry: cache device-state
//                                            scalars (registers / block smem) so
//                                            elem() never chains on global loads
#pragma once

#include "ts_common.cuh"

namespace ts {

// Input-vector transform applied on load: identity, or v -> s * v, or
// v -> s * max(v, 0) (the TA pivot preimage rho c / ||c||, c+ for the LP).
// `s` is read from device state at kernel entry.
struct XS {
  const double* sp = nullptr;  // nullptr: identity
  int relu = 0;
  double s = 1.0;
  __device__ __forceinline__ void load() {
    if (sp) s = *sp;
  }
  __device__ __forceinline__ double operator()(double v) const {
    if (!sp) return v;
    if (relu) v = (v >= 0.0 || v != v) ? v : 0.0;  // numpy.maximum(c, 0.0) (NaN kept)
    return __dmul_rn(s, v);
  }
};

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// ------------------------------------------------------------ accessors ----
struct DenseRows {
  const double* a;
  int64_t lda, m, n;
  __device__ __forceinline__ int64_t rows() const { return m; }
  // whole row, one thread, column order (short-row path)
  template <bool kCoh = false>
  __device__ __forceinline__ double row_serial(int64_t r, const double* x, const XS& xs) const {
    const double* row = a + r * lda;
    double s = 0.0;
    for (int64_t c = 0; c < n; ++c) s = fma(row[c], xs(ldx<kCoh>(x + c)), s);
    return s;
  }
};

struct CsrRows {
  const int* rp;
  const int* ci;
  const double* val;
  int64_t m, nnz;
  __device__ __forceinline__ int64_t rbeg(int64_t r) const { return __ldg(rp + r); }
  __device__ __forceinline__ int64_t rend(int64_t r) const { return __ldg(rp + r + 1); }
  __device__ __forceinline__ int64_t total() const { return nnz; }
  __device__ __forceinline__ int64_t rows() const { return m; }
  __device__ __forceinline__ double seg(int64_t r, int64_t k0, int64_t k1, const double* x,
                                        const XS& xs, int lane) const {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t k = k0 + lane;
    for (; k + 224 < k1; k += 256) {
      double v[8], xv[8];
      int j[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = ld_stream(val + k + 32 * u);
        j[u] = ld_stream_i(ci + k + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = __ldg(x + j[u]);
#pragma unroll
      for (int u = 0; u < 8; u += 4) {
        a0 = fma(v[u], xs(xv[u]), a0);
        a1 = fma(v[u + 1], xs(xv[u + 1]), a1);
        a2 = fma(v[u + 2], xs(xv[u + 2]), a2);
        a3 = fma(v[u + 3], xs(xv[u + 3]), a3);
      }
    }
    for (; k < k1; k += 32) a0 = fma(ld_stream(val + k), xs(__ldg(x + ld_stream_i(ci + k))), a0);
    return (a0 + a1) + (a2 + a3);
  }
  // scipy csr_matvec order: sum = 0; sum += A_ij * x_j left to right; no FMA
  template <bool kCoh = false>
  __device__ __forceinline__ double row_serial(int64_t r, const double* x, const XS& xs) const {
    return row_serial_k<kCoh>(__ldg(rp + r), __ldg(rp + r + 1), x, xs);
  }
  template <bool kCoh = false>
  __device__ __forceinline__ double row_serial_k(int k0, int k1, const double* x, const XS& xs) const {
    double s = 0.0;
    int k = k0;
    for (; k + 4 <= k1; k += 4) {
      double v[4], xv[4];
      int j[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = ld_stream(val + k + u);
        j[u] = ld_stream_i(ci + k + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = ldx<kCoh>(x + j[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) s = __dadd_rn(s, __dmul_rn(v[u], xs(xv[u])));
    }
    // the last 0-3 entries: loads batched (one index -> gather round trip,
    // not one per entry), sums still left to right
    const int rem = k1 - k;
    double v[3], xv[3];
    int j[3];
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (u < rem) {
        v[u] = ld_stream(val + k + u);
        j[u] = ld_stream_i(ci + k + u);
      }
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (u < rem) xv[u] = ldx<kCoh>(x + j[u]);
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (u < rem) s = __dadd_rn(s, __dmul_rn(v[u], xs(xv[u])));
    return s;
  }
};

// block containing flat element p when [0,E) is split as floor(b E / P)
__device__ __forceinline__ int64_t blk_of(int64_t p, int64_t E, int64_t P) {
  return ((p + 1) * P + E - 1) / E - 1;
}

// ------------------------------------------------------------ finishers ----
// Single-kernel pass: the last block to arrive reduces the `nb` block partials
// (+ split fixes) in fixed order and runs the finisher / finish_block.
template <class Epi>
__device__ __forceinline__ void finish_last(Epi& epi, const Work& wk, const double* facc, int nb,
                                            double* sm, int* sflag) {
  constexpr int K = Epi::K;
  if (nb == 1 && !facc) {
    // a single block (vector passes of small systems): no arrival counter, no
    // fences, no reload — the value reduce_partials would return (identity
    // combined with the block's sums, then zeros added across the block)
    if (threadIdx.x == 0) {
      double red[K];
#pragma unroll
      for (int k = 0; k < K; ++k)
        red[k] = red_combine(epi.op(k), red_identity(epi.op(k)), wk.bacc[k]);  // block slot 0: the only one
      ktimer_end(epi.timer());
      epi.finish(red);
    }
    __syncthreads();
    epi.finish_block();
    return;
  }
  if (arrive_last(wk.done, (unsigned)nb, sflag)) {
    double red[K];
    reduce_partials<K>(wk.bacc, facc, nb, red, sm, epi);
    if (threadIdx.x == 0) {
      ktimer_end(epi.timer());
      epi.finish(red);
    }
    __syncthreads();
    epi.finish_block();
  }
}

// ----------------------------------------------------------- k_rows_flat ----
// 3 blocks/SM (85 registers): at 64 the 8-deep gather loop spilled
constexpr int kFlatBlocks = 3;
template <class Acc, class Epi>
__global__ void __launch_bounds__(kNT, kFlatBlocks) k_rows_flat(Acc A, const double* __restrict__ x, XS xs,
                                                   Epi epi, Work wk,
                                                   const int* __restrict__ wrow) {
  constexpr int K = Epi::K;
  __shared__ double sm[kWarps * kKMax];
  __shared__ double wacc[kWarps][K];
  __shared__ long long prow[kWarps][2];
  __shared__ double psum[kWarps][2];
  __shared__ int pcnt[kWarps];
  __shared__ int sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  xs.load();
  KTimer* kt = epi.timer();
  ktimer_begin(kt);
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
  __syncthreads();
  const int64_t P = gridDim.x, b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t E = A.total();
  const int64_t S0 = E * b / P, S1 = E * (b + 1) / P;
  const int64_t L = S1 - S0;
  const int64_t s = S0 + L * wid / kWarps, e = S0 + L * (wid + 1) / kWarps;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  int np = 0;
  long long pr[2] = {0, 0};
  double ps[2] = {0.0, 0.0};
  if (s < e) {
    const bool gl_last = (b == P - 1) && (wid == kWarps - 1);
    for (int64_t r = wrow[b * kWarps + wid]; r < A.rows(); ++r) {
      const int64_t rb = A.rbeg(r), re = A.rend(r);
      if (!(rb < e || (gl_last && rb == e))) break;
      const int64_t k0 = rb > s ? rb : s, k1 = re < e ? re : e;
      double v = (k1 > k0) ? A.seg(r, k0, k1, x, xs, lane) : 0.0;
      v = warp_reduce(v, RED_SUM);
      if (k0 == rb && k1 == re) {
        if (lane == 0) epi.elem(r, v, acc);
      } else if (np < 2) {
        pr[np] = r;
        ps[np] = v;
        ++np;
      }
    }
  }
  if (lane == 0) {
    pcnt[wid] = np;
    prow[wid][0] = pr[0];
    prow[wid][1] = pr[1];
    psum[wid][0] = ps[0];
    psum[wid][1] = ps[1];
#pragma unroll
    for (int k = 0; k < K; ++k) wacc[wid][k] = acc[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double macc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) macc[k] = red_identity(epi.op(k));
    // merge warp pieces in warp order; rows wholly inside the block finish here
    long long cur = -1;
    double csum = 0.0;
    long long brow_first = -1, brow_last = -1;
    double bsum_first = 0.0, bsum_last = 0.0;
    auto flush = [&](long long row, double sum) {
      const int64_t rb = A.rbeg(row), re = A.rend(row);
      const bool before = rb < S0, after = re > S1;
      if (!before && !after) {
        epi.elem(row, sum, macc);
      } else if (before) {
        brow_first = row;
        bsum_first = sum;
      } else {
        brow_last = row;
        bsum_last = sum;
      }
    };
    for (int j = 0; j < kWarps; ++j) {
      for (int i = 0; i < pcnt[j]; ++i) {
        const long long row = prow[j][i];
        const double sum = psum[j][i];
        if (cur == row) {
          csum += sum;
        } else {
          if (cur >= 0) flush(cur, csum);
          cur = row;
          csum = sum;
        }
      }
    }
    if (cur >= 0) flush(cur, csum);
    // block accumulator: warps in order, then the merged rows
    double bacc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double v = wacc[0][k];
      for (int j = 1; j < kWarps; ++j) v = red_combine(epi.op(k), v, wacc[j][k]);
      bacc[k] = red_combine(epi.op(k), v, macc[k]);
      wk.bacc[b * kKMax + k] = bacc[k];
    }
    // is this block the end block of a row that started in an earlier block?
    bool end_block = false;
    if (brow_first >= 0 && A.rend(brow_first) <= S1) end_block = true;
    if (!end_block) {
      for (int k = 0; k < K; ++k) wk.facc[b * kKMax + k] = red_identity(epi.op(k));
    }
    // publish boundary pieces, then take part in the split-row merges
    if (brow_first >= 0) wk.bpart[b * 2 + 0] = bsum_first;
    if (brow_last >= 0) wk.bpart[b * 2 + 1] = bsum_last;
    for (int which = 0; which < 2; ++which) {
      const long long row = which == 0 ? brow_first : brow_last;
      if (row < 0) continue;
      const int64_t rb = A.rbeg(row), re = A.rend(row);
      const int64_t ba = blk_of(rb, E, P), bb = blk_of(re - 1, E, P);
      __threadfence();
      const unsigned prev = atomicAdd(wk.cnt + bb, 1u);
      if (prev == (unsigned)(bb - ba)) {
        __threadfence();
        double y = __ldcg(wk.bpart + ba * 2 + 1);
        for (int64_t q = ba + 1; q <= bb; ++q) y += __ldcg(wk.bpart + q * 2 + 0);
        double facc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) facc[k] = red_identity(epi.op(k));
        epi.elem(row, y, facc);
#pragma unroll
        for (int k = 0; k < K; ++k) wk.facc[bb * kKMax + k] = facc[k];
        wk.cnt[bb] = 0u;
      }
    }
  }
  if (arrive_last(wk.done, (unsigned)P, &sflag)) {
    double red[K];
    reduce_partials<K>(wk.bacc, wk.facc, (int)P, red, sm, epi);
    if (threadIdx.x == 0) {
      ktimer_end(kt);
      epi.finish(red);
    }
    __syncthreads();
    epi.finish_block();
  }
}

// ---------------------------------------------------------- k_rows_short ----
// kb/ke: the thread's first CSR row bounds when the kernel loaded them
// before its state read (-1: not loaded)
template <class Acc, class Epi, bool kP>
__device__ __forceinline__ void body_rows_short(const Acc& A, const double* __restrict__ x, XS xs,
                                                Epi& epi, const Work& wk, int64_t b, int64_t P,
                                                int kb = -1, int ke = -1) {
  constexpr int K = Epi::K;
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  xs.load();
  ktimer_begin(epi.timer());
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
  __syncthreads();
  const int64_t m = A.rows();
  const int64_t R0 = m * b / P, R1 = m * (b + 1) / P;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  int64_t r = R0 + threadIdx.x;
  if constexpr (std::is_same_v<Acc, CsrRows>) {
    if (kb >= 0 && r < R1) {
      epi.elem(r, A.template row_serial_k<kP>(kb, ke, x, xs), acc);
      r += kNT;
    }
  }
  for (; r < R1; r += kNT) epi.elem(r, A.template row_serial<kP>(r, x, xs), acc);
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[b * kKMax + k] = acc[k];
  }
  if constexpr (!kP) finish_last(epi, wk, nullptr, (int)P, sm, &sflag);
}

template <class Acc, class Epi>
__global__ void __launch_bounds__(kNT, kMinBlocks) k_rows_short(Acc A, const double* __restrict__ x, XS xs,
                                                    Epi epi, Work wk) {
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  // L2-resident passes are a chain of dependent loads: the first row's bounds
  // do not depend on the state word, so both are in flight together
  int kb = -1, ke = -1;
  if constexpr (std::is_same_v<Acc, CsrRows>) {
    const int64_t m = A.rows(), P = gridDim.x, b = blockIdx.x;
    const int64_t r = m * b / P + threadIdx.x;
    if (r < m * (b + 1) / P) {
      kb = __ldg(A.rp + r);
      ke = __ldg(A.rp + r + 1);
    }
  }
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  body_rows_short<Acc, Epi, false>(A, x, xs, epi, wk, blockIdx.x, gridDim.x, kb, ke);
}

// ------------------------------------------------------------ k_pair_band ----
// One CTA moments pair in ONE kernel for a square banded CSR matrix that is
// L2-resident (C3: tridiagonal, n = 100001): q = A^T p, then p' = A q.  A pass
// over such a matrix is a chain of dependent latencies, and the pair needs a
// grid-wide dependency only because p'_i reads q at the columns of row i —
// with bandwidth bw those are [i - bw, i + bw].  So block b, owning rows [R0,
// R1), computes q on [R0 - bw, R1 + bw) into shared memory (the halo rows
// redundantly, from p which is complete), stores its own q rows and runs the
// q epilogue on them, then computes p' on its rows from shared memory and
// runs the p' epilogue; one reduction of both epilogues' sums, the last block
// finishes both.  Every row keeps scipy's operation sequence (left to right,
// no FMA) and the thread <-> row mapping of k_rows_short, so q, p' and their
// block sums are the bits the two separate passes produce.
struct OpsSum {
  __device__ __forceinline__ int op(int) const { return RED_SUM; }
};

// scipy csr_matvec order over entries [k0, k1) with a generic gather pointer
__device__ __forceinline__ double row_serial_any(const CsrRows& A, int k0, int k1, const double* xq) {
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
    for (int u = 0; u < 4; ++u) xv[u] = xq[j[u]];
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
    if (u < rem) xv[u] = xq[j[u]];
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (u < rem) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
  return s;
}

template <class EpiQ, class EpiP>
__global__ void __launch_bounds__(kNT, kMinBlocks) k_pair_band(CsrRows AT, CsrRows A, const double* pprev, int bw,
                                                             EpiQ eq, EpiP ep, Work wk) {
  constexpr int KQ = EpiQ::K, KP = EpiP::K, K = KQ + KP;
  extern __shared__ double qs[];  // q on [lo, hi)
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) ep.count_launch();
  const int64_t m = A.m, P = gridDim.x, b = blockIdx.x;
  const int64_t R0 = m * b / P, R1 = m * (b + 1) / P;
  const int64_t lo = R0 - bw > 0 ? R0 - bw : 0, hi = R1 + bw < m ? R1 + bw : m;
  // p is complete and the matrix immutable: the thread's first q row is computed
  // (loads and arithmetic only) while the state word is in flight
  int64_t j = R0 + threadIdx.x;
  double qfirst = 0.0;
  if (j < R1) qfirst = row_serial_any(AT, __ldg(AT.rp + j), __ldg(AT.rp + j + 1), pprev);
  if (!ep.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ep.idle();
    return;
  }
  ktimer_begin(ep.timer());
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  double (&aq)[KQ] = *reinterpret_cast<double (*)[KQ]>(&acc[0]);
  double (&ap)[KP] = *reinterpret_cast<double (*)[KP]>(&acc[KQ]);
  // q on the block's own rows (k_rows_short's thread <-> row mapping), then the halo rows
  for (bool first = true; j < R1; j += kNT, first = false) {
    const double qv = first ? qfirst : row_serial_any(AT, __ldg(AT.rp + j), __ldg(AT.rp + j + 1), pprev);
    qs[j - lo] = qv;
    eq.elem(j, qv, aq);
  }
  for (int64_t h = lo + threadIdx.x; h < R0; h += kNT)
    qs[h - lo] = row_serial_any(AT, __ldg(AT.rp + h), __ldg(AT.rp + h + 1), pprev);
  for (int64_t h = R1 + threadIdx.x; h < hi; h += kNT)
    qs[h - lo] = row_serial_any(AT, __ldg(AT.rp + h), __ldg(AT.rp + h + 1), pprev);
  __syncthreads();
  const double* xq = qs - lo;
  for (int64_t r = R0 + threadIdx.x; r < R1; r += kNT)
    ep.elem(r, row_serial_any(A, __ldg(A.rp + r), __ldg(A.rp + r + 1), xq), ap);
  const OpsSum ops;
  block_reduce<K>(acc, sm, ops);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[b * kKMax + k] = acc[k];
  }
  if (arrive_last(wk.done, (unsigned)P, &sflag)) {
    double red[K];
    reduce_partials<K>(wk.bacc, nullptr, (int)P, red, sm, ops);
    if (threadIdx.x == 0) {
      ktimer_end(ep.timer(), 2);
      double rq[KQ], rp2[KP];
#pragma unroll
      for (int k = 0; k < KQ; ++k) rq[k] = red[k];
#pragma unroll
      for (int k = 0; k < KP; ++k) rp2[k] = red[KQ + k];
      eq.finish(rq);
      ep.finish(rp2);
    }
    __syncthreads();
    ep.finish_block();
  }
}

// ----------------------------------------------------------- k_rows_sell ----
// Short CSR rows, HBM-sized (C4 both ways, C5's A^T v): a sliced-ELL copy
// (SELL-32) built once at matrix creation.  Slice s holds rows [32 s, 32 s +
// 32) interleaved — entry k of row 32 s + l sits at sp[s] + 32 k + l — padded
// to the slice's longest row with column kSellPad.  One thread per row: every
// load of a warp is one coalesced request, no row pointers are chased, and
// each thread adds ITS row's products left to right without FMA, skipping the
// padding — scipy's csr_matvec operation sequence, so the result is bitwise
// the reference's.  tools/microbench/spmv_sell.cu (cold L2): C4 28.7 -> 22.6
// us, C5^T 46.1 -> 30.8 us against the warp-cooperative CSR kernel it
// replaces.
constexpr int kSellPad = INT32_MIN;  // padding column (local indices of row shards may be negative)
constexpr int kSellU = 8;            // entries of a row in flight per thread

struct SellRows {
  const int* sp;      // [nslices + 1] padded entry offsets (multiples of 32)
  const int* ci;      // column per slot, kSellPad on padding
  const double* val;  // value per slot (0 on padding)
  int64_t m;
};

template <class Epi>
__global__ void __launch_bounds__(kNT, kMinBlocks) k_rows_sell(SellRows A, const double* __restrict__ x, XS xs,
                                                             Epi epi, Work wk) {
  constexpr int K = Epi::K;
  constexpr int U = kSellU;
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  xs.load();
  ktimer_begin(epi.timer());
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (A.m + 31) >> 5;
  const int64_t W = (int64_t)gridDim.x * kWarps;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  // the next slice's offsets are loaded a slice ahead: one dependent round trip
  // (offsets -> entries -> gathers) less per slice
  int64_t s = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  int nb0 = 0, nb1 = 0;
  if (s < nsl) {
    nb0 = __ldg(A.sp + s);
    nb1 = __ldg(A.sp + s + 1);
  }
  for (; s < nsl; s += W) {
    const int b0 = nb0;
    const int wd = (nb1 - b0) >> 5;
    if (s + W < nsl) {
      nb0 = __ldg(A.sp + s + W);
      nb1 = __ldg(A.sp + s + W + 1);
    }
    const int* cp = A.ci + b0 + lane;
    const double* vp = A.val + b0 + lane;
    double sum = 0.0;
    for (int k0 = 0; k0 < wd; k0 += U) {
      double v[U], xv[U];
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // independent loads first ...
        const bool ok = k0 + u < wd;
        c[u] = ok ? ld_stream_i(cp + 32 * (k0 + u)) : kSellPad;
        v[u] = ok ? ld_stream(vp + 32 * (k0 + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = c[u] != kSellPad ? __ldg(x + c[u]) : 0.0;  // ... then the gathers
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] != kSellPad) sum = __dadd_rn(sum, __dmul_rn(v[u], xs(xv[u])));
    }
    const int64_t r = s * 32 + lane;
    if (r < A.m) epi.elem(r, sum, acc);
  }
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[blockIdx.x * kKMax + k] = acc[k];
  }
  finish_last(epi, wk, nullptr, (int)gridDim.x, sm, &sflag);
}

// ----------------------------------------------------------- k_rows_wrow ----
// Long, near-uniform CSR rows (C5's A v: 10^4 rows of ~1000 entries gathering
// x at random from 8 MB): one warp per row, lanes striding the row 32 entries
// at a time, with the next kWrowU chunks' values and column indices loaded
// before the current chunk's x gathers are issued, so every warp always has
// matrix loads AND gathers in flight.  tools/microbench/spmv_long.cu on C5:
// 49 us vs 64 us for the flat split kernel (whose warps wait on one chunk's
// gathers before loading the next).  Four partial accumulators per lane
// (entry k of a lane goes to accumulator (k / 32) % 4), then the xor tree.
constexpr int kWrowU = 6;
constexpr int kWrowBlocks = 3;  // 85 registers: no spills with the epilogues

template <class Epi>
__global__ void __launch_bounds__(kNT, kWrowBlocks) k_rows_wrow(CsrRows A, const double* __restrict__ x, XS xs,
                                                             Epi epi, Work wk) {
  constexpr int K = Epi::K;
  constexpr int U = kWrowU;
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  xs.load();
  ktimer_begin(epi.timer());
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * kNT) >> 5;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  for (int64_t r = w; r < A.m; r += W) {
    const int k0 = __ldg(A.rp + r), k1 = __ldg(A.rp + r + 1);
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    double pv[U];
    int pj[U];
    int k = k0 + lane;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = k + 32 * u;
      pv[u] = kk < k1 ? ld_stream(A.val + kk) : 0.0;
      pj[u] = kk < k1 ? ld_stream_i(A.ci + kk) : 0;
    }
    for (; k < k1; k += 32 * U) {
      double v[U];
      int j[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = pv[u];
        j[u] = pj[u];
      }
      const int kn = k + 32 * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kn + 32 * u;
        pv[u] = kk < k1 ? ld_stream(A.val + kk) : 0.0;
        pj[u] = kk < k1 ? ld_stream_i(A.ci + kk) : 0;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = xs(__ldg(x + j[u]));  // j = 0 past the end: v = 0
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], xv[u], a[u & 3]);
    }
    const double sum = warp_reduce((a[0] + a[1]) + (a[2] + a[3]), RED_SUM);
    if (lane == 0) epi.elem(r, sum, acc);
  }
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[blockIdx.x * kKMax + k] = acc[k];
  }
  finish_last(epi, wk, nullptr, (int)gridDim.x, sm, &sflag);
}

// ------------------------------------------------------------- k_slab_av ----
// Long-row CSR A v over a WIDE matrix (C5: 10^4 rows x 10^6 columns, ~1000
// entries per row, x = 8 MB): the warp-per-row kernel is bound by its random
// 8-byte gathers of x, each one 32-byte L2 sector.  Here the columns are cut
// into P slabs of equal nnz (P = #SMs, one 1024-thread block per slab), each
// block stages its slab of x — transformed once by `xs` — in shared memory,
// so every gather is a shared-memory read.  Inside a slab the rows are sorted
// by their in-slab length (descending, stable) and cut into slices of 32
// whose entries are interleaved (SELL-32-sigma: entry k of lane l at sp + 32 k
// + l; fp64 values, in-slab column offsets as u16, padding 0xFFFF).  Each warp
// streams a contiguous run of slices as one coalesced stream, register
// double-buffered: the next kSlabU k-steps are in flight while the current
// ones are consumed (slice ends from the slab's offsets in shared memory).
// A slice's row sums (FMA chain in the row's column order) go to shared
// memory in SLICE order — no permutation load and no scattered store inside
// the stream (1.5 M scattered 8-byte stores cost ~10 us of L2 sector traffic
// on C5) — and the block writes part[s][0..m) coalesced at the end through
// the inverse permutation `pos`.  k_slab_combine then adds the P partials of
// a row in slab order and runs the pass epilogue.
// tools/microbench/spmv_slab.cu on C5 (warm, in-kernel clocks): staged 2.1 us,
// streamed by 18.8 us (100.5 MB in 16.7 us = 6.0 TB/s), flushed by 21.0 us.
constexpr int kSlabT = 1024;       // threads of a slab block
constexpr int kSlabU = 4;          // k-steps per register buffer (two buffers in flight)
constexpr int kSlabMaxW = 24576;   // columns per slab at most (u16 offsets, shared memory)
constexpr int kSlabSmemMax = 220 * 1024;  // x slab + slice sums + slice offsets
constexpr unsigned kSlabPad = 0xFFFFu;

// dynamic shared memory of a slab block: x slab (padded to 16 doubles), one
// sum per (slice, lane), the slab's slice offsets
__host__ __device__ inline int slab_accn(int nsl) { return nsl * 32; }
inline size_t slab_smem(int maxw, int nsl) {
  return (size_t)((maxw + 15) & ~15) * 8 + (size_t)slab_accn(nsl) * 8 + ((size_t)nsl + 1) * 4 + 16;
}

struct SlabRows {
  int m, P, nsl;          // rows, slabs, slices per slab
  int xcap;               // doubles reserved for the x slab
  const int* cb;          // [P + 1] slab column boundaries
  const int* sp;          // [P * nsl + 1] slot offset of every slice
  const int2* wr;         // [P * 33] each warp's run: (first in-slab slice, its slot offset)
  const int* pos;         // [P * m] position (slice * 32 + lane) of every row in its slab's order
  const uint16_t* col;    // in-slab column, kSlabPad on padding
  const double* val;
};

__device__ __forceinline__ unsigned ld_stream_u16(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

template <class Epi>
__global__ void __launch_bounds__(kSlabT, 1) k_slab_av(SlabRows S, const double* __restrict__ x, XS xs, Epi epi,
                                                       double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char slab_raw[];
  double* xsl = reinterpret_cast<double*>(slab_raw);              // [xcap]
  double* accs = xsl + S.xcap;                                    // [slab_accn(nsl)]
  int* sps = reinterpret_cast<int*>(accs + slab_accn(S.nsl));     // [nsl + 1]
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  unsigned long long t_in = 0;  // entry time (thread 0): hoisted work stays inside the accounted interval
  if (threadIdx.x == 0) t_in = globaltimer();
  // The tables are immutable and x is complete: the table chain (slab bounds ->
  // run bounds -> first k-steps) and the thread's part of the x slab are in
  // flight before the state word decides whether the pass runs at all.
  constexpr int U = kSlabU;
  constexpr int XR = 8;  // x entries per thread staged through registers (slabs of <= 8192 columns)
  const int s = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cb0 = __ldg(S.cb + s), cw = __ldg(S.cb + s + 1) - cb0;
  const int2 w0 = __ldg(S.wr + s * 33 + w), w1 = __ldg(S.wr + s * 33 + w + 1);
  const int q0 = w0.x, q1 = w1.x, E0 = w0.y, E1 = w1.y;
  const int g0 = s * S.nsl;
  const int KT = (E1 - E0) >> 5;  // k-steps (32 slots each) of this warp's run
  const double* vp = S.val + E0 + lane;
  const uint16_t* cp = S.col + E0 + lane;
  double va[U], vb[U];
  unsigned ca[U], cc[U];
  auto load = [&](double (&v)[U], unsigned (&c)[U], int k0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = k0 + u < KT;
      v[u] = ok ? ld_stream(vp + 32 * (k0 + u)) : 0.0;
      c[u] = ok ? ld_stream_u16(cp + 32 * (k0 + u)) : kSlabPad;
    }
  };
  load(va, ca, 0);  // in flight with the staging below
  double xr[XR];
#pragma unroll
  for (int u = 0; u < XR; ++u) {
    const int i = threadIdx.x + u * kSlabT;
    xr[u] = i < cw ? __ldg(x + cb0 + i) : 0.0;
  }
  if (!epi.active()) return;  // k_slab_combine owns idle()
  xs.load();
  ktimer_begin_at(epi.timer(), t_in);
  for (int i = threadIdx.x; i <= S.nsl; i += kSlabT) sps[i] = __ldg(S.sp + g0 + i);
#pragma unroll
  for (int u = 0; u < XR; ++u) {
    const int i = threadIdx.x + u * kSlabT;
    if (i < cw) xsl[i] = xs(xr[u]);
  }
  for (int i = threadIdx.x + XR * kSlabT; i < cw; i += kSlabT) xsl[i] = xs(__ldg(x + cb0 + i));
  __syncthreads();
  int q = q0;
  int kend = q0 < q1 ? (sps[q0 + 1] - E0) >> 5 : INT32_MAX;
  double acc = 0.0;
  auto emit = [&]() {  // the slice's rows are complete: park the sums, move to the next slice
    accs[q * 32 + lane] = acc;
    acc = 0.0;
    ++q;
    kend = q < q1 ? (sps[q + 1] - E0) >> 5 : INT32_MAX;
  };
  auto consume = [&](const double (&v)[U], const unsigned (&c)[U], int k0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u;
      if (k >= KT) break;
      while (k == kend) emit();
      if (c[u] != kSlabPad) acc = fma(v[u], xsl[c[u]], acc);
    }
  };
  for (int k0 = 0; k0 < KT; k0 += 2 * U) {
    load(vb, cc, k0 + U);
    consume(va, ca, k0);
    load(va, ca, k0 + 2 * U);
    consume(vb, cc, k0 + U);
  }
  while (q < q1) emit();
  __syncthreads();
  double* out = part + (size_t)s * S.m;
  const int* pv = S.pos + (size_t)s * S.m;
  for (int r = threadIdx.x; r < S.m; r += kSlabT) out[r] = accs[__ldg(pv + r)];
}

// y_r = sum over slabs of part[s][r], slabs in order: 32 rows per block, warp
// g adds the contiguous slab range [g P / 8, (g + 1) P / 8) with all its loads
// in flight, the 8 warp sums are added in warp order; then the epilogue
template <class Epi>
__global__ void __launch_bounds__(kNT) k_slab_combine(int m, int P, const double* __restrict__ part, Epi epi,
                                                      Work wk) {
  constexpr int K = Epi::K;
  __shared__ double sm[kWarps * kKMax];
  __shared__ double red[kWarps][33];
  __shared__ int sflag;
  __shared__ double epi_smem[kEpiSmem];
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int qa = P * g / kWarps, qb = P * (g + 1) / kWarps;
  const int ngroups = (m + 31) >> 5;
  // slab sums of one row over this warp's slab range, every load of a batch in
  // flight (a serial tail costs a round trip per slab)
  auto range_sum = [&](int r) -> double {
    double sum = 0.0;
    if (r < m) {
      for (int q = qa; q < qb; q += 10) {
        double t[10];
#pragma unroll
        for (int u = 0; u < 10; ++u) t[u] = q + u < qb ? __ldcg(part + (size_t)(q + u) * m + r) : 0.0;
#pragma unroll
        for (int u = 0; u < 10; ++u) sum += t[u];
      }
    }
    return sum;
  };
  // the partials are complete (the slab kernel wrote them): the block's first
  // row group is summed while the state word is in flight
  double sum0 = 0.0;
  if ((int)blockIdx.x < ngroups) sum0 = range_sum((int)blockIdx.x * 32 + lane);
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  epi.prepare(epi_smem);
  __syncthreads();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  for (int rg = blockIdx.x; rg < ngroups; rg += gridDim.x) {
    const int r = rg * 32 + lane;
    const double sum = rg == (int)blockIdx.x ? sum0 : range_sum(r);
    red[g][lane] = sum;
    __syncthreads();
    if (g == 0 && r < m) {
      double y = red[0][lane];
#pragma unroll
      for (int j = 1; j < kWarps; ++j) y += red[j][lane];
      epi.elem(r, y, acc);
    }
    __syncthreads();
  }
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[blockIdx.x * kKMax + k] = acc[k];
  }
  finish_last(epi, wk, nullptr, (int)gridDim.x, sm, &sflag);
}

// ----------------------------------------------------------- k_cols_tile ----
// VW columns per thread (2: 128-bit loads, 4: 256-bit loads); tile = VW * kNT
// k_cols_tile occupancy and depth: 3 blocks/SM with 12 rows in flight per
// thread streams the C2 matrix in 118 us vs 122 us at 4 x 8
// (tools/microbench/dense_av.cu); RU is even, so rows keep alternating
// between the two accumulators exactly as before.
constexpr int kTileTBlocks = 3;
constexpr int kTileTRows = 12;

template <class Epi, int VW, bool kP, int RU0 = 8>
__device__ __forceinline__ void body_cols_tile(const DenseRows& A, const double* __restrict__ x, XS xs,
                                               Epi& epi, const Work& wk, int64_t b, int64_t P) {
  constexpr int K = Epi::K;
  constexpr int TW = VW * kNT;       // tile width (columns)
  constexpr int RU = VW == 4 ? 4 : RU0;  // rows in flight per thread
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  xs.load();
  ktimer_begin(epi.timer());
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
  __syncthreads();
  const int64_t m = A.m, n = A.n, lda = A.lda;
  const int64_t nct = (n + TW - 1) / TW;
  const int64_t U = nct * m;
  const int64_t U0 = U * b / P, U1 = U * (b + 1) / P;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  long long ct_first = -1, ct_last = -1;
  for (int64_t u = U0; u < U1;) {
    const int64_t ct = u / m, r0 = u - ct * m;
    const int64_t r1 = (m < r0 + (U1 - u)) ? m : r0 + (U1 - u);
    const int64_t c = ct * TW + VW * threadIdx.x;
    const int64_t nv = n - c < VW ? (n - c > 0 ? n - c : 0) : VW;  // valid columns of this thread
    double ac[2][VW];
#pragma unroll
    for (int j = 0; j < VW; ++j) ac[0][j] = ac[1][j] = 0.0;
    const double* base = A.a + c;
    int64_t r = r0;
    if (nv == VW) {
      for (; r + RU <= r1; r += RU) {
        double v[RU][VW];
        double xr[RU];
#pragma unroll
        for (int i = 0; i < RU; ++i) {
          if constexpr (VW == 4) {
            ld_stream4(base + (r + i) * lda, v[i]);
          } else {
            const double2 t2 = ld_stream2(base + (r + i) * lda);
            v[i][0] = t2.x;
            v[i][1] = t2.y;
          }
        }
#pragma unroll
        for (int i = 0; i < RU; ++i) xr[i] = xs(ldx<kP>(x + r + i));
#pragma unroll
        for (int i = 0; i < RU; ++i)
#pragma unroll
          for (int j = 0; j < VW; ++j) ac[i & 1][j] = fma(v[i][j], xr[i], ac[i & 1][j]);
      }
      for (; r < r1; ++r) {
        const double xr = xs(ldx<kP>(x + r));
#pragma unroll
        for (int j = 0; j < VW; ++j) ac[0][j] = fma(ld_stream(base + r * lda + j), xr, ac[0][j]);
      }
    } else if (nv > 0) {
      for (; r < r1; ++r) {
        const double xr = xs(ldx<kP>(x + r));
        for (int j = 0; j < nv; ++j) ac[0][j] = fma(ld_stream(base + r * lda + j), xr, ac[0][j]);
      }
    }
    double sv[VW];
#pragma unroll
    for (int j = 0; j < VW; ++j) sv[j] = ac[0][j] + ac[1][j];
    if (r0 == 0 && r1 == m) {
#pragma unroll
      for (int j = 0; j < VW; ++j)
        if (j < nv) epi.elem(c + j, sv[j], acc);
    } else {
      const int which = (r0 > 0) ? 0 : 1;  // 0: tile began in an earlier block
      double* dst = wk.tpart + ((size_t)b * 2 + which) * kCW + VW * threadIdx.x;
#pragma unroll
      for (int j = 0; j < VW; ++j) dst[j] = sv[j];
      if (which == 0) ct_first = ct; else ct_last = ct;
    }
    u += r1 - r0;
  }
  // split-tile merges (whole block participates in a finalisation)
  bool end_block = false;
  if (ct_first >= 0 && ct_first * m + m <= U1) end_block = true;
  for (int which = 0; which < 2; ++which) {
    const long long ct = which == 0 ? ct_first : ct_last;
    if (ct < 0) continue;
    const int64_t ba = blk_of(ct * m, U, P), bb = blk_of(ct * m + m - 1, U, P);
    __threadfence();  // every thread's tpart stores before the arrival
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(wk.cnt + bb, 1u);
      sflag = (prev == (unsigned)(bb - ba));
    }
    __syncthreads();
    if (sflag) {
      __threadfence();
      const int64_t c = ct * TW + VW * threadIdx.x;
      double y[VW];
#pragma unroll
      for (int j = 0; j < VW; ++j) y[j] = __ldcg(wk.tpart + ((size_t)ba * 2 + 1) * kCW + VW * threadIdx.x + j);
      for (int64_t q = ba + 1; q <= bb; ++q)
#pragma unroll
        for (int j = 0; j < VW; ++j) y[j] += __ldcg(wk.tpart + ((size_t)q * 2) * kCW + VW * threadIdx.x + j);
      double facc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) facc[k] = red_identity(epi.op(k));
#pragma unroll
      for (int j = 0; j < VW; ++j)
        if (c + j < n) epi.elem(c + j, y[j], facc);
      block_reduce<K>(facc, sm, epi);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) wk.facc[bb * kKMax + k] = facc[k];
        wk.cnt[bb] = 0u;
      }
    }
  }
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      wk.bacc[b * kKMax + k] = acc[k];
      if (!end_block) wk.facc[b * kKMax + k] = red_identity(epi.op(k));
    }
  }
  if constexpr (!kP) finish_last(epi, wk, wk.facc, (int)P, sm, &sflag);
}

template <class Epi, int VW>
__global__ void __launch_bounds__(kNT, kTileTBlocks) k_cols_tile(DenseRows A, const double* __restrict__ x,
                                                               XS xs, Epi epi, Work wk) {
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  body_cols_tile<Epi, VW, false, kTileTRows>(A, x, xs, epi, wk, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------- k_rows_wdense ----
// Small dense A v (L2-resident, n <= kWdMaxN; C1 both ways, A^T v over the
// transposed copy): the pass is a chain of dependent latencies, not a stream,
// so the chain is kept as short as it gets — ONE warp per row, the whole x in
// shared memory, the row's first 1024 columns in flight before x is staged,
// the epilogue straight from the warp sum, one block reduction, the last
// block finishes.  No (tile, row) partials, no group counters, no combine
// stage (k_rows_tile_fused on C1: 7.2-8.2 us per pass).  Lane l owns columns
// 64 k + 2 l, 64 k + 2 l + 1; chunk k feeds FMA chain k & 1; lanes are added
// by the xor butterfly.
constexpr int kWdMaxN = 4096;   // x in 32 KB of shared memory
constexpr int kWdChunks = 16;   // 64-column chunks of a row in flight per lane

__host__ __device__ inline bool wdense_fits(int64_t m, int64_t n) {
  return n >= 128 && n <= kWdMaxN && m >= 1 && 8 * m * n <= (32ll << 20);
}
inline int wdense_grid(int64_t m, int sms) {
  int64_t p = (m + kWarps - 1) / kWarps;
  const int64_t pmax = (int64_t)sms * kMinBlocks;
  if (p > pmax) p = pmax;
  return (int)(p < 1 ? 1 : p);
}

template <class Epi>
__global__ void __launch_bounds__(kNT, 2) k_rows_wdense(DenseRows A, const double* __restrict__ x, XS xs, Epi epi,
                                                       Work wk) {
  constexpr int K = Epi::K;
  constexpr int C = kWdChunks;
  __shared__ double sm[kWarps * kKMax];
  __shared__ __align__(16) double xsl[kWdMaxN + 64];
  __shared__ int sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  unsigned long long t_in = 0;  // entry time (thread 0): hoisted work stays inside the accounted interval
  if (threadIdx.x == 0) t_in = globaltimer();
  const int64_t m = A.m, n = A.n, lda = A.lda, P = gridDim.x, b = blockIdx.x;
  const int64_t r0 = m * b / P, r1 = m * (b + 1) / P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // the matrix does not depend on the solver state: the first row's leading
  // chunks are in flight with the state word and the x slab
  double2 v[C];
  auto load = [&](int64_t r, int64_t c0) {
    const double* row = A.a + r * lda + 2 * lane;
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int64_t c = c0 + 64 * k + 2 * lane;
      v[k] = c < lda ? ld_stream2(row + c0 + 64 * k) : make_double2(0.0, 0.0);
    }
  };
  int64_t r = r0 + wid;
  if (r < r1) load(r, 0);
  // x is complete (the previous kernel wrote it): its loads go out before the state word too
  const int npad = (int)((n + 63) & ~(int64_t)63);
  double xr[kWdMaxN / kNT];
#pragma unroll
  for (int q = 0; q < kWdMaxN / kNT; ++q) {
    const int k = threadIdx.x + q * kNT;
    xr[q] = k < n ? __ldg(x + k) : 0.0;
  }
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  xs.load();
  ktimer_begin_at(epi.timer(), t_in);
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
#pragma unroll
  for (int q = 0; q < kWdMaxN / kNT; ++q) {
    const int k = threadIdx.x + q * kNT;
    if (k < npad) xsl[k] = k < n ? xs(xr[q]) : 0.0;
  }
  __syncthreads();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  bool first = true;
  for (; r < r1; r += kWarps) {
    double a0 = 0.0, a1 = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += 64 * C) {
      if (!(first && c0 == 0)) load(r, c0);
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
    if (lane == 0) epi.elem(r, y, acc);
  }
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[blockIdx.x * kKMax + k] = acc[k];
  }
  finish_last(epi, wk, nullptr, (int)gridDim.x, sm, &sflag);
}

// ---------------------------------------------------------- k_pair_wdense ----
// One CTA moments pair q = A^T p, p' = A q in ONE cooperative kernel for a small
// L2-resident dense matrix (C1; both orientations on the warp-per-row scheme,
// A^T from the transposed copy).  Phase 1 computes this block's rows of q and
// runs the q epilogue on them; a grid barrier makes q complete; phase 2 stages
// q in shared memory and computes the block's rows of p' with the p' epilogue.
// Against two kernels this saves the first kernel's whole reduction chain
// (block sums -> arrival -> last block -> finisher), a kernel boundary and the
// second state read; A's first rows are in flight across the barrier.  One
// reduction for both epilogues' sums, the last block finishes both.  Row
// arithmetic and each phase's row -> (block, warp) mapping are k_rows_wdense's,
// so q, p' and their block sums are the bits of the two passes.
// Grid barrier of a cooperative launch (every block resident).  The counter only
// grows inside a kernel: barrier number k waits for k * nblocks arrivals, one
// atomic and one polled load per block; the kernel's last block (its final
// arrival) puts the counter back to zero for the next launch.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(count, 1u);
    unsigned c;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(count) : "memory");
    } while (c < target);
  }
  __syncthreads();
}

// XN: vector entries per thread staged through registers (vectors of <= XN * 256 entries)
template <class EpiQ, class EpiP, int XN>
__global__ void __launch_bounds__(kNT, 2) k_pair_wdense(const __grid_constant__ DenseRows AT,
                                                       const __grid_constant__ DenseRows A, const double* pprev,
                                                       const double* q, const __grid_constant__ EpiQ eq,
                                                       const __grid_constant__ EpiP ep,
                                                       const __grid_constant__ Work wk, int PT, int PN) {
  constexpr int KQ = EpiQ::K, KP = EpiP::K, K = KQ + KP;
  constexpr int C = kWdChunks;
  __shared__ double sm[kWarps * kKMax];
  __shared__ __align__(16) double xsl[kWdMaxN + 64];
  __shared__ int sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) ep.count_launch();
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
  // rows [r0, r1) of D times the vector staged in xsl; `first`: row r's leading chunks are loaded
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
  auto stage = [&](const double (&xr)[XN], int64_t n) {
    const int npad = (int)((n + 63) & ~(int64_t)63);
#pragma unroll
    for (int u = 0; u < XN; ++u) {
      const int k = threadIdx.x + u * kNT;
      if (k < npad) xsl[k] = k < n ? xr[u] : 0.0;
    }
  };
  // ---- phase 1: q = A^T p on rows [t0, t1) of the transposed copy
  // (each phase keeps the row split of its stand-alone pass: blocks [0, PT) / [0, PN))
  const int64_t t0 = b < PT ? AT.m * b / PT : 0, t1 = b < PT ? AT.m * (b + 1) / PT : 0;
  int64_t r = t0 + wid;
  if (r < t1) load(AT, r, 0);
  double xr[XN];
#pragma unroll
  for (int u = 0; u < XN; ++u) {
    const int k = threadIdx.x + u * kNT;
    xr[u] = k < AT.n ? __ldg(pprev + k) : 0.0;  // p is complete: written by an earlier kernel
  }
  if (!ep.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ep.idle();
    return;
  }
  ktimer_begin_at(ep.timer(), t_in);
  stage(xr, AT.n);
  __syncthreads();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  double (&aq)[KQ] = *reinterpret_cast<double (*)[KQ]>(&acc[0]);
  double (&ap)[KP] = *reinterpret_cast<double (*)[KP]>(&acc[KQ]);
  rows(AT, r, t1, [&](int64_t row, double y) { eq.elem(row, y, aq); });
  // ---- A's first rows in flight across the barrier (the matrix is immutable)
  const int64_t r0 = b < PN ? A.m * b / PN : 0, r1 = b < PN ? A.m * (b + 1) / PN : 0;
  r = r0 + wid;
  if (r < r1) load(A, r, 0);
  grid_barrier(wk.done + 2, (unsigned)P);
  // ---- phase 2: p' = A q; q was written inside this kernel: L2-coherent loads
#pragma unroll
  for (int u = 0; u < XN; ++u) {
    const int k = threadIdx.x + u * kNT;
    xr[u] = k < A.n ? __ldcg(q + k) : 0.0;
  }
  stage(xr, A.n);
  __syncthreads();
  rows(A, r, r1, [&](int64_t row, double y) { ep.elem(row, y, ap); });
  const OpsSum ops;
  block_reduce<K>(acc, sm, ops);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[b * kKMax + k] = acc[k];
  }
  if (arrive_last(wk.done, (unsigned)P, &sflag)) {
    if (threadIdx.x == 0) wk.done[2] = 0u;  // the barrier counter, for the next launch
    double red[K];
    reduce_partials<K>(wk.bacc, nullptr, (int)P, red, sm, ops);
    if (threadIdx.x == 0) {
      ktimer_end(ep.timer(), 2);
      double rq[KQ], rp2[KP];
#pragma unroll
      for (int k = 0; k < KQ; ++k) rq[k] = red[k];
#pragma unroll
      for (int k = 0; k < KP; ++k) rp2[k] = red[KQ + k];
      eq.finish(rq);
      ep.finish(rp2);
    }
    __syncthreads();
    ep.finish_block();
  }
}

// ------------------------------------------------------ k_rows_tile_fused ----
// Dense A v in ONE kernel.  The (tile, row) units are ordered group-major:
// 256-row groups one after another, inside a group tile by tile, so a group's
// 512-column tiles are produced by consecutive blocks and groups complete
// progressively while the rest of the matrix streams.  Each block, after a
// segment (one tile of rows of one group), adds the rows it finished to the
// group's counter; the block that completes a group combines it at once: one
// thread per row sums the row's tile partials in tile order, runs the
// epilogue, and the block's reduction lands in the group's slot gacc[g]; the
// last block to arrive reduces the slots in group order.  Only the last
// group's combine is left on the tail, instead of a second kernel (C2:
// k_rows_tile + k_tile_combine 137 us).  Work::npart = [m x tiles partials |
// gacc | group counters] (zeroed once, self-resetting).
constexpr int kGroupRows = kNT;  // rows per combine group: one per thread
// tools/microbench/dense_av.cu on C2: 141 us with the slice in registers and
// one chunk per warp at 4 blocks/SM, 124 us (6.44 TB/s) with 2 row chunks in
// flight per warp at 2 blocks/SM
constexpr int kTileNBlocks = 2;  // blocks per SM (128 registers)
constexpr int kTileNRows = 2;    // row chunks in flight per warp

__host__ __device__ inline int64_t tile_groups(int64_t m) { return (m + kGroupRows - 1) / kGroupRows; }

template <class Epi>
__global__ void __launch_bounds__(kNT, kTileNBlocks) k_rows_tile_fused(DenseRows A, const double* __restrict__ x,
                                                                     XS xs, Epi epi, Work wk) {
  constexpr int K = Epi::K;
  constexpr int TW = 2 * kNT;
  constexpr int R = kTileNRows;
  __shared__ double sm[kWarps * kKMax];
  __shared__ __align__(16) double xsl[TW];
  __shared__ int sdone, sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  xs.load();
  ktimer_begin(epi.timer());
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
  const int64_t P = gridDim.x, b = blockIdx.x;
  const int64_t m = A.m, n = A.n, lda = A.lda, nct = (n + TW - 1) / TW;
  const int64_t ng = tile_groups(m), GU = nct * kGroupRows;
  const int64_t U = nct * m, U0 = U * b / P, U1 = U * (b + 1) / P;
  double* part = wk.npart;
  double* gacc = part + nct * m;
  unsigned* gcnt = reinterpret_cast<unsigned*>(gacc + ng * kKMax);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto dot = [&](const double2 (&v)[8]) -> double {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const double2 x0 = *reinterpret_cast<const double2*>(xsl + 64 * k + 2 * lane);
      const double2 x1 = *reinterpret_cast<const double2*>(xsl + 64 * (k + 1) + 2 * lane);
      a0 = fma(v[k].x, x0.x, a0); a0 = fma(v[k].y, x0.y, a0);
      a1 = fma(v[k + 1].x, x1.x, a1); a1 = fma(v[k + 1].y, x1.y, a1);
    }
    return warp_reduce(a0 + a1, RED_SUM);
  };
  for (int64_t u = U0; u < U1;) {
    const int64_t g = (u / GU < ng - 1) ? u / GU : ng - 1;
    const int64_t gb = g * kGroupRows, rows_g = (m - gb < kGroupRows) ? m - gb : kGroupRows;
    const int64_t off = u - g * GU, ct = off / rows_g, rr = off - ct * rows_g;
    const int64_t seg = (rows_g - rr < U1 - u) ? rows_g - rr : U1 - u;
    const int64_t r0 = gb + rr, r1 = r0 + seg, cb = ct * TW;
    const bool full = cb + TW <= n;
    __syncthreads();  // previous slice consumed
    for (int k = threadIdx.x; k < TW; k += kNT) xsl[k] = (cb + k < n) ? xs(__ldg(x + cb + k)) : 0.0;
    __syncthreads();
    int64_t r = r0 + wid;
    if (full) {
      for (; r + 8 * (R - 1) < r1; r += 8 * R) {
        double2 v[R][8];
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) v[q][k] = ld_stream2(A.a + (r + 8 * q) * lda + cb + 2 * lane + 64 * k);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const double sum = dot(v[q]);
          if (lane == 0) part[(r + 8 * q) * nct + ct] = sum;
        }
      }
      for (; r < r1; r += 8) {
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ld_stream2(A.a + r * lda + cb + 2 * lane + 64 * k);
        const double sum = dot(v);
        if (lane == 0) part[r * nct + ct] = sum;
      }
    } else {
      for (; r < r1; r += 8) {
        const double* row = A.a + r * lda + cb + 2 * lane;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t c = cb + 64 * k + 2 * lane;
          if (c < n) a0 = fma(ld_stream(row + 64 * k), xsl[64 * k + 2 * lane], a0);
          if (c + 1 < n) a1 = fma(ld_stream(row + 64 * k + 1), xsl[64 * k + 2 * lane + 1], a1);
        }
        const double sum = warp_reduce(a0 + a1, RED_SUM);
        if (lane == 0) part[r * nct + ct] = sum;
      }
    }
    // the rows of this segment are in: count them for group g
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned add = (unsigned)seg;
      sdone = (atomicAdd(gcnt + g, add) + add == (unsigned)(nct * rows_g)) ? 1 : 0;
    }
    __syncthreads();
    if (sdone) {  // this block completed group g: combine it (thread per row, tiles in order)
      __threadfence();
      double acc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
      const int64_t row = gb + threadIdx.x;
      if (threadIdx.x < rows_g) {
        // tiles in order; with many tiles (C2: 40) the loads of 16 tiles are
        // issued before their adds, so the group's combine on the kernel's
        // tail costs ~nct/16 L2 round trips (C2 A v 135.5 -> 132.4 us)
        const double* pr = part + row * nct;
        double y = __ldcg(pr);
        if (nct < 16) {
          for (int64_t t = 1; t < nct; ++t) y += __ldcg(pr + t);
        } else {
          for (int64_t t = 1; t < nct; t += 16) {
            double p[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) p[q] = (t + q < nct) ? __ldcg(pr + t + q) : 0.0;
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (t + q < nct) y += p[q];
          }
        }
        epi.elem(row, y, acc);
      }
      block_reduce<K>(acc, sm, epi);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) gacc[g * kKMax + k] = acc[k];
        gcnt[g] = 0u;  // self-reset for the next launch
      }
    }
    u += seg;
  }
  if (arrive_last(wk.done, (unsigned)P, &sflag)) {
    double red[K];
    reduce_partials<K>(gacc, nullptr, (int)ng, red, sm, epi);
    if (threadIdx.x == 0) {
      ktimer_end(epi.timer());
      epi.finish(red);
    }
    __syncthreads();
    epi.finish_block();
  }
}

// ----------------------------------------------------------------- k_vec ----
// `prepared`: the caller has run epi.prepare() already (k_vec: ahead of the
// activity test, so the two state reads overlap)
template <class Epi, bool kP>
__device__ __forceinline__ void body_vec(int64_t len, Epi& epi, const Work& wk, int64_t b, int64_t P,
                                         bool prepared = false) {
  constexpr int K = Epi::K;
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  ktimer_begin(epi.timer());
  __shared__ double epi_smem[kEpiSmem];
  if (!prepared) epi.prepare(epi_smem);
  __syncthreads();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  const int64_t stride = P * kNT;
  if constexpr (kPairOf<Epi>) {
    // pair epilogues: elements (2i, 2i+1) per call with 128-bit loads (twice
    // the bytes in flight per thread on the multi-vector CTA passes)
    const int64_t np = (len + 1) >> 1;
    for (int64_t ip = b * kNT + threadIdx.x; ip < np; ip += stride) epi.elem2(2 * ip, acc);
  } else {
    for (int64_t i = b * kNT + threadIdx.x; i < len; i += stride) epi.elem(i, acc);
  }
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[b * kKMax + k] = acc[k];
  }
  if constexpr (!kP) finish_last(epi, wk, nullptr, (int)P, sm, &sflag);
}

template <class Epi>
__global__ void __launch_bounds__(kNT, kVecBlocksOf<Epi>) k_vec(int64_t len, Epi epi, Work wk) {
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  // the epilogue's scalars (shared memory only: no side effect) are fetched
  // together with the words the activity test reads: one round trip, not two
  __shared__ double pre_smem[kEpiSmem];
  epi.prepare(pre_smem);
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  body_vec<Epi, false>(len, epi, wk, blockIdx.x, gridDim.x, true);
}

// Two single-block vector passes in one kernel (systems of <= 1024 unknowns: the
// CTA candidate and update passes of C1): the second pass starts after the first
// one's finisher has written the state, in the same block — one launch, one
// kernel boundary less.  Each pass keeps its own activity test, accounting,
// thread <-> element mapping and finisher.
template <class EA, class EB>
__global__ void __launch_bounds__(kNT, (kVecBlocksOf<EA> < kVecBlocksOf<EB> ? kVecBlocksOf<EA> : kVecBlocksOf<EB>))
    k_vec2(int64_t len_a, EA ea, int64_t len_b, EB eb, Work wk) {
  if (threadIdx.x == 0) ea.count_launch();
  if (!ea.active()) {
    if (threadIdx.x == 0) ea.idle();
  } else {
    body_vec<EA, false>(len_a, ea, wk, 0, 1);
  }
  __syncthreads();  // the first finisher's state, visible to the whole block
  if (!eb.active()) {
    if (threadIdx.x == 0) eb.idle();
    return;
  }
  body_vec<EB, false>(len_b, eb, wk, 0, 1);
}

}  // namespace ts
