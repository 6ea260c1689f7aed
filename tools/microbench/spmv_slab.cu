// Long-row CSR A v (C5: 1e4 rows x 1e6 columns, ~1000 entries per row) as
// column slabs, one per SM (design study for the library's k_slab_av; not
// part of the library).
//
// The columns are cut into P = #SM slabs of equal nnz.  Inside slab s the
// rows are sorted by their in-slab length (descending) and cut into slices of
// 32; a slice stores its rows interleaved (SELL-32-sigma: entry k of lane l at
// sp + 32 k + l), values fp64, in-slab column offsets u16 (padding 0xFFFF).
// One 1024-thread block per slab stages the slab's x (<= 64 K columns) in
// shared memory, so every gather is a shared-memory read; each warp streams a
// contiguous run of slices as ONE coalesced stream (U loads in flight per
// lane, slice boundaries from registers, no per-slice pointer chase) and
// writes each row's partial to part[s][row].  A second kernel sums the P
// partials of every row in fixed slab order.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/microbench/spmv_slab tools/microbench/spmv_slab.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_stream_u16(const unsigned short* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream_i(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// L2 eviction-priority hints (createpolicy): the matrix stream is evict_first,
// so it does not push x, the position table and the partials out of L2
__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_stream_h(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned ld_stream_u16_h(const unsigned short* p, unsigned long long pol) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_keep_i(const int* p, unsigned long long pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(double* p, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

struct SlabStream {
  int m, n, P, nsl;      // rows, columns, slabs, slices per slab
  const int* cb;         // [P + 1] slab column boundaries
  const int* sp;         // [P * nsl + 1] slot offset of every slice (global)
  const int* wr;         // [P * 33] first slice (in-slab) of each warp's run
  const int* perm;       // [P * nsl * 32] row of (slice, lane), -1 past m
  const unsigned short* col;
  const double* val;
};

constexpr int kT = 1024;
constexpr int kW = kT / 32;

template <int U>
__global__ void __launch_bounds__(kT, 1) k_slab(SlabStream S, const double* __restrict__ x,
                                                double* __restrict__ part) {
  extern __shared__ double xs[];
  const int s = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cb0 = S.cb[s], cw = S.cb[s + 1] - cb0;
  const int q0 = S.wr[s * 33 + w], q1 = S.wr[s * 33 + w + 1];
  // first chunk's slice boundaries and the first slice's rows: in flight
  // together with the x slab loads
  const int g0 = s * S.nsl;
  int nq = min(q1 - q0, 31);
  int bnd = (lane <= nq && q0 < q1) ? __ldg(S.sp + g0 + q0 + lane) : 0;
  int prow = (q0 < q1) ? __ldg(S.perm + (size_t)(g0 + q0) * 32 + lane) : -1;
  for (int i = threadIdx.x; i < cw; i += kT) xs[i] = __ldg(x + cb0 + i);
  __syncthreads();
  double* out = part + (size_t)s * S.m;
  for (int qc = q0; qc < q1;) {
    nq = min(q1 - qc, 31);
    const int gq = g0 + qc;
    const int e0 = __shfl_sync(0xffffffffu, bnd, 0);
    const int K = (__shfl_sync(0xffffffffu, bnd, nq) - e0) >> 5;
    int j = 0;
    int kend = (__shfl_sync(0xffffffffu, bnd, 1) - e0) >> 5;
    int row = prow;
    prow = (nq > 1) ? __ldg(S.perm + (size_t)(gq + 1) * 32 + lane) : -1;
    double acc = 0.0;
    auto emit = [&]() {
      if (row >= 0) out[row] = acc;
      acc = 0.0;
      ++j;
      row = prow;
      if (j + 1 < nq) prow = __ldg(S.perm + (size_t)(gq + j + 1) * 32 + lane);
      kend = (__shfl_sync(0xffffffffu, bnd, min(j + 1, nq)) - e0) >> 5;
    };
    const double* vp = S.val + e0 + lane;
    const unsigned short* cp = S.col + e0 + lane;
    for (int k0 = 0; k0 < K; k0 += U) {
      double v[U];
      unsigned c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = k0 + u < K;
        v[u] = ok ? ld_stream(vp + 32 * (k0 + u)) : 0.0;
        c[u] = ok ? ld_stream_u16(cp + 32 * (k0 + u)) : 0xFFFFu;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u;
        if (k >= K) break;
        while (k == kend && j < nq) emit();
        if (c[u] != 0xFFFFu) acc = fma(v[u], xs[c[u]], acc);
      }
    }
    while (j < nq) emit();
    qc += nq;
    if (qc < q1) {  // next chunk of boundaries and its first slice's rows
      const int nn = min(q1 - qc, 31);
      bnd = (lane <= nn) ? __ldg(S.sp + g0 + qc + lane) : 0;
      prow = __ldg(S.perm + (size_t)(g0 + qc) * 32 + lane);
    }
  }
}


// ---------------------------------------------------------------- TMA ring --
// The same slab layout streamed through per-warp shared-memory rings by bulk
// copies (cp.async.bulk + mbarrier): each warp's run of slices is ONE
// contiguous range of val[] and col[], so lane 0 keeps ST chunks of CH slots in
// flight for its warp, independent of the register budget; the consumer reads
// its operands from shared memory, lane-contiguous (conflict-free).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{ .reg .pred p; TS_WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; "
      "@!p bra TS_WAIT_%=; }" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// MODE 0: full kernel; 1: no partial stores; 2: no x gather (constant)
template <int NW, int ST, int CH, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) k_slab_tma(SlabStream S, const double* __restrict__ x,
                                                         double* __restrict__ part, int xcap) {
  constexpr int CK_ = CH / 32;  // k-steps per chunk
  extern __shared__ __align__(128) unsigned char raw[];
  double* xs = reinterpret_cast<double*>(raw);                           // [xcap]
  double* rv = xs + xcap;                                                // [NW][ST][CH]
  unsigned short* rc = reinterpret_cast<unsigned short*>(rv + (size_t)NW * ST * CH);  // [NW][ST][CH]
  __shared__ __align__(8) unsigned long long full[NW * ST];
  const int s = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int RUNS = 32 / NW;  // warp runs of the table per warp
  const int cb0 = S.cb[s], cw = S.cb[s + 1] - cb0;
  const int q0 = S.wr[s * 33 + w * RUNS], q1 = S.wr[s * 33 + (w + 1) * RUNS];
  const int g0 = s * S.nsl;
  const int E0 = __ldg(S.sp + g0 + q0), E1 = __ldg(S.sp + g0 + q1);
  const int KT = (E1 - E0) >> 5;             // k-steps of this warp
  const int NC = (KT + CK_ - 1) / CK_;       // chunks
  double* mv = rv + (size_t)w * ST * CH;
  unsigned short* mc = rc + (size_t)w * ST * CH;
  unsigned long long* mb = full + w * ST;
  auto issue = [&](int c) {  // lane 0
    const int st = c % ST;
    const int e = E0 + c * CH;
    const int cnt = min(CH, E1 - e);
    mbar_expect_tx(&mb[st], (unsigned)cnt * 10u);
    bulk_g2s(mv + st * CH, S.val + e, (unsigned)cnt * 8u, &mb[st]);
    bulk_g2s(mc + st * CH, S.col + e, (unsigned)cnt * 2u, &mb[st]);
  };
  if (lane == 0) {
    for (int i = 0; i < ST; ++i) mbar_init(&mb[i], 1);
    fence_mbar_init();
    for (int c = 0; c < ST && c < NC; ++c) issue(c);
  }
  int nq = min(q1 - q0, 31);
  int bnd = (lane <= nq && q0 < q1) ? __ldg(S.sp + g0 + q0 + lane) : 0;
  int prow = (q0 < q1) ? __ldg(S.perm + (size_t)(g0 + q0) * 32 + lane) : -1;
  for (int i = threadIdx.x; i < cw; i += NW * 32) xs[i] = __ldg(x + cb0 + i);
  __syncthreads();
  double* out = part + (size_t)s * S.m;
  // slice bookkeeping: bounds of up to 31 slices live across the lanes of bnd
  int qc = q0, j = 0;
  int row = prow;
  prow = (nq > 1) ? __ldg(S.perm + (size_t)(g0 + qc + 1) * 32 + lane) : -1;
  int kend = (q0 < q1) ? (__shfl_sync(0xffffffffu, bnd, 1) - E0) >> 5 : 0;
  double acc = 0.0;
  auto emit = [&]() {  // the slice's rows are complete
    if (MODE != 1) { if (row >= 0) out[row] = acc; }
    acc = 0.0;
    ++j;
    if (j == nq) {  // next group of slice bounds
      qc += nq;
      j = 0;
      nq = min(q1 - qc, 31);
      if (nq > 0) {
        bnd = (lane <= nq) ? __ldg(S.sp + g0 + qc + lane) : 0;
        row = __ldg(S.perm + (size_t)(g0 + qc) * 32 + lane);
        prow = (nq > 1) ? __ldg(S.perm + (size_t)(g0 + qc + 1) * 32 + lane) : -1;
        kend = (__shfl_sync(0xffffffffu, bnd, 1) - E0) >> 5;
      } else {
        kend = 0x7fffffff;
      }
      return;
    }
    row = prow;
    if (j + 1 < nq) prow = __ldg(S.perm + (size_t)(g0 + qc + j + 1) * 32 + lane);
    kend = (__shfl_sync(0xffffffffu, bnd, j + 1) - E0) >> 5;
  };
  for (int c = 0; c < NC; ++c) {
    const int st = c % ST;
    mbar_wait(&mb[st], (unsigned)((c / ST) & 1));
    const double* cv = mv + st * CH + lane;
    const unsigned short* cc = mc + st * CH + lane;
    const int kb = c * CK_;
    const int kn = min(CK_, KT - kb);
    constexpr int U = 8;
    for (int k0 = 0; k0 < kn; k0 += U) {
      double v[U];
      unsigned ci_[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = k0 + u < kn;
        v[u] = ok ? cv[32 * (k0 + u)] : 0.0;
        ci_[u] = ok ? cc[32 * (k0 + u)] : 0xFFFFu;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = (MODE == 2) ? 1.0 : (ci_[u] != 0xFFFFu ? xs[ci_[u]] : 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kb + k0 + u;
        if (k0 + u >= kn) break;
        while (k == kend) emit();
        if (ci_[u] != 0xFFFFu) acc = fma(v[u], xv[u], acc);
      }
    }
    __syncwarp();
    if (lane == 0 && c + ST < NC) issue(c + ST);
  }
  while (qc < q1 && nq > 0) emit();
}


// ------------------------------------------------- smem-accumulated slab ----
// Variant 2: (a) every slice's row sums go to shared memory in SLICE order
// (conflict-free), no permutation load and no scattered global store inside
// the stream; the block writes part[s][0..m) coalesced at the end through the
// inverse permutation; (b) the slab's slice offsets live in shared memory;
// (c) PIPE: register double buffering, the next batch of U k-steps is in
// flight while the current one is consumed.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned map_peer(const void* p, unsigned rank) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_dsmem(unsigned addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int NW, int U, int PIPE, int CL = 1, int HINT = 0>
__global__ void __launch_bounds__(NW * 32, 1) k_slab2(SlabStream S, const int* __restrict__ inv,
                                                      const double* __restrict__ x, double* __restrict__ part,
                                                      int xcap, unsigned long long* ts) {
  extern __shared__ __align__(16) unsigned char raw2[];
  double* xs = reinterpret_cast<double*>(raw2);   // [xcap]
  double* accs = xs + xcap;                       // [nsl * 32]
  int* sps = reinterpret_cast<int*>(accs + (size_t)S.nsl * 32);  // [nsl + 1]
  __shared__ unsigned long long tl;
  constexpr int NT_ = NW * 32;
  constexpr int RUNS = 32 / NW;
  const int s = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (ts && threadIdx.x == 0) { ts[s * 4 + 0] = gtimer(); tl = 0; }
  const int cb0 = S.cb[s], cw = S.cb[s + 1] - cb0;
  const int q0 = S.wr[s * 33 + w * RUNS], q1 = S.wr[s * 33 + (w + 1) * RUNS];
  const int g0 = s * S.nsl;
  const int E0 = __ldg(S.sp + g0 + q0), E1 = __ldg(S.sp + g0 + q1);
  const int KT = (E1 - E0) >> 5;
  const double* vp = S.val + E0 + lane;
  const unsigned short* cp = S.col + E0 + lane;
  double va[U], vb[U];
  unsigned ca[U], cbf[U];
  const unsigned long long pf = HINT ? pol_first() : 0ull, pl = HINT ? pol_last() : 0ull;
  auto load = [&](double (&v)[U], unsigned (&c)[U], int k0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = k0 + u < KT;
      if (HINT) {
        v[u] = ok ? ld_stream_h(vp + 32 * (k0 + u), pf) : 0.0;
        c[u] = ok ? ld_stream_u16_h(cp + 32 * (k0 + u), pf) : 0xFFFFu;
      } else {
        v[u] = ok ? ld_stream(vp + 32 * (k0 + u)) : 0.0;
        c[u] = ok ? ld_stream_u16(cp + 32 * (k0 + u)) : 0xFFFFu;
      }
    }
  };
  load(va, ca, 0);  // in flight with the staging below
  for (int i = threadIdx.x; i <= S.nsl; i += NT_) sps[i] = HINT ? ld_keep_i(S.sp + g0 + i, pl) : __ldg(S.sp + g0 + i);
  for (int i = threadIdx.x; i < cw; i += NT_) xs[i] = HINT ? ld_keep(x + cb0 + i, pl) : __ldg(x + cb0 + i);
  __syncthreads();
  if (ts && threadIdx.x == 0) ts[s * 4 + 1] = gtimer();
  int q = q0;
  int kend = q0 < q1 ? (sps[q0 + 1] - E0) >> 5 : 0x7fffffff;
  double acc = 0.0;
  auto emit = [&]() {
    accs[q * 32 + lane] = acc;
    acc = 0.0;
    ++q;
    kend = q < q1 ? (sps[q + 1] - E0) >> 5 : 0x7fffffff;
  };
  auto consume = [&](const double (&v)[U], const unsigned (&c)[U], int k0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u;
      if (k >= KT) break;
      while (k == kend) emit();
      if (c[u] != 0xFFFFu) acc = fma(v[u], xs[c[u]], acc);
    }
  };
  if (PIPE) {
    for (int k0 = 0; k0 < KT; k0 += 2 * U) {
      load(vb, cbf, k0 + U);
      consume(va, ca, k0);
      load(va, ca, k0 + 2 * U);
      consume(vb, cbf, k0 + U);
    }
  } else {
    for (int k0 = 0; k0 < KT; k0 += U) {
      if (k0) load(va, ca, k0);
      consume(va, ca, k0);
    }
  }
  while (q < q1) emit();
  if (ts && lane == 0) atomicMax(&tl, gtimer());
  __syncthreads();
  if (ts && threadIdx.x == 0) ts[s * 4 + 2] = tl;
  if (CL == 1) {
    double* out = part + (size_t)s * S.m;
    const int* iv = inv + (size_t)s * S.m;
    if (HINT) {
      for (int r = threadIdx.x; r < S.m; r += NT_) st_keep(out + r, accs[ld_keep_i(iv + r, pl)], pl);
    } else {
      for (int r = threadIdx.x; r < S.m; r += NT_) out[r] = accs[__ldg(iv + r)];
    }
  } else {
    // pair reduce over distributed shared memory: block `rank` of the pair owns
    // rows [rank m/2, (rank+1) m/2): slab 2c's sum + slab 2c+1's sum, in that order
    cluster_sync_all();
    const int rank = s & 1, c = s >> 1;
    const unsigned a0 = map_peer(accs, 0), a1 = map_peer(accs, 1);
    const int* iv0 = inv + (size_t)(2 * c) * S.m;
    const int* iv1 = iv0 + S.m;
    double* out = part + (size_t)c * S.m;
    const int rb = rank ? S.m / 2 : 0, re = rank ? S.m : S.m / 2;
    for (int r = rb + threadIdx.x; r < re; r += NT_) {
      const int i0 = __ldg(iv0 + r), i1 = __ldg(iv1 + r);
      out[r] = ld_dsmem(a0 + 8u * i0) + ld_dsmem(a1 + 8u * i1);
    }
    cluster_sync_all();
  }
  if (ts) {
    __syncthreads();
    if (threadIdx.x == 0) ts[s * 4 + 3] = gtimer();
  }
}

// 32 rows per block; warp g adds slabs g, g + 8, ... (4 loads in flight), the
// 8 warp sums are combined in warp order: a fixed order
__global__ void __launch_bounds__(256) k_sum(const double* __restrict__ part, int m, int P, double* y) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + lane;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (r < m) {
    int q = g;
    for (; q + 24 < P; q += 32) {
      s0 += __ldcg(part + (size_t)q * m + r);
      s1 += __ldcg(part + (size_t)(q + 8) * m + r);
      s2 += __ldcg(part + (size_t)(q + 16) * m + r);
      s3 += __ldcg(part + (size_t)(q + 24) * m + r);
    }
    for (; q < P; q += 8) s0 += __ldcg(part + (size_t)q * m + r);
  }
  red[g][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (g == 0 && r < m) {
    double t = red[0][lane];
    for (int j = 1; j < 8; ++j) t += red[j][lane];
    y[r] = t;
  }
}

// 32 rows per block of 1024 threads: warp g adds slabs g, g + 32, ... (all
// its ~P/32 loads in flight at once), then the 32 warp sums are combined in
// warp order
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_sum32(const double* __restrict__ part, int m, int P, double* y) {
  __shared__ double red[NW][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (r < m) {
    constexpr int L = 8;  // loads per batch
    int q = g;
    for (; q + (L - 1) * NW < P; q += L * NW) {
      double t[L];
#pragma unroll
      for (int u = 0; u < L; ++u) t[u] = __ldcg(part + (size_t)(q + u * NW) * m + r);
#pragma unroll
      for (int u = 0; u < L; ++u) s += t[u];
    }
    for (; q < P; q += NW) s += __ldcg(part + (size_t)q * m + r);
  }
  red[g][lane] = s;
  __syncthreads();
  if (g == 0 && r < m) {
    double t = red[0][lane];
    for (int j = 1; j < NW; ++j) t += red[j][lane];
    y[r] = t;
  }
}

// 32 rows per block; warp g adds the contiguous slab range [g P / NW, (g + 1) P / NW)
// with up to L loads in flight, then the NW warp sums are added in warp order
template <int NW, int L>
__global__ void __launch_bounds__(NW * 32) k_sumA(const double* __restrict__ part, int m, int P, double* y) {
  __shared__ double red[NW][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + lane;
  const int qa = P * g / NW, qb = P * (g + 1) / NW;
  double s = 0.0;
  if (r < m) {
    int q = qa;
    for (; q < qb; q += L) {
      double t[L];
#pragma unroll
      for (int u = 0; u < L; ++u) t[u] = q + u < qb ? __ldcg(part + (size_t)(q + u) * m + r) : 0.0;
#pragma unroll
      for (int u = 0; u < L; ++u) s += t[u];
    }
  }
  red[g][lane] = s;
  __syncthreads();
  if (g == 0 && r < m) {
    double t = red[0][lane];
    for (int j = 1; j < NW; ++j) t += red[j][lane];
    y[r] = t;
  }
}

// library baseline: warp per row, next chunks prefetched (k_rows_wrow)
constexpr int kWrowU = 6;
__global__ void __launch_bounds__(256, 3) k_wrow(const int* rp, const int* ci, const double* val, int m,
                                                 const double* __restrict__ x, double* y) {
  constexpr int U = kWrowU;
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * 256) >> 5;
  for (long long r = w; r < m; r += W) {
    const int k0 = __ldg(rp + r), k1 = __ldg(rp + r + 1);
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    double pv[U];
    int pj[U];
    int k = k0 + lane;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = k + 32 * u;
      pv[u] = kk < k1 ? ld_stream(val + kk) : 0.0;
      pj[u] = kk < k1 ? ld_stream_i(ci + kk) : 0;
    }
    for (; k < k1; k += 32 * U) {
      double v[U];
      int j[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { v[u] = pv[u]; j[u] = pj[u]; }
      const int kn = k + 32 * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kn + 32 * u;
        pv[u] = kk < k1 ? ld_stream(val + kk) : 0.0;
        pj[u] = kk < k1 ? ld_stream_i(ci + kk) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], __ldg(x + j[u]), a[u & 3]);
    }
    double t = (a[0] + a[1]) + (a[2] + a[3]);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) y[r] = t;
  }
}

// ------------------------------------------------------------------ host ----
static double* g_flush = nullptr;
static void flush_l2() {
  if (!g_flush) CK(cudaMalloc(&g_flush, 256 << 20));
  CK(cudaMemset(g_flush, 1, 256 << 20));
}
template <class F>
static float timeit(F f, int reps = 20, bool flush = true) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  std::vector<float> t;
  for (int i = 0; i < reps; ++i) {
    if (flush) flush_l2();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}
template <class T>
static T* up(const std::vector<T>& v) {
  T* p;
  CK(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)));
  CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

int main() {
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, 0));
  const int P = pr.multiProcessorCount;
  const int m = 10000, n = 1000000;
  // C5: 10 distinct random rows per column, values U(0.1, 1)
  std::mt19937_64 g(5);
  std::uniform_int_distribution<int> ui(0, m - 1);
  std::uniform_real_distribution<double> ur(0.1, 1.0);
  std::vector<int> rows(10LL * n);
  std::vector<double> vals(10LL * n);
  for (int j = 0; j < n; ++j) {
    int c[10];
    for (int i = 0; i < 10; ++i) {
      bool dup;
      do { c[i] = ui(g); dup = false; for (int q = 0; q < i; ++q) dup |= c[q] == c[i]; } while (dup);
    }
    std::sort(c, c + 10);
    for (int i = 0; i < 10; ++i) { rows[10LL * j + i] = c[i]; vals[10LL * j + i] = ur(g); }
  }
  // CSR of A (columns ascending per row)
  std::vector<int> rp(m + 1, 0), ci(rows.size());
  std::vector<double> v(rows.size());
  for (int r : rows) rp[r + 1]++;
  for (int r = 0; r < m; ++r) rp[r + 1] += rp[r];
  {
    std::vector<int> pos(rp.begin(), rp.end() - 1);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < 10; ++i) {
        const int e = pos[rows[10LL * j + i]]++;
        ci[e] = j;
        v[e] = vals[10LL * j + i];
      }
  }
  const long long nnz = (long long)ci.size();
  const double bytes = 12.0 * nnz + 4.0 * (m + 1) + 8.0 * (m + n);
  std::vector<double> hx(n);
  std::uniform_real_distribution<double> ux(-1, 1);
  for (auto& e : hx) e = ux(g);
  std::vector<long double> yr(m);
  for (int r = 0; r < m; ++r) {
    long double s = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) s += (long double)v[k] * hx[ci[k]];
    yr[r] = s;
  }
  // ---- slab layout: equal-nnz column slabs, SELL-32-sigma inside
  std::vector<long long> cnz(n + 1, 0);
  for (int c : ci) cnz[c + 1]++;
  for (int c = 0; c < n; ++c) cnz[c + 1] += cnz[c];
  std::vector<int> cb(P + 1);
  for (int s = 0; s <= P; ++s)
    cb[s] = (int)(std::lower_bound(cnz.begin(), cnz.end(), nnz * s / P) - cnz.begin());
  cb[0] = 0;
  cb[P] = n;
  int maxw = 0;
  for (int s = 0; s < P; ++s) maxw = std::max(maxw, cb[s + 1] - cb[s]);
  const int nsl = (m + 31) / 32;
  std::vector<int> sp((size_t)P * nsl + 1), perm((size_t)P * nsl * 32, -1), wr((size_t)P * 33);
  std::vector<int> cur(rp.begin(), rp.end() - 1);  // per-row cursor into its CSR run
  std::vector<int> len(m), ord(m), start(m);
  long long slots = 0;
  std::vector<std::vector<int>> sub_begin(P);
  std::vector<unsigned short> scol;
  std::vector<double> sval;
  scol.reserve(nnz * 105 / 100);
  sval.reserve(nnz * 105 / 100);
  for (int s = 0; s < P; ++s) {
    for (int r = 0; r < m; ++r) {
      start[r] = cur[r];
      int e = cur[r];
      while (e < rp[r + 1] && ci[e] < cb[s + 1]) ++e;
      len[r] = e - cur[r];
      cur[r] = e;
    }
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return len[a] > len[b]; });
    std::vector<long long> wsl(nsl);
    for (int q = 0; q < nsl; ++q) {
      sp[(size_t)s * nsl + q] = (int)slots;
      int wd = 0;
      for (int l = 0; l < 32 && q * 32 + l < m; ++l) wd = std::max(wd, len[ord[q * 32 + l]]);
      for (int k = 0; k < wd; ++k)
        for (int l = 0; l < 32; ++l) {
          const int qi = q * 32 + l;
          if (qi < m && k < len[ord[qi]]) {
            const int e = start[ord[qi]] + k;
            scol.push_back((unsigned short)(ci[e] - cb[s]));
            sval.push_back(v[e]);
          } else {
            scol.push_back(0xFFFF);
            sval.push_back(0.0);
          }
        }
      for (int l = 0; l < 32; ++l)
        perm[((size_t)s * nsl + q) * 32 + l] = (q * 32 + l < m) ? ord[q * 32 + l] : -1;
      wsl[q] = 32LL * wd;
      slots += 32LL * wd;
    }
    // warp runs: contiguous slices, equal slots
    long long tot = 0;
    for (long long x_ : wsl) tot += x_;
    long long acc = 0;
    int q = 0;
    for (int w = 0; w <= 32; ++w) {
      const long long target = tot * w / 32;
      while (q < nsl && acc + wsl[q] / 2 < target) acc += wsl[q++];
      wr[(size_t)s * 33 + w] = (w == 32) ? nsl : q;
    }
    for (int w = 1; w <= 32; ++w) wr[(size_t)s * 33 + w] = std::max(wr[(size_t)s * 33 + w], wr[(size_t)s * 33 + w - 1]);
  }
  sp[(size_t)P * nsl] = (int)slots;
  printf("C5 A v: %d slabs, widest %d columns (%.0f KB of x), %lld slots for %lld entries (%.2f %% padding)\n",
         P, maxw, maxw * 8.0 / 1024, slots, nnz, 100.0 * (slots - nnz) / nnz);
  std::vector<int> hinv((size_t)P * m);
  for (int s_ = 0; s_ < P; ++s_)
    for (int i = 0; i < nsl * 32; ++i) {
      const int r = perm[(size_t)s_ * nsl * 32 + i];
      if (r >= 0) hinv[(size_t)s_ * m + r] = i;
    }
  int* dinv = up(hinv);
  unsigned long long* dts;
  CK(cudaMalloc(&dts, P * 4 * 8));
  SlabStream S{m, n, P, nsl, up(cb), up(sp), up(wr), up(perm), up(scol), up(sval)};
  double* x = up(hx);
  double *y, *part;
  CK(cudaMalloc(&y, m * sizeof(double)));
  CK(cudaMalloc(&part, (size_t)P * m * sizeof(double)));
  std::vector<double> hy(m);
  auto report = [&](const char* k, float ms) {
    CK(cudaMemcpy(hy.data(), y, m * sizeof(double), cudaMemcpyDeviceToHost));
    double err = 0;
    for (int r = 0; r < m; ++r) err = std::max(err, (double)(fabsl(hy[r] - yr[r]) / fabsl(yr[r])));
    printf("%-34s %8.2f us %7.1f GB/s (%.2f of 6457)  max rel err %.1e\n", k, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / 6457.4, err);
    CK(cudaMemset(y, 0, m * sizeof(double)));
  };
  int* drp = up(rp);
  int* dci = up(ci);
  double* dv = up(v);
  for (int fl = 1; fl >= 0; --fl) {
    printf("--- %s\n", fl ? "cold (L2 flushed before every launch)" : "warm (back to back, as inside a solve)");
    report("k_rows_wrow (library)", timeit([&] { k_wrow<<<P * 3, 256>>>(drp, dci, dv, m, x, y); }, 20, fl));
    const int smem = maxw * 8;
#define SLAB(U)                                                                                \
    {                                                                                          \
      CK(cudaFuncSetAttribute(k_slab<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));  \
      float t = timeit([&] {                                                                   \
        k_slab<U><<<P, kT, smem>>>(S, x, part);                                                \
        k_sum<<<(m + 31) / 32, 256>>>(part, m, P, y);                                          \
      }, 20, fl);                                                                              \
      report("slab stream U" #U " + sum", t);                                                  \
      float t1 = timeit([&] { k_slab<U><<<P, kT, smem>>>(S, x, part); }, 20, fl);              \
      float t2 = timeit([&] { k_sum<<<(m + 31) / 32, 256>>>(part, m, P, y); }, 20, fl);        \
      printf("      slab kernel %.2f us, sum kernel %.2f us\n", t1 * 1e3, t2 * 1e3);           \
    }
    SLAB(8)
    {
      const int smem = maxw * 8;
      CK(cudaFuncSetAttribute(k_slab<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      float t = timeit([&] {
        k_slab<8><<<P, kT, smem>>>(S, x, part);
        k_sum32<32><<<(m + 31) / 32, 1024>>>(part, m, P, y);
      }, 20, fl);
      report("slab stream U8 + sum32x32", t);
      float t2 = timeit([&] { k_sum32<32><<<(m + 31) / 32, 1024>>>(part, m, P, y); }, 20, fl);
      float t3 = timeit([&] { k_sum32<16><<<(m + 31) / 32, 512>>>(part, m, P, y); }, 20, fl);
      printf("      sum32x32 %.2f us, sum32x16 %.2f us\n", t2 * 1e3, t3 * 1e3);
    }

#define SLABT(NW, ST, CH, MODE)                                                                          \
    {                                                                                                    \
      const int xcap = (maxw + 15) & ~15;                                                                \
      const int sm_ = xcap * 8 + NW * ST * CH * 10;                                                      \
      if (sm_ <= 232448 - 1024) {                                                                        \
      CK(cudaFuncSetAttribute(k_slab_tma<NW, ST, CH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_)); \
      float t = timeit([&] {                                                                             \
        k_slab_tma<NW, ST, CH, MODE><<<P, NW * 32, sm_>>>(S, x, part, xcap);                             \
        k_sum32<32><<<(m + 31) / 32, 1024>>>(part, m, P, y);                                             \
      }, 20, fl);                                                                                        \
      report("slab TMA NW" #NW " ST" #ST " CH" #CH " mode" #MODE " + sum32", t);                        \
      float t1 = timeit([&] { k_slab_tma<NW, ST, CH, MODE><<<P, NW * 32, sm_>>>(S, x, part, xcap); }, 20, fl); \
      printf("      slab kernel %.2f us (smem %d)\n", t1 * 1e3, sm_);                                    \
      } else printf("slab TMA NW" #NW " ST" #ST " CH" #CH ": smem %d too large\n", sm_);                 \
    }

#define SLAB2(NW, U, PIPE)                                                                               \
    {                                                                                                    \
      const int xcap = (maxw + 15) & ~15;                                                                \
      const int sm_ = xcap * 8 + nsl * 32 * 8 + (nsl + 1) * 4 + 16;                                      \
      CK(cudaFuncSetAttribute(k_slab2<NW, U, PIPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_));   \
      float t = timeit([&] {                                                                             \
        k_slab2<NW, U, PIPE><<<P, NW * 32, sm_>>>(S, dinv, x, part, xcap, nullptr);                       \
        k_sum32<32><<<(m + 31) / 32, 1024>>>(part, m, P, y);                                             \
      }, 20, fl);                                                                                        \
      report("slab2 NW" #NW " U" #U " PIPE" #PIPE " + sum32", t);                                        \
      float t1 = timeit([&] { k_slab2<NW, U, PIPE><<<P, NW * 32, sm_>>>(S, dinv, x, part, xcap, nullptr); }, 20, fl); \
      if (fl) flush_l2();                                                                                \
      k_slab2<NW, U, PIPE><<<P, NW * 32, sm_>>>(S, dinv, x, part, xcap, dts);                            \
      CK(cudaDeviceSynchronize());                                                                       \
      std::vector<unsigned long long> hts(P * 4);                                                        \
      CK(cudaMemcpy(hts.data(), dts, P * 32, cudaMemcpyDeviceToHost));                                   \
      unsigned long long T0 = ~0ull; double a0 = 0, a1 = 0, a2 = 0, a3 = 0, mx = 0;                       \
      for (int b = 0; b < P; ++b) T0 = std::min(T0, hts[b * 4]);                                         \
      for (int b = 0; b < P; ++b) { a0 += hts[b*4]-T0; a1 += hts[b*4+1]-T0; a2 += hts[b*4+2]-T0; a3 += hts[b*4+3]-T0; mx = std::max(mx, (double)(hts[b*4+3]-T0)); } \
      printf("      slab kernel %.2f us; phases (mean over blocks, us from first start): start %.2f staged %.2f streamed %.2f flushed %.2f (max %.2f)\n", \
             t1 * 1e3, a0 / P * 1e-3, a1 / P * 1e-3, a2 / P * 1e-3, a3 / P * 1e-3, mx * 1e-3);           \
    }
    SLAB2(32, 8, 0)
    SLAB2(32, 4, 1)

#define SLAB2C(NW, U, PIPE, SNW, SL)                                                                     \
    {                                                                                                    \
      const int xcap = (maxw + 15) & ~15;                                                                \
      const int sm_ = xcap * 8 + nsl * 32 * 8 + (nsl + 1) * 4 + 16;                                      \
      CK(cudaFuncSetAttribute(k_slab2<NW, U, PIPE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_)); \
      cudaLaunchConfig_t cfg = {};                                                                       \
      cfg.gridDim = dim3(P); cfg.blockDim = dim3(NW * 32); cfg.dynamicSmemBytes = sm_;                   \
      cudaLaunchAttribute at[1];                                                                         \
      at[0].id = cudaLaunchAttributeClusterDimension;                                                    \
      at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;                \
      cfg.attrs = at; cfg.numAttrs = 1;                                                                  \
      unsigned long long* nots = nullptr;                                                                \
      float t = timeit([&] {                                                                             \
        CK(cudaLaunchKernelEx(&cfg, k_slab2<NW, U, PIPE, 2>, S, (const int*)dinv, (const double*)x, part, xcap, nots)); \
        k_sumA<SNW, SL><<<(m + 31) / 32, SNW * 32>>>(part, m, P / 2, y);                                 \
      }, 20, fl);                                                                                        \
      report("slab2 pair NW" #NW " U" #U " PIPE" #PIPE " + sumA" #SNW "x" #SL, t);                       \
      float t1 = timeit([&] { CK(cudaLaunchKernelEx(&cfg, k_slab2<NW, U, PIPE, 2>, S, (const int*)dinv, (const double*)x, part, xcap, nots)); }, 20, fl); \
      float t2 = timeit([&] { k_sumA<SNW, SL><<<(m + 31) / 32, SNW * 32>>>(part, m, P / 2, y); }, 20, fl); \
      if (fl) flush_l2();                                                                                \
      CK(cudaLaunchKernelEx(&cfg, k_slab2<NW, U, PIPE, 2>, S, (const int*)dinv, (const double*)x, part, xcap, dts)); \
      CK(cudaDeviceSynchronize());                                                                       \
      std::vector<unsigned long long> hts(P * 4);                                                        \
      CK(cudaMemcpy(hts.data(), dts, P * 32, cudaMemcpyDeviceToHost));                                   \
      unsigned long long T0 = ~0ull; double a0 = 0, a1 = 0, a2 = 0, a3 = 0, mx = 0;                       \
      for (int b = 0; b < P; ++b) T0 = std::min(T0, hts[b * 4]);                                         \
      for (int b = 0; b < P; ++b) { a0 += hts[b*4]-T0; a1 += hts[b*4+1]-T0; a2 += hts[b*4+2]-T0; a3 += hts[b*4+3]-T0; mx = std::max(mx, (double)(hts[b*4+3]-T0)); } \
      printf("      slab kernel %.2f us, sum %.2f us; phases: start %.2f staged %.2f streamed %.2f flushed %.2f (max %.2f)\n", \
             t1 * 1e3, t2 * 1e3, a0 / P * 1e-3, a1 / P * 1e-3, a2 / P * 1e-3, a3 / P * 1e-3, mx * 1e-3); \
    }

#define SLAB2H(NW, U, PIPE, HINT)                                                                        \
    {                                                                                                    \
      const int xcap = (maxw + 15) & ~15;                                                                \
      const int sm_ = xcap * 8 + nsl * 32 * 8 + (nsl + 1) * 4 + 16;                                      \
      CK(cudaFuncSetAttribute(k_slab2<NW, U, PIPE, 1, HINT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_)); \
      float t = timeit([&] {                                                                             \
        k_slab2<NW, U, PIPE, 1, HINT><<<P, NW * 32, sm_>>>(S, dinv, x, part, xcap, nullptr);              \
        k_sumA<8, 10><<<(m + 31) / 32, 256>>>(part, m, P, y);                                            \
      }, 40, fl);                                                                                        \
      report("slab2 NW" #NW " U" #U " PIPE" #PIPE " HINT" #HINT " + sumA8x10", t);                       \
      if (fl) flush_l2();                                                                                \
      k_slab2<NW, U, PIPE, 1, HINT><<<P, NW * 32, sm_>>>(S, dinv, x, part, xcap, nullptr);                \
      k_slab2<NW, U, PIPE, 1, HINT><<<P, NW * 32, sm_>>>(S, dinv, x, part, xcap, dts);                    \
      CK(cudaDeviceSynchronize());                                                                       \
      std::vector<unsigned long long> hts(P * 4);                                                        \
      CK(cudaMemcpy(hts.data(), dts, P * 32, cudaMemcpyDeviceToHost));                                   \
      unsigned long long T0 = ~0ull; double a1 = 0, a2 = 0, a3 = 0, mx = 0;                               \
      for (int b = 0; b < P; ++b) T0 = std::min(T0, hts[b * 4]);                                         \
      for (int b = 0; b < P; ++b) { a1 += hts[b*4+1]-T0; a2 += hts[b*4+2]-T0; a3 += hts[b*4+3]-T0; mx = std::max(mx, (double)(hts[b*4+3]-T0)); } \
      printf("      phases: staged %.2f streamed %.2f flushed %.2f (max %.2f)\n", a1 / P * 1e-3, a2 / P * 1e-3, a3 / P * 1e-3, mx * 1e-3); \
    }
    SLAB2H(32, 4, 1, 0)
    SLAB2H(32, 4, 1, 1)
    SLAB2H(32, 4, 1, 0)
    SLAB2H(32, 4, 1, 1)
    {
      float a = timeit([&] { k_sumA<8, 10><<<(m + 31) / 32, 256>>>(part, m, P, y); }, 20, fl);
      float b = timeit([&] { k_sumA<16, 10><<<(m + 31) / 32, 512>>>(part, m, P, y); }, 20, fl);
      float c = timeit([&] { k_sumA<32, 5><<<(m + 31) / 32, 1024>>>(part, m, P, y); }, 20, fl);
      float d = timeit([&] { k_sumA<8, 19><<<(m + 31) / 32, 256>>>(part, m, P, y); }, 20, fl);
      float e = timeit([&] { k_sum32<32><<<1, 32>>>(part, 1, 1, y); }, 20, fl);
      printf("      full-P sums: sumA8x10 %.2f sumA16x10 %.2f sumA32x5 %.2f sumA8x19 %.2f; empty kernel %.2f us\n", a * 1e3, b * 1e3, c * 1e3, d * 1e3, e * 1e3);
    }
  }
  return 0;
}
