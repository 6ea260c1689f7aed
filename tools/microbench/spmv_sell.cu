// Round-2 sparse pass study (not part of the library):
//
//  * short rows (C4: 5-point stencil, n = 1e6; C5^T: 1e6 rows of 10 random
//    columns of 1e4): the library's warp-cooperative k_rows_warp against a
//    sliced-ELL (SELL-32) layout with one thread per row — slice s keeps its
//    32 rows interleaved (entry k of lane l at base_s + 32 k + l), so every
//    load of a warp is one coalesced 256 / 128 B request and no row pointers
//    are chased; padding slots carry column -1 and are skipped, so each row is
//    still summed left to right without FMA (scipy's order, bitwise).  Variants:
//    int32 vs uint16 column indices, x gathered through L1 vs staged in smem.
//  * long rows (C5's A v: 1e4 rows of ~1000 entries over 1e6 columns): the
//    library's warp-per-row k_rows_wrow (random 8 B gathers from the 8 MB x,
//    one L2 sector each) against a slab-major layout: the columns are cut into
//    slabs of kSlab columns; an item is (row range of G rows, slab); a block
//    walks a contiguous run of items (row range major, slab minor), each
//    thread keeps its rows' accumulators in registers across the slabs, and
//    the run's x gathers stay inside one slab (L1-resident).  Partials per
//    (row range, contributing block) are summed in block order by a combine
//    kernel.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/microbench/spmv_sell tools/microbench/spmv_sell.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstring>
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
__device__ __forceinline__ int ld_stream_i(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned short ld_stream_u16(const unsigned short* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

// stand-in epilogue: y = v and a per-block sum of y^2
__device__ __forceinline__ void block_out(double acc, double* part) {
  __shared__ double sm[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sm[i];
    part[blockIdx.x] = s;
  }
}

struct Csr {
  int m, n;
  long long nnz;
  int *rp, *ci;
  double* val;
};

// ------------------------------------------------- library short rows ----
constexpr int kWCh = 256;
__global__ void __launch_bounds__(256, 4) k_warp(Csr A, const double* __restrict__ x, double* y, double* part) {
  __shared__ double buf[8][kWCh];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long m = A.m, ngroups = (m + 31) / 32;
  const long long W = (long long)gridDim.x * 8, w = (long long)blockIdx.x * 8 + wid;
  const long long g0 = ngroups * w / W, g1 = ngroups * (w + 1) / W;
  double acc = 0.0;
  double* sb = buf[wid];
  for (long long g = g0; g < g1; ++g) {
    const long long r = g * 32 + lane;
    const bool live = r < m;
    const long long rlast = (g * 32 + 32 < m) ? g * 32 + 32 : m;
    const int kb = live ? __ldg(A.rp + r) : 0, ke = live ? __ldg(A.rp + r + 1) : 0;
    const int gb = __shfl_sync(0xffffffffu, kb, 0), ge = __ldg(A.rp + rlast);
    double sum = 0.0;
    for (int cs = gb; cs < ge; cs += kWCh) {
      constexpr int J = kWCh / 32;
      double vv[J], xv[J];
      int cc[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = cs + j * 32 + lane;
        const bool ok = k < ge;
        vv[j] = ok ? ld_stream(A.val + k) : 0.0;
        cc[j] = ok ? ld_stream_i(A.ci + k) : 0;
      }
#pragma unroll
      for (int j = 0; j < J; ++j) xv[j] = __ldg(x + cc[j]);
#pragma unroll
      for (int j = 0; j < J; ++j) sb[j * 32 + lane] = __dmul_rn(vv[j], xv[j]);
      __syncwarp();
      const int lo = kb > cs ? kb : cs, hi = ke < cs + kWCh ? ke : cs + kWCh;
      for (int k = lo; k < hi; ++k) sum = __dadd_rn(sum, sb[k - cs]);
      __syncwarp();
    }
    if (live) {
      y[r] = sum;
      acc = fma(sum, sum, acc);
    }
  }
  block_out(acc, part);
}

// ------------------------------------------------------------- SELL-32 ----
// slice s: rows [32 s, 32 s + 32), width w_s = max row length, entries at
// sp[s] + 32 k + lane (k < w_s); padding: column = -1 (int) / 0xFFFF (u16)
template <class IT>
struct Sell {
  int m;
  const int* sp;  // [nslices + 1] (entries, padded)
  const IT* ci;
  const double* val;
};

template <class IT>
__device__ __forceinline__ int ld_col(const IT* p);
template <>
__device__ __forceinline__ int ld_col<int>(const int* p) { return ld_stream_i(p); }
template <>
__device__ __forceinline__ int ld_col<unsigned short>(const unsigned short* p) {
  const unsigned short v = ld_stream_u16(p);
  return v == 0xFFFFu ? -1 : (int)v;
}

// thread per row; U entries of the row in flight per step
template <class IT, int U, int NB, bool kSmemX, int NT = 256>
__global__ void __launch_bounds__(NT, NB) k_sell(Sell<IT> A, const double* __restrict__ x, int nx,
                                                 double* y, double* part) {
  extern __shared__ double xsm[];
  if constexpr (kSmemX) {
    for (int i = threadIdx.x; i < nx; i += blockDim.x) xsm[i] = __ldg(x + i);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const long long nsl = (A.m + 31) / 32;
  const long long W = (long long)gridDim.x * (NT / 32);
  const long long w = (long long)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  double acc = 0.0;
  for (long long s = w; s < nsl; s += W) {
    const int b0 = __ldg(A.sp + s), b1 = __ldg(A.sp + s + 1);
    const int wd = (b1 - b0) >> 5;
    const long long r = s * 32 + lane;
    double sum = 0.0;
    for (int k0 = 0; k0 < wd; k0 += U) {
      double v[U], xv[U];
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u;
        const int e = b0 + 32 * k + lane;
        c[u] = k < wd ? ld_col<IT>(A.ci + e) : -1;
        v[u] = k < wd ? ld_stream(A.val + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (kSmemX) xv[u] = c[u] >= 0 ? xsm[c[u]] : 0.0;
        else xv[u] = c[u] >= 0 ? __ldg(x + c[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
    }
    if (r < A.m) {
      y[r] = sum;
      acc = fma(sum, sum, acc);
    }
  }
  block_out(acc, part);
}

// --------------------------------------------------- library long rows ----
constexpr int kWrowU = 6;
__global__ void __launch_bounds__(256, 3) k_wrow(Csr A, const double* __restrict__ x, double* y, double* part) {
  constexpr int U = kWrowU;
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * 256) >> 5;
  double acc = 0.0;
  for (long long r = w; r < A.m; r += W) {
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
      for (int u = 0; u < U; ++u) { v[u] = pv[u]; j[u] = pj[u]; }
      const int kn = k + 32 * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kn + 32 * u;
        pv[u] = kk < k1 ? ld_stream(A.val + kk) : 0.0;
        pj[u] = kk < k1 ? ld_stream_i(A.ci + kk) : 0;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + j[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], xv[u], a[u & 3]);
    }
    const double sum = ((a[0] + a[1]) + (a[2] + a[3]));
    double t = sum;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) {
      y[r] = t;
      acc = fma(t, t, acc);
    }
  }
  block_out(acc, part);
}

// ---------------------------------------------------------- slab-major ----
// entries sorted (slab, row, col); srp[s * (m + 1) + r] = first entry of
// (slab s, row r) (srp[s * (m + 1) + m] = end of slab s).  Items q = (row
// range i, slab s) with q = i * nslab + s; block b owns items [Q b / P, Q (b+1) / P).
// Each thread owns RPT rows of the range (G = RPT * blockDim rows).
struct Slab {
  int m, n, nslab, slab;
  const int* srp;
  const unsigned short* sc;  // in-slab column
  const double* sv;
};

__host__ __device__ inline long long blk_of(long long q, long long Q, long long P) {
  return ((q + 1) * P + Q - 1) / Q - 1;
}

template <int RPT, int NT, int NB, bool kL1>
__global__ void __launch_bounds__(NT, NB) k_slab(Slab A, const double* __restrict__ x, double* part,
                                               int maxc) {
  constexpr int G = RPT * NT;
  const long long nr = (A.m + G - 1) / G;
  const long long Q = nr * A.nslab, P = gridDim.x, b = blockIdx.x;
  const long long q0 = Q * b / P, q1 = Q * (b + 1) / P;
  long long q = q0;
  while (q < q1) {
    const long long i = q / A.nslab;
    const long long qe = ((i + 1) * A.nslab < q1) ? (i + 1) * A.nslab : q1;
    double acc[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) acc[j] = 0.0;
    for (; q < qe; ++q) {
      const int s = (int)(q - i * A.nslab);
      const int* rp = A.srp + (long long)s * (A.m + 1);
      const double* xs = x + (long long)s * A.slab;
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const long long r = i * G + j * NT + threadIdx.x;
        if (r < A.m) {
          const int e0 = __ldg(rp + r), e1 = __ldg(rp + r + 1);
          double a0 = 0.0, a1 = 0.0;
          int e = e0;
          for (; e + 4 <= e1; e += 4) {
            double v[4];
            int c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if constexpr (kL1) { v[u] = __ldg(A.sv + e + u); c[u] = __ldg(A.sc + e + u); }
              else { v[u] = ld_stream(A.sv + e + u); c[u] = ld_stream_u16(A.sc + e + u); }
            }
            a0 = fma(v[0], __ldg(xs + c[0]), a0);
            a1 = fma(v[1], __ldg(xs + c[1]), a1);
            a0 = fma(v[2], __ldg(xs + c[2]), a0);
            a1 = fma(v[3], __ldg(xs + c[3]), a1);
          }
          for (; e < e1; ++e) a0 = fma(__ldg(A.sv + e), __ldg(xs + __ldg(A.sc + e)), a0);
          acc[j] += a0 + a1;
        }
      }
    }
    // this block's partial for row range i, slot = b - first block of range i
    const long long slot = b - blk_of(i * A.nslab, Q, P);
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const long long r = i * G + j * NT + threadIdx.x;
      if (r < A.m) part[(slot * A.m) + r] = acc[j];
    }
  }
}

template <int RPT, int NT>
__global__ void k_slab_combine(Slab A, long long P, const double* __restrict__ part, double* y, double* bp) {
  constexpr int G = RPT * NT;
  const long long nr = (A.m + G - 1) / G, Q = nr * A.nslab;
  double acc = 0.0;
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < A.m; r += (long long)gridDim.x * blockDim.x) {
    const long long i = r / G;
    const long long ba = blk_of(i * A.nslab, Q, P), bb = blk_of((i + 1) * A.nslab - 1, Q, P);
    double s = part[r];
    for (long long k = 1; k <= bb - ba; ++k) s += part[k * A.m + r];
    y[r] = s;
    acc = fma(s, s, acc);
  }
  block_out(acc, bp);
}

// ----------------------------------------------------- slab SELL-32-sigma ----
// Per slab (kW columns), the slab's rows are sorted by their in-slab length
// (descending, stable) and cut into slices of 32; slice q of slab s keeps its
// rows interleaved (entry k of lane l at sp[item] + 32 k + l, in-slab column
// as u16, padding 0xFFFF).  item = s * nsl + q (nsl = ceil(m / 32)); the x slab
// is staged in shared memory once per (block, slab); row sums go to
// part[s * m + perm].
struct SlabSell {
  int m, n, nslab, nsl, slab;
  const int* sp;               // [nslab * nsl + 1]
  const unsigned short* sc;
  const double* sv;
  const int* perm;             // [nslab * nsl * 32] row of each (item, lane), -1 past m
};
template <int U, int NT, int NB>
__global__ void __launch_bounds__(NT, NB) k_slab_sell(SlabSell A, const double* __restrict__ x, double* part) {
  extern __shared__ double xsm[];
  const long long Q = (long long)A.nslab * A.nsl, P = gridDim.x, b = blockIdx.x;
  const long long q0 = Q * b / P, q1 = Q * (b + 1) / P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  long long q = q0;
  while (q < q1) {
    const int s = (int)(q / A.nsl);
    const long long qe = ((long long)(s + 1) * A.nsl < q1) ? (long long)(s + 1) * A.nsl : q1;
    const int c0 = s * A.slab, cw = (A.n - c0 < A.slab) ? A.n - c0 : A.slab;
    __syncthreads();
    for (int i = threadIdx.x; i < cw; i += NT) xsm[i] = __ldg(x + c0 + i);
    __syncthreads();
    for (long long it = q + wid; it < qe; it += NW) {
      const int b0 = __ldg(A.sp + it), b1 = __ldg(A.sp + it + 1);
      const int wd = (b1 - b0) >> 5;
      double a0 = 0.0, a1 = 0.0;
      for (int k0 = 0; k0 < wd; k0 += U) {
        double v[U];
        unsigned c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u;
          const int e = b0 + 32 * k + lane;
          c[u] = k < wd ? (unsigned)ld_stream_u16(A.sc + e) : 0xFFFFu;
          v[u] = k < wd ? ld_stream(A.sv + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c[u] != 0xFFFFu) {
            if (u & 1) a1 = fma(v[u], xsm[c[u]], a1);
            else a0 = fma(v[u], xsm[c[u]], a0);
          }
      }
      const int r = __ldg(A.perm + it * 32 + lane);
      if (r >= 0) part[(long long)s * A.m + r] = a0 + a1;
    }
    q = qe;
  }
}
__global__ void k_slab_sum(const double* __restrict__ part, int m, int nslab, double* y, double* bp) {
  double acc = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    int q = 0;
    for (; q + 16 <= nslab; q += 16) {
      double t[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) t[u] = __ldcg(part + (long long)(q + u) * m + r);
#pragma unroll
      for (int u = 0; u < 16; ++u) s += t[u];
    }
    for (; q < nslab; ++q) s += part[(long long)q * m + r];
    y[r] = s;
    acc = fma(s, s, acc);
  }
  block_out(acc, bp);
}

// 32 rows per block; warp g sums slabs g, g + 8, ... (4 loads in flight), the
// 8 warp partials are added in warp order
__global__ void __launch_bounds__(256) k_slab_sum2(const double* __restrict__ part, int m, int nslab, double* y,
                                                   double* bp) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + lane;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (r < m) {
    int q = g;
    for (; q + 24 < nslab; q += 32) {
      s0 += __ldcg(part + (long long)q * m + r);
      s1 += __ldcg(part + (long long)(q + 8) * m + r);
      s2 += __ldcg(part + (long long)(q + 16) * m + r);
      s3 += __ldcg(part + (long long)(q + 24) * m + r);
    }
    for (; q < nslab; q += 8) s0 += __ldcg(part + (long long)q * m + r);
  }
  red[g][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  double acc = 0.0;
  if (g == 0 && r < m) {
    double t = red[0][lane];
    for (int j = 1; j < 8; ++j) t += red[j][lane];
    y[r] = t;
    acc = t * t;
  }
  block_out(acc, bp);
}

// ------------------------------------------------------------------ host ----
static double* g_flush = nullptr;
static void flush_l2() {
  if (!g_flush) CK(cudaMalloc(&g_flush, 256 << 20));
  CK(cudaMemset(g_flush, 1, 256 << 20));
}
template <class F>
static float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  std::vector<float> t;
  for (int i = 0; i < reps; ++i) {
    flush_l2();
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

static int g_sms = 148;

static void run_short(const char* name, const std::vector<int>& rp, const std::vector<int>& ci,
                      const std::vector<double>& v, int m, int n) {
  const long long nnz = (long long)ci.size();
  const double bytes = 12.0 * nnz + 4.0 * (m + 1) + 8.0 * (m + n);
  std::vector<double> hx(n);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> ur(-1, 1);
  for (auto& e : hx) e = ur(g);
  // reference y (host, scipy order)
  std::vector<double> yr(m);
  for (int r = 0; r < m; ++r) {
    double s = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) s = s + v[k] * hx[ci[k]];
    yr[r] = s;
  }
  Csr A{m, n, nnz, up(rp), up(ci), up(v)};
  double* x = up(hx);
  double *y, *part;
  CK(cudaMalloc(&y, m * sizeof(double)));
  CK(cudaMalloc(&part, 4096 * sizeof(double)));
  std::vector<double> hy(m);
  auto report = [&](const char* k, float ms) {
    CK(cudaMemcpy(hy.data(), y, m * sizeof(double), cudaMemcpyDeviceToHost));
    long long bad = 0;
    for (int r = 0; r < m; ++r) bad += memcmp(&hy[r], &yr[r], 8) != 0;
    printf("%-5s %-28s %8.2f us %7.1f GB/s (%.2f of 6457)  bitwise-mismatch %lld\n", name, k, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / 6457.4, bad);
    CK(cudaMemset(y, 0, m * sizeof(double)));
  };
  {
    float ms = timeit([&] { k_warp<<<g_sms * 4, 256>>>(A, x, y, part); });
    report("k_rows_warp (library)", ms);
  }
  // SELL-32 layouts
  const int nsl = (m + 31) / 32;
  std::vector<int> sp(nsl + 1);
  long long tot = 0;
  for (int s = 0; s < nsl; ++s) {
    sp[s] = (int)tot;
    int wd = 0;
    for (int r = 32 * s; r < std::min(m, 32 * s + 32); ++r) wd = std::max(wd, rp[r + 1] - rp[r]);
    tot += 32LL * wd;
  }
  sp[nsl] = (int)tot;
  std::vector<int> sci(tot, -1);
  std::vector<unsigned short> sci16(tot, 0xFFFF);
  std::vector<double> sv(tot, 0.0);
  for (int s = 0; s < nsl; ++s)
    for (int r = 32 * s; r < std::min(m, 32 * s + 32); ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) {
        const long long e = sp[s] + 32LL * (k - rp[r]) + (r - 32 * s);
        sci[e] = ci[k];
        sci16[e] = (unsigned short)ci[k];
        sv[e] = v[k];
      }
  printf("%-5s SELL-32 padding: %lld slots for %lld entries (%.2f %%)\n", name, tot, nnz, 100.0 * (tot - nnz) / nnz);
  Sell<int> S32{m, up(sp), up(sci), up(sv)};
  Sell<unsigned short> S16{m, S32.sp, up(sci16), S32.val};
  const bool u16ok = n < 0xFFFF;
  const int smx = n * 8;
#define SELL(IT, SS, U, NB, SM, GR)                                                                      \
  {                                                                                                      \
    const int sm = SM ? smx : 0;                                                                         \
    if (SM) CK(cudaFuncSetAttribute(k_sell<IT, U, NB, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    float ms = timeit([&] { k_sell<IT, U, NB, SM><<<g_sms * GR, 256, sm>>>(SS, x, n, y, part); });      \
    report("sell " #IT " U" #U " nb" #NB " smx" #SM " g" #GR, ms);                                      \
  }
  SELL(int, S32, 4, 4, false, 4)
  SELL(int, S32, 8, 4, false, 4)
  SELL(int, S32, 8, 3, false, 3)
  SELL(int, S32, 5, 6, false, 6)
  SELL(int, S32, 8, 6, false, 6)
  SELL(int, S32, 8, 8, false, 8)
  SELL(int, S32, 10, 4, false, 4)
  SELL(int, S32, 10, 6, false, 6)
  SELL(int, S32, 10, 8, false, 8)
  if (u16ok) {
    SELL(unsigned short, S16, 8, 4, false, 4)
    SELL(unsigned short, S16, 10, 6, false, 6)
    SELL(unsigned short, S16, 10, 8, false, 8)
  }
  if (smx <= 100 * 1024) {
    SELL(int, S32, 10, 2, true, 2)
    if (u16ok) SELL(unsigned short, S16, 10, 2, true, 2)
#define SELLT(IT, SS, U, NB, NT, GR)                                                                     \
  {                                                                                                      \
    CK(cudaFuncSetAttribute(k_sell<IT, U, NB, true, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smx)); \
    float ms = timeit([&] { k_sell<IT, U, NB, true, NT><<<g_sms * GR, NT, smx>>>(SS, x, n, y, part); }); \
    report("sell " #IT " U" #U " nb" #NB " smx t" #NT " g" #GR, ms);                                    \
  }
    SELLT(int, S32, 10, 2, 512, 2)
    SELLT(int, S32, 10, 1, 1024, 1)
    SELLT(int, S32, 5, 2, 512, 2)
    if (u16ok) SELLT(unsigned short, S16, 10, 2, 512, 2)
  }
  cudaFree(A.rp); cudaFree(A.ci); cudaFree(A.val); cudaFree(x); cudaFree(y); cudaFree(part);
  cudaFree((void*)S32.sp); cudaFree((void*)S32.ci); cudaFree((void*)S32.val); cudaFree((void*)S16.ci);
}

static void run_long(const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<double>& v, int m,
                     int n) {
  const long long nnz = (long long)ci.size();
  const double bytes = 12.0 * nnz + 4.0 * (m + 1) + 8.0 * (m + n);
  std::vector<double> hx(n);
  std::mt19937_64 g(2);
  std::uniform_real_distribution<double> ur(-1, 1);
  for (auto& e : hx) e = ur(g);
  std::vector<long double> yr(m);
  for (int r = 0; r < m; ++r) {
    long double s = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) s += (long double)v[k] * hx[ci[k]];
    yr[r] = s;
  }
  Csr A{m, n, nnz, up(rp), up(ci), up(v)};
  double* x = up(hx);
  double *y, *part;
  CK(cudaMalloc(&y, m * sizeof(double)));
  CK(cudaMalloc(&part, 4096 * sizeof(double)));
  std::vector<double> hy(m);
  auto report = [&](const char* k, float ms) {
    CK(cudaMemcpy(hy.data(), y, m * sizeof(double), cudaMemcpyDeviceToHost));
    double err = 0;
    for (int r = 0; r < m; ++r) err = std::max(err, (double)(fabsl(hy[r] - yr[r]) / fabsl(yr[r])));
    printf("C5Av  %-28s %8.2f us %7.1f GB/s (%.2f of 6457)  max rel err %.1e\n", k, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / 6457.4, err);
    CK(cudaMemset(y, 0, m * sizeof(double)));
  };
  {
    float ms = timeit([&] { k_wrow<<<g_sms * 3, 256>>>(A, x, y, part); });
    report("k_rows_wrow (library)", ms);
  }
  for (int slab : {8192, (n + g_sms - 1) / g_sms, (n + 2 * g_sms - 1) / (2 * g_sms)}) {
    const int nslab = (n + slab - 1) / slab;
    // (slab, row, col) order: stable partition of the CSR by slab
    std::vector<int> srp((size_t)nslab * (m + 1));
    std::vector<long long> cnt((size_t)nslab * m, 0);
    for (int r = 0; r < m; ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) cnt[(size_t)(ci[k] / slab) * m + r]++;
    long long run = 0;
    for (int s = 0; s < nslab; ++s) {
      for (int r = 0; r < m; ++r) {
        srp[(size_t)s * (m + 1) + r] = (int)run;
        run += cnt[(size_t)s * m + r];
      }
      srp[(size_t)s * (m + 1) + m] = (int)run;
    }
    std::vector<unsigned short> sc(nnz);
    std::vector<double> sv(nnz);
    std::vector<int> pos(srp);
    for (int r = 0; r < m; ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) {
        const int s = ci[k] / slab;
        const long long e = pos[(size_t)s * (m + 1) + r]++;
        sc[e] = (unsigned short)(ci[k] - s * slab);
        sv[e] = v[k];
      }
    Slab S{m, n, nslab, slab, up(srp), up(sc), up(sv)};
    double* dpart;
    CK(cudaMalloc(&dpart, (size_t)64 * m * sizeof(double)));
    char nm[96];
#define SLAB(RPT, NT, NB, L1, PF)                                                                       \
  {                                                                                                     \
    const int P = g_sms * PF;                                                                           \
    float ms = timeit([&] {                                                                             \
      k_slab<RPT, NT, NB, L1><<<P, NT>>>(S, x, dpart, 0);                                               \
      k_slab_combine<RPT, NT><<<(m + 63) / 64, 64>>>(S, P, dpart, y, part);                             \
    });                                                                                                 \
    snprintf(nm, sizeof nm, "slab%d r%d t%d nb%d L1%d p%d", slab, RPT, NT, NB, (int)L1, PF);            \
    report(nm, ms);                                                                                     \
    float m1 = timeit([&] { k_slab<RPT, NT, NB, L1><<<P, NT>>>(S, x, dpart, 0); });                     \
    printf("      main %.2f us\n", m1 * 1e3);                                                          \
  }

    // slab SELL-32-sigma
    if (slab <= 16384) {
      const int nsl = (m + 31) / 32;
      std::vector<int> ssp((size_t)nslab * nsl + 1), perm((size_t)nslab * nsl * 32, -1);
      long long tot2 = 0;
      std::vector<int> ord(m);
      for (int s2 = 0; s2 < nslab; ++s2) {
        const int* rps = srp.data() + (size_t)s2 * (m + 1);
        for (int r = 0; r < m; ++r) ord[r] = r;
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return rps[a + 1] - rps[a] > rps[b + 1] - rps[b]; });
        for (int q2 = 0; q2 < nsl; ++q2) {
          ssp[(size_t)s2 * nsl + q2] = (int)tot2;
          int wd = 0;
          for (int l = 0; l < 32 && q2 * 32 + l < m; ++l) {
            const int r = ord[q2 * 32 + l];
            wd = std::max(wd, rps[r + 1] - rps[r]);
            perm[((size_t)s2 * nsl + q2) * 32 + l] = r;
          }
          tot2 += 32LL * wd;
        }
      }
      ssp[(size_t)nslab * nsl] = (int)tot2;
      std::vector<unsigned short> ssc(tot2, 0xFFFF);
      std::vector<double> ssv(tot2, 0.0);
      for (int s2 = 0; s2 < nslab; ++s2) {
        const int* rps = srp.data() + (size_t)s2 * (m + 1);
        for (int q2 = 0; q2 < nsl; ++q2)
          for (int l = 0; l < 32; ++l) {
            const int r = perm[((size_t)s2 * nsl + q2) * 32 + l];
            if (r < 0) continue;
            for (int k = rps[r]; k < rps[r + 1]; ++k) {
              const long long e = ssp[(size_t)s2 * nsl + q2] + 32LL * (k - rps[r]) + l;
              ssc[e] = sc[k];
              ssv[e] = sv[k];
            }
          }
      }
      printf("C5Av  slab-sell %d: padding %.2f %%\n", slab, 100.0 * (tot2 - nnz) / nnz);
      SlabSell SS{m, n, nslab, nsl, slab, up(ssp), up(ssc), up(ssv), up(perm)};
      double* sp2;
      CK(cudaMalloc(&sp2, (size_t)nslab * m * sizeof(double)));
      const int smb = slab * 8;
#define SSELL(U, NT, NB)                                                                                   \
  {                                                                                                        \
    CK(cudaFuncSetAttribute(k_slab_sell<U, NT, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));   \
    const int P = g_sms * NB;                                                                              \
    float ms = timeit([&] {                                                                                \
      k_slab_sell<U, NT, NB><<<P, NT, smb>>>(SS, x, sp2);                                                  \
      k_slab_sum<<<(m + 63) / 64, 64>>>(sp2, m, nslab, y, part);                                           \
    });                                                                                                    \
    snprintf(nm, sizeof nm, "slab-sell%d U%d t%d nb%d", slab, U, NT, NB);                                 \
    report(nm, ms);                                                                                        \
    float m1 = timeit([&] { k_slab_sell<U, NT, NB><<<P, NT, smb>>>(SS, x, sp2); });                      \
    float m2 = timeit([&] { k_slab_sum<<<(m + 63) / 64, 64>>>(sp2, m, nslab, y, part); });                \
    printf("      main %.2f us, combine %.2f us\n", m1 * 1e3, m2 * 1e3);                                  \
  }
#define SSELLP(U, NT, NB, PB)                                                                             \
  {                                                                                                        \
    CK(cudaFuncSetAttribute(k_slab_sell<U, NT, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));   \
    const int P = PB;                                                                                      \
    const int gc = (m + 31) / 32;                                                                          \
    float ms = timeit([&] {                                                                                \
      k_slab_sell<U, NT, NB><<<P, NT, smb>>>(SS, x, sp2);                                                  \
      k_slab_sum2<<<gc, 256>>>(sp2, m, nslab, y, part);                                                    \
    });                                                                                                    \
    snprintf(nm, sizeof nm, "slab-sell%d U%d t%d nb%d P%d", slab, U, NT, NB, P);                           \
    report(nm, ms);                                                                                        \
    float m1 = timeit([&] { k_slab_sell<U, NT, NB><<<P, NT, smb>>>(SS, x, sp2); });                      \
    float m2 = timeit([&] { k_slab_sum2<<<gc, 256>>>(sp2, m, nslab, y, part); });                          \
    printf("      main %.2f us, combine %.2f us\n", m1 * 1e3, m2 * 1e3);                                  \
  }
      if (slab == 8192) { SSELL(12, 512, 2) SSELL(8, 1024, 1) SSELLP(8, 1024, 1, g_sms) SSELLP(8, 512, 2, 2 * g_sms) }
      else if (nslab == g_sms) { SSELLP(8, 1024, 1, nslab) SSELLP(4, 1024, 1, nslab) SSELLP(8, 768, 1, nslab) }
      else { SSELLP(8, 512, 2, nslab) SSELLP(4, 512, 2, nslab) SSELLP(8, 1024, 2, nslab) }
      cudaFree((void*)SS.sp); cudaFree((void*)SS.sc); cudaFree((void*)SS.sv); cudaFree((void*)SS.perm); cudaFree(sp2);
    }
    cudaFree((void*)S.srp); cudaFree((void*)S.sc); cudaFree((void*)S.sv); cudaFree(dpart);
  }
}

int main() {
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, 0));
  g_sms = pr.multiProcessorCount;
  printf("device %s, %d SMs\n", pr.name, g_sms);
  {  // C4: 5-point stencil on a 1000 x 1000 grid
    const int G = 1000, m = G * G;
    std::vector<int> rp(m + 1), ci;
    std::vector<double> v;
    ci.reserve(5 * m); v.reserve(5 * m);
    for (int iy = 0; iy < G; ++iy)
      for (int ix = 0; ix < G; ++ix) {
        const int k = ix + G * iy;
        rp[k] = (int)ci.size();
        if (iy > 0) { ci.push_back(k - G); v.push_back(-1.025); }
        if (ix > 0) { ci.push_back(k - 1); v.push_back(-1.05); }
        ci.push_back(k); v.push_back(4.075);
        if (ix < G - 1) { ci.push_back(k + 1); v.push_back(-1.0); }
        if (iy < G - 1) { ci.push_back(k + G); v.push_back(-1.0); }
      }
    rp[m] = (int)ci.size();
    run_short("c4", rp, ci, v, m, m);
  }
  {  // C5: 1e4 x 1e6, 10 distinct random rows per column
    const int m = 10000, n = 1000000;
    std::mt19937_64 g(5);
    std::uniform_int_distribution<int> ui(0, m - 1);
    std::uniform_real_distribution<double> ur(0.1, 1.0);
    std::vector<int> trp(n + 1), tci;  // A^T as CSR (columns of A)
    std::vector<double> tv;
    tci.reserve(10LL * n); tv.reserve(10LL * n);
    for (int j = 0; j < n; ++j) {
      trp[j] = (int)tci.size();
      int c[10];
      for (int i = 0; i < 10; ++i) {
        bool dup;
        do { c[i] = ui(g); dup = false; for (int q = 0; q < i; ++q) dup |= c[q] == c[i]; } while (dup);
      }
      std::sort(c, c + 10);
      for (int i = 0; i < 10; ++i) { tci.push_back(c[i]); tv.push_back(ur(g)); }
    }
    trp[n] = (int)tci.size();
    run_short("c5T", trp, tci, tv, n, m);
    // A as CSR (rows of A, columns ascending)
    std::vector<int> rp(m + 1, 0), ci(tci.size());
    std::vector<double> v(tv.size());
    for (int c : tci) rp[c + 1]++;
    for (int r = 0; r < m; ++r) rp[r + 1] += rp[r];
    std::vector<int> pos(rp.begin(), rp.end() - 1);
    for (int j = 0; j < n; ++j)
      for (int k = trp[j]; k < trp[j + 1]; ++k) {
        const int e = pos[tci[k]]++;
        ci[e] = j;
        v[e] = tv[k];
      }
    run_long(rp, ci, v, m, n);
  }
  return 0;
}
