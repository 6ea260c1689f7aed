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
  }
  return 0;
}
