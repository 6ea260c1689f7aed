// Wide long-row CSR A v (C5: 1e4 x 1e6, 1000 nnz per row, x = 8 MB gathered
// at random): variants of the flat-split kernel's per-warp loop (loads in
// flight, occupancy) and a column-tiled variant whose x gathers hit shared
// memory.  Design study behind k_rows_flat<CsrRows> / k_csr_ctile; not part
// of the library.  Row sums are compared against the flat kernel to 1e-13.
// k_wrow_pfn / k_wrow_ix: block-size and index-only-prefetch sweeps of the
// library loop (profiles/round1/spmv_long_variants.txt: all within 4 %).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/microbench/spmv_long tools/microbench/spmv_long.cu
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2304_12168_b200/csrc/ts_common.cuh"

namespace ts {
void set_error(const char*, ...) {}
const char* last_error() { return ""; }
}  // namespace ts
using namespace ts;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

// warp per row (rows are long and uniform here): U loads of 32 entries in flight
template <int U, int NB>
__global__ void __launch_bounds__(256, NB) k_wrow(const int* __restrict__ rp, const int* __restrict__ ci,
                                                 const double* __restrict__ val, int m,
                                                 const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * 256 + threadIdx.x) >> 5, W = (gridDim.x * 256) >> 5;
  for (int r = w; r < m; r += W) {
    const int k0 = __ldg(rp + r), k1 = __ldg(rp + r + 1);
    double a[4] = {0, 0, 0, 0};
    int k = k0 + lane;
    for (; k + 32 * (U - 1) < k1; k += 32 * U) {
      double v[U], xv[U];
      int j[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = ld_stream(val + k + 32 * u);
        j[u] = ld_stream_i(ci + k + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + j[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], xv[u], a[u & 3]);
    }
    for (; k < k1; k += 32) a[0] = fma(ld_stream(val + k), __ldg(x + ld_stream_i(ci + k)), a[0]);
    const double s = warp_reduce((a[0] + a[1]) + (a[2] + a[3]), RED_SUM);
    if (lane == 0) y[r] = s;
  }
}

// warp per row with software prefetch: the next U-chunk's values and indices
// are loaded before the current chunk's gathers
template <int U, int NB>
__global__ void __launch_bounds__(256, NB) k_wrow_pf(const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const double* __restrict__ val, int m,
                                                    const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * 256 + threadIdx.x) >> 5, W = (gridDim.x * 256) >> 5;
  for (int r = w; r < m; r += W) {
    const int k0 = __ldg(rp + r), k1 = __ldg(rp + r + 1);
    double a[4] = {0, 0, 0, 0};
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
      for (int u = 0; u < U; ++u) {
        v[u] = pv[u];
        j[u] = pj[u];
      }
      const int kn = k + 32 * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kn + 32 * u;
        pv[u] = kk < k1 ? ld_stream(val + kk) : 0.0;
        pj[u] = kk < k1 ? ld_stream_i(ci + kk) : 0;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + j[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], xv[u], a[u & 3]);
    }
    const double s = warp_reduce((a[0] + a[1]) + (a[2] + a[3]), RED_SUM);
    if (lane == 0) y[r] = s;
  }
}

// k_wrow_pf with the block size as a parameter (occupancy at fixed registers)
template <int U, int NT, int NB>
__global__ void __launch_bounds__(NT, NB) k_wrow_pfn(const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const double* __restrict__ val, int m,
                                                    const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * NT + threadIdx.x) >> 5, W = (gridDim.x * NT) >> 5;
  for (int r = w; r < m; r += W) {
    const int k0 = __ldg(rp + r), k1 = __ldg(rp + r + 1);
    double a[4] = {0, 0, 0, 0};
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
      for (int u = 0; u < U; ++u) {
        v[u] = pv[u];
        j[u] = pj[u];
      }
      const int kn = k + 32 * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kn + 32 * u;
        pv[u] = kk < k1 ? ld_stream(val + kk) : 0.0;
        pj[u] = kk < k1 ? ld_stream_i(ci + kk) : 0;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + j[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], xv[u], a[u & 3]);
    }
    const double s = warp_reduce((a[0] + a[1]) + (a[2] + a[3]), RED_SUM);
    if (lane == 0) y[r] = s;
  }
}

// index-only prefetch: the next chunk's column indices are loaded ahead, the
// current chunk's values are loaded together with its x gathers (both ~L2 /
// DRAM latency), so fewer registers per entry in flight -> more warps
template <int U, int NT, int NB>
__global__ void __launch_bounds__(NT, NB) k_wrow_ix(const int* __restrict__ rp, const int* __restrict__ ci,
                                                   const double* __restrict__ val, int m,
                                                   const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * NT + threadIdx.x) >> 5, W = (gridDim.x * NT) >> 5;
  for (int r = w; r < m; r += W) {
    const int k0 = __ldg(rp + r), k1 = __ldg(rp + r + 1);
    double a[4] = {0, 0, 0, 0};
    int pj[U];
    int k = k0 + lane;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = k + 32 * u;
      pj[u] = kk < k1 ? ld_stream_i(ci + kk) : -1;
    }
    for (; k < k1; k += 32 * U) {
      int j[U];
#pragma unroll
      for (int u = 0; u < U; ++u) j[u] = pj[u];
      const int kn = k + 32 * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kn + 32 * u;
        pj[u] = kk < k1 ? ld_stream_i(ci + kk) : -1;
      }
      double v[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = j[u] >= 0;
        v[u] = ok ? ld_stream(val + k + 32 * u) : 0.0;
        xv[u] = ok ? __ldg(x + j[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], xv[u], a[u & 3]);
    }
    const double s = warp_reduce((a[0] + a[1]) + (a[2] + a[3]), RED_SUM);
    if (lane == 0) y[r] = s;
  }
}

// the library's k_rows_wrow structure, built up step by step (XS functor,
// epilogue + block reduction, last-block finisher) to find what costs time
struct XSm {
  const double* sp = nullptr;
  int relu = 0;
  double s = 1.0;
  __device__ __forceinline__ double operator()(double v) const {
    if (!sp) return v;
    if (relu) v = (v >= 0.0 || v != v) ? v : 0.0;
    return __dmul_rn(s, v);
  }
};
// branch-free form: identity is scale 1.0 (exact), relu a select
struct XSb {
  int relu = 0;
  double s = 1.0;
  __device__ __forceinline__ double operator()(double v) const {
    const double r = (v >= 0.0 || v != v) ? v : 0.0;
    return __dmul_rn(s, relu ? r : v);
  }
};
template <int STAGE, class XT, int U = 8, int NB = 4>
__global__ void __launch_bounds__(256, NB) k_lib(const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double* __restrict__ val, int64_t m,
                                               const double* __restrict__ x, XT xs, double* __restrict__ y,
                                               double* bacc, unsigned* done, double* out) {
  __shared__ double sm[8];
  __shared__ int sflag;
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * 256) >> 5;
  double acc = 0.0;
  for (int64_t r = w; r < m; r += W) {
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
      for (int u = 0; u < U; ++u) {
        v[u] = pv[u];
        j[u] = pj[u];
      }
      const int kn = k + 32 * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kn + 32 * u;
        pv[u] = kk < k1 ? ld_stream(val + kk) : 0.0;
        pj[u] = kk < k1 ? ld_stream_i(ci + kk) : 0;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = STAGE >= 1 ? xs(__ldg(x + j[u])) : __ldg(x + j[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u & 3] = fma(v[u], xv[u], a[u & 3]);
    }
    const double sum = warp_reduce((a[0] + a[1]) + (a[2] + a[3]), RED_SUM);
    if (lane == 0) {
      y[r] = sum;
      if (STAGE >= 2) acc = fma(sum, sum, acc);
    }
  }
  if (STAGE >= 2) {
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sm[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int i = 0; i < 8; ++i) t += sm[i];
      bacc[blockIdx.x] = t;
    }
  }
  if (STAGE >= 3 && arrive_last(done, gridDim.x, &sflag)) {
    double t = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 256) t += __ldcg(bacc + b);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      double q = 0;
      for (int i = 0; i < 8; ++i) q += sm[i];
      *out = q;
    }
  }
}

// column tiles: block = (tile t, row range); x slice of the tile in smem; the
// tile's entries of each row are contiguous (tile-major CSR: rp_t[t*m + r]);
// warp per row inside the tile; partials part[t * m + r] (tile-major, so a
// warp's 32 rows store one coalesced line), summed over tiles afterwards
constexpr int TWC = 8192;
template <int NB>
__global__ void __launch_bounds__(256, NB) k_ctile(const int* __restrict__ trp, const unsigned short* __restrict__ tci,
                                                  const double* __restrict__ tval, int m, int n, int rows_per_blk,
                                                  const double* __restrict__ x, double* __restrict__ part) {
  extern __shared__ double xs[];
  const int nrb = (m + rows_per_blk - 1) / rows_per_blk;
  const int t = blockIdx.x / nrb, rb = blockIdx.x % nrb;
  const int cb = t * TWC;
  for (int k = threadIdx.x; k < TWC; k += 256) xs[k] = (cb + k < n) ? __ldg(x + cb + k) : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int r0 = rb * rows_per_blk, r1 = min(m, r0 + rows_per_blk);
  for (int rg = r0 + wid * 32; rg < r1; rg += 8 * 32) {  // warp: 32 rows, lane = row for the store
    double mine = 0.0;
    for (int q = 0; q < 32 && rg + q < r1; ++q) {
      const int r = rg + q;
      const int k0 = __ldg(trp + (size_t)t * m + r), k1 = __ldg(trp + (size_t)t * m + r + 1);
      double a = 0.0;
      for (int k = k0 + lane; k < k1; k += 32) a = fma(ld_stream(tval + k), xs[tci[k]], a);
      a = warp_reduce(a, RED_SUM);
      if (lane == q) mine = a;
    }
    if (rg + lane < r1) part[(size_t)t * m + rg + lane] = mine;
  }
}
__global__ void k_tsum(const double* __restrict__ part, int m, int nt, double* __restrict__ y) {
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r >= m) return;
  double s = 0.0;
  for (int t = 0; t < nt; ++t) s += __ldg(part + (size_t)t * m + r);
  y[r] = s;
}

template <class F>
static float timeit(F f, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

static std::vector<char> slurp(const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) { printf("cannot open %s\n", path); exit(1); }
  fseek(f, 0, SEEK_END);
  long sz = ftell(f);
  fseek(f, 0, SEEK_SET);
  std::vector<char> b(sz);
  if (fread(b.data(), 1, sz, f) != (size_t)sz) exit(1);
  fclose(f);
  return b;
}

int main(int argc, char** argv) {
  const int m = 10000, n = 1000000, per_col = 10;
  std::mt19937_64 g(7);
  std::uniform_int_distribution<int> ui(0, m - 1);
  std::uniform_real_distribution<double> ur(0.1, 1.0);
  // columns with 10 distinct rows -> CSR by rows
  std::vector<std::vector<std::pair<int, double>>> rows(m);
  for (int j = 0; j < n; ++j) {
    int rr[per_col];
    for (int i = 0; i < per_col; ++i) {
      bool dup;
      do {
        rr[i] = ui(g);
        dup = false;
        for (int q = 0; q < i; ++q) dup |= rr[q] == rr[i];
      } while (dup);
      rows[rr[i]].push_back({j, ur(g)});
    }
  }
  std::vector<int> rp(m + 1), ci;
  std::vector<double> val;
  for (int r = 0; r < m; ++r) {
    rp[r] = (int)ci.size();
    for (auto& e : rows[r]) {
      ci.push_back(e.first);
      val.push_back(e.second);
    }
  }
  rp[m] = (int)ci.size();
  if (argc > 1) {  // argv[1]: prefix of raw int32 indptr / int32 indices / fp64 data files
    const std::string pre = argv[1];
    auto b0 = slurp((pre + ".indptr").c_str()), b1 = slurp((pre + ".indices").c_str()),
         b2 = slurp((pre + ".data").c_str());
    memcpy(rp.data(), b0.data(), b0.size());
    ci.assign(reinterpret_cast<int*>(b1.data()), reinterpret_cast<int*>(b1.data() + b1.size()));
    val.assign(reinterpret_cast<double*>(b2.data()), reinterpret_cast<double*>(b2.data() + b2.size()));
    printf("loaded %s: nnz %zu\n", argv[1], ci.size());
  }
  const long long nnz = rp[m];
  // tile-major CSR of the column tiles
  const int nt = (n + TWC - 1) / TWC;
  std::vector<int> trp((size_t)nt * m + 1);
  std::vector<unsigned short> tci(nnz);
  std::vector<double> tval(nnz);
  {
    std::vector<long long> cnt((size_t)nt * m, 0);
    for (int r = 0; r < m; ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) cnt[(size_t)(ci[k] / TWC) * m + r]++;
    long long s = 0;
    for (size_t u = 0; u < cnt.size(); ++u) {
      trp[u] = (int)s;
      s += cnt[u];
    }
    trp[cnt.size()] = (int)s;
    std::vector<long long> pos(trp.begin(), trp.end() - 1);
    for (int r = 0; r < m; ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) {
        const size_t u = (size_t)(ci[k] / TWC) * m + r;
        tci[pos[u]] = (unsigned short)(ci[k] % TWC);
        tval[pos[u]] = val[k];
        pos[u]++;
      }
  }
  int *drp, *dci, *dtrp;
  unsigned short* dtci;
  double *dval, *dtval, *x, *y, *yref, *part;
  CK(cudaMalloc(&drp, (m + 1) * 4));
  CK(cudaMalloc(&dci, nnz * 4));
  CK(cudaMalloc(&dval, nnz * 8));
  CK(cudaMalloc(&dtrp, trp.size() * 4));
  CK(cudaMalloc(&dtci, nnz * 2));
  CK(cudaMalloc(&dtval, nnz * 8));
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&y, m * 8));
  CK(cudaMalloc(&yref, m * 8));
  CK(cudaMalloc(&part, (size_t)nt * m * 8));
  CK(cudaMemcpy(drp, rp.data(), (m + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dval, val.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtrp, trp.data(), trp.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtci, tci.data(), nnz * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtval, tval.data(), nnz * 8, cudaMemcpyHostToDevice));
  std::vector<double> xh(n);
  for (auto& v : xh) v = ur(g);
  CK(cudaMemcpy(x, xh.data(), n * 8, cudaMemcpyHostToDevice));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = 12.0 * nnz + 4.0 * (m + 1) + 8.0 * (m + n);
  std::vector<double> h0(m), h1(m);
  auto report = [&](const char* name, float ms, const double* out) {
    CK(cudaMemcpy(h1.data(), out, m * 8, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int r = 0; r < m; ++r) err = std::max(err, std::fabs(h1[r] - h0[r]) / (std::fabs(h0[r]) + 1e-300));
    printf("%-26s %8.2f us %7.1f GB/s  max rel diff %.1e\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9, err);
  };
  float ms = timeit([&] { k_wrow<8, 4><<<sms * 4, 256>>>(drp, dci, dval, m, x, yref); }, 20);
  CK(cudaMemcpy(h0.data(), yref, m * 8, cudaMemcpyDeviceToHost));
  report("wrow U8 4blk (ref)", ms, yref);
#define WR(U, NB) { float t = timeit([&] { k_wrow<U, NB><<<sms * NB, 256>>>(drp, dci, dval, m, x, y); }, 20); report("wrow U" #U " " #NB "blk", t, y); }
#define WP(U, NB) { float t = timeit([&] { k_wrow_pf<U, NB><<<sms * NB, 256>>>(drp, dci, dval, m, x, y); }, 20); report("wrow_pf U" #U " " #NB "blk", t, y); }
  WR(16, 2) WR(16, 4) WR(32, 2) WP(8, 4) WP(8, 2) WP(16, 2) WP(12, 3)
  // occupancy / register-budget variants of the library loop (k_rows_wrow = pf U6, 256 x 3)
#define WPN(U, NT, NB) { float t = timeit([&] { k_wrow_pfn<U, NT, NB><<<sms * NB, NT>>>(drp, dci, dval, m, x, y); }, 20); report("wrow_pf U" #U " " #NT "x" #NB, t, y); }
#define WIX(U, NT, NB) { float t = timeit([&] { k_wrow_ix<U, NT, NB><<<sms * NB, NT>>>(drp, dci, dval, m, x, y); }, 20); report("wrow_ix U" #U " " #NT "x" #NB, t, y); }
  WPN(6, 256, 3) WPN(6, 128, 7) WPN(6, 64, 14) WPN(4, 128, 8) WPN(8, 128, 6)
  WIX(6, 256, 3) WIX(8, 256, 3) WIX(8, 256, 4) WIX(8, 128, 8) WIX(12, 256, 3) WIX(16, 256, 2) WIX(6, 128, 8)
  {
    double *bacc, *outp;
    unsigned* done;
    CK(cudaMalloc(&bacc, 4096 * 8));
    CK(cudaMalloc(&outp, 8));
    CK(cudaMalloc(&done, 16));
    CK(cudaMemset(done, 0, 16));
    XSm xsm;
    XSb xsb;
#define LB(ST) { float t = timeit([&] { k_lib<ST, XSm><<<sms * 4, 256>>>(drp, dci, dval, (int64_t)m, x, xsm, y, bacc, done, outp); }, 20); report("lib stage " #ST, t, y); }
#define LBB(ST) { float t = timeit([&] { k_lib<ST, XSb><<<sms * 4, 256>>>(drp, dci, dval, (int64_t)m, x, xsb, y, bacc, done, outp); }, 20); report("lib branch-free xs stage " #ST, t, y); }
    LB(0) LB(1) LB(3) LBB(1)
#define LV(U, NB) { float t = timeit([&] { k_lib<3, XSm, U, NB><<<sms * NB, 256>>>(drp, dci, dval, (int64_t)m, x, xsm, y, bacc, done, outp); }, 20); report("lib stage3 U" #U " " #NB "blk", t, y); }
    LV(8, 3) LV(8, 2) LV(6, 4) LV(4, 4) LV(6, 3) LV(12, 2)
  }
#define CT(RPB, NB)                                                                              \
  {                                                                                              \
    const int nrb = (m + RPB - 1) / RPB;                                                         \
    CK(cudaFuncSetAttribute(k_ctile<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, TWC * 8));  \
    float t = timeit([&] {                                                                       \
      k_ctile<NB><<<nt * nrb, 256, TWC * 8>>>(dtrp, dtci, dtval, m, n, RPB, x, part);            \
      k_tsum<<<(m + 255) / 256, 256>>>(part, m, nt, y);                                          \
    }, 20);                                                                                      \
    report("ctile rows" #RPB " " #NB "blk", t, y);                                               \
  }
  return 0;
}
