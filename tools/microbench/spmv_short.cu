// Short-row CSR SpMV variants on C4-like (5-point stencil, n = 1e6) and
// C5^T-like (1e6 rows x 10 random columns of 1e4) matrices: the kernel
// design study behind k_rows_warp / k_rows_stream (not part of the library).
// Every variant adds a row's products left to right without FMA (scipy's
// order), so all outputs must agree bitwise.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/microbench/spmv_short tools/microbench/spmv_short.cu
#include <algorithm>
#include <cstdio>
#include <cstring>
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

struct Csr {
  int m, n;
  long long nnz;
  int *rp, *ci;
  double* val;
};

// epilogue stand-in: store y, reduce sum y^2 per block
__device__ __forceinline__ void epi(double* y, int r, double v, double& acc) {
  y[r] = v;
  acc = fma(v, v, acc);
}
__device__ __forceinline__ void block_out(double acc, double* part) {
  __shared__ double sm[8];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sm[i];
    part[blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------- V1 warp ---
constexpr int kWCh = 256;
__global__ void __launch_bounds__(256, 4) k_warp(Csr A, const double* __restrict__ x, double* y, double* part) {
  __shared__ double buf[8][kWCh];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long m = A.m, ngroups = (m + 31) / 32;
  const long long W = (long long)gridDim.x * 8, w = (long long)blockIdx.x * 8 + wid;
  const long long g0 = ngroups * w / W, g1 = ngroups * (w + 1) / W;
  double acc = 0;
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
    if (live) epi(y, (int)r, sum, acc);
  }
  block_out(acc, part);
}

// ------------------------------------------------ V2 warp + prefetch (R rows/lane)
// A warp owns G = 32*R consecutive rows per step; their entries are staged in
// CH-entry chunks.  The first chunk of the NEXT step is loaded into registers
// before the current step's gathers/sums, so a load is always in flight.
template <int R, int J>
__global__ void __launch_bounds__(256, 4) k_warp_pf(Csr A, const double* __restrict__ x, double* y, double* part) {
  constexpr int CH = 32 * J;
  constexpr int G = 32 * R;
  __shared__ double buf[8][CH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long m = A.m, ngroups = (m + G - 1) / G;
  const long long W = (long long)gridDim.x * 8, w = (long long)blockIdx.x * 8 + wid;
  const long long g0 = ngroups * w / W, g1 = ngroups * (w + 1) / W;
  double acc = 0;
  double* sb = buf[wid];
  double pv[J];
  int pc[J];
  auto load = [&](int cs, int ge) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = cs + j * 32 + lane;
      const bool ok = k < ge;
      pv[j] = ok ? ld_stream(A.val + k) : 0.0;
      pc[j] = ok ? ld_stream_i(A.ci + k) : 0;
    }
  };
  auto gbounds = [&](long long g, int* gb, int* ge) {
    const long long rf = g * G, rl = (rf + G < m) ? rf + G : m;
    *gb = __ldg(A.rp + rf);
    *ge = __ldg(A.rp + rl);
  };
  int gb = 0, ge = 0;
  if (g0 < g1) {
    gbounds(g0, &gb, &ge);
    load(gb, ge);
  }
  for (long long g = g0; g < g1; ++g) {
    int kb[R], ke[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const long long r = g * G + i * 32 + lane;
      kb[i] = r < m ? __ldg(A.rp + r) : 0;
      ke[i] = r < m ? __ldg(A.rp + r + 1) : 0;
    }
    double sum[R];
#pragma unroll
    for (int i = 0; i < R; ++i) sum[i] = 0.0;
    int ngb = 0, nge = 0;
    const bool more = g + 1 < g1;
    if (more) gbounds(g + 1, &ngb, &nge);
    for (int cs = gb; cs < ge; cs += CH) {
      double vv[J];
      int cc[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        vv[j] = pv[j];
        cc[j] = pc[j];
      }
      // prefetch: next chunk of this group, else the first chunk of the next group
      if (cs + CH < ge) load(cs + CH, ge);
      else if (more) load(ngb, nge);
      double xv[J];
#pragma unroll
      for (int j = 0; j < J; ++j) xv[j] = __ldg(x + cc[j]);
#pragma unroll
      for (int j = 0; j < J; ++j) sb[j * 32 + lane] = __dmul_rn(vv[j], xv[j]);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int lo = kb[i] > cs ? kb[i] : cs, hi = ke[i] < cs + CH ? ke[i] : cs + CH;
        for (int k = lo; k < hi; ++k) sum[i] = __dadd_rn(sum[i], sb[k - cs]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const long long r = g * G + i * 32 + lane;
      if (r < m) epi(y, (int)r, sum[i], acc);
    }
    gb = ngb;
    ge = nge;
  }
  block_out(acc, part);
}

// ------------------------------------------------------ V3 block TMA stream --
template <int CAP, int ROWS>
struct __align__(16) Stage {
  double val[CAP + 2];
  int idx[CAP + 4];
  int rp[ROWS + 8];
};

template <int CAP, int ROWS, int S, int NB>
__global__ void __launch_bounds__(256, NB) k_stream(Csr A, const int2* __restrict__ chunks, const int* __restrict__ blk,
                                                   const double* __restrict__ x, double* y, double* part) {
  using St = Stage<CAP, ROWS>;
  extern __shared__ __align__(128) unsigned char raw[];
  St* stg = reinterpret_cast<St*>(raw);
  __shared__ __align__(8) unsigned long long full[S];
  const int tid = threadIdx.x;
  const int c0 = blk[blockIdx.x], c1 = blk[blockIdx.x + 1];
  auto issue = [&](int c, int s) {
    const int2 a = __ldg(chunks + c), z = __ldg(chunks + c + 1);
    const int e0v = a.y & ~1, e0i = a.y & ~3, r0 = a.x & ~3;
    const unsigned bv = (unsigned)(((z.y - e0v) * 8 + 15) & ~15);
    const unsigned bi = (unsigned)(((z.y - e0i) * 4 + 15) & ~15);
    const unsigned br = (unsigned)(((z.x + 1 - r0) * 4 + 15) & ~15);
    mbar_expect_tx(&full[s], bv + bi + br);
    bulk_g2s(stg[s].val, A.val + e0v, bv, &full[s]);
    bulk_g2s(stg[s].idx, A.ci + e0i, bi, &full[s]);
    bulk_g2s(stg[s].rp, A.rp + r0, br, &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    for (int s = 0; s < S && c0 + s < c1; ++s) issue(c0 + s, s);
  }
  __syncthreads();
  double acc = 0;
  int2 a = c0 < c1 ? __ldg(chunks + c0) : make_int2(0, 0);
  for (int c = c0, g = 0; c < c1; ++c, ++g) {
    const int s = g % S;
    const int2 z = __ldg(chunks + c + 1);
    const int ne = z.y - a.y, nr = z.x - a.x;
    mbar_wait(&full[s], (unsigned)((g / S) & 1));
    double* sv = stg[s].val + (a.y & 1);
    const int* si = stg[s].idx + (a.y & 3);
    const int* sr = stg[s].rp + (a.x & 3);
    for (int k0 = tid; k0 < ne; k0 += 4 * 256) {
      double xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u * 256;
        xv[u] = k < ne ? __ldg(x + si[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u * 256;
        if (k < ne) sv[k] = __dmul_rn(sv[k], xv[u]);
      }
    }
    __syncthreads();
    for (int r = tid; r < nr; r += 256) {
      const int kb = sr[r] - a.y, ke = sr[r + 1] - a.y;
      double sum = 0.0;
      for (int k = kb; k < ke; ++k) sum = __dadd_rn(sum, sv[k]);
      epi(y, a.x + r, sum, acc);
    }
    __syncthreads();
    if (tid == 0 && c + S < c1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + S, s);
    }
    a = z;
  }
  block_out(acc, part);
}

// ---------------------------------------------------- V4 per-warp TMA ring --
// Each warp owns a contiguous run of chunks (<= WROWS rows, <= WCAP entries)
// and its own S-stage ring; lane 0 issues the bulk copies.  No block barriers:
// warps overlap each other's gather / sum phases.
template <int WCAP, int WROWS, int S, int NB>
__global__ void __launch_bounds__(256, NB) k_wstream(Csr A, const int2* __restrict__ chunks, const int* __restrict__ wrun,
                                                    const double* __restrict__ x, double* y, double* part) {
  using St = Stage<WCAP, WROWS>;
  extern __shared__ __align__(128) unsigned char raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  St* stg = reinterpret_cast<St*>(raw) + wid * S;
  __shared__ __align__(8) unsigned long long full[8][S];
  const int w = blockIdx.x * 8 + wid;
  const int c0 = wrun[w], c1 = wrun[w + 1];
  auto issue = [&](int c, int s) {
    const int2 a = __ldg(chunks + c), z = __ldg(chunks + c + 1);
    const int e0v = a.y & ~1, e0i = a.y & ~3, r0 = a.x & ~3;
    const unsigned bv = (unsigned)(((z.y - e0v) * 8 + 15) & ~15);
    const unsigned bi = (unsigned)(((z.y - e0i) * 4 + 15) & ~15);
    const unsigned br = (unsigned)(((z.x + 1 - r0) * 4 + 15) & ~15);
    mbar_expect_tx(&full[wid][s], bv + bi + br);
    bulk_g2s(stg[s].val, A.val + e0v, bv, &full[wid][s]);
    bulk_g2s(stg[s].idx, A.ci + e0i, bi, &full[wid][s]);
    bulk_g2s(stg[s].rp, A.rp + r0, br, &full[wid][s]);
  };
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[wid][s], 1);
    fence_mbar_init();
    for (int s = 0; s < S && c0 + s < c1; ++s) issue(c0 + s, s);
  }
  __syncwarp();
  double acc = 0;
  int2 a = c0 < c1 ? __ldg(chunks + c0) : make_int2(0, 0);
  for (int c = c0, g = 0; c < c1; ++c, ++g) {
    const int s = g % S;
    const int2 z = __ldg(chunks + c + 1);
    const int ne = z.y - a.y, nr = z.x - a.x;
    mbar_wait(&full[wid][s], (unsigned)((g / S) & 1));
    double* sv = stg[s].val + (a.y & 1);
    const int* si = stg[s].idx + (a.y & 3);
    const int* sr = stg[s].rp + (a.x & 3);
    for (int k0 = lane; k0 < ne; k0 += 8 * 32) {
      double xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u * 32;
        xv[u] = k < ne ? __ldg(x + si[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u * 32;
        if (k < ne) sv[k] = __dmul_rn(sv[k], xv[u]);
      }
    }
    __syncwarp();
    for (int r = lane; r < nr; r += 32) {
      const int kb = sr[r] - a.y, ke = sr[r + 1] - a.y;
      double sum = 0.0;
      for (int k = kb; k < ke; ++k) sum = __dadd_rn(sum, sv[k]);
      epi(y, a.x + r, sum, acc);
    }
    __syncwarp();
    if (lane == 0 && c + S < c1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + S, s);
    }
    a = z;
  }
  block_out(acc, part);
}

// ------------------------------------------------------------------ host ---
static void chunk_plan(const std::vector<int>& rp, int m, int cap, int rows, int P, std::vector<int2>& ch,
                       std::vector<int>& run) {
  ch.clear();
  int r = 0;
  while (r < m) {
    ch.push_back(make_int2(r, rp[r]));
    int e = r + 1;
    while (e < m && e - r < rows && rp[e + 1] - rp[r] <= cap) ++e;
    r = e;
  }
  const long long nnz = rp[m];
  ch.push_back(make_int2(m, (int)nnz));
  const int nc = (int)ch.size() - 1;
  run.assign(P + 1, 0);
  for (int b = 0; b <= P; ++b) {
    if (b == P) { run[b] = nc; continue; }
    const long long t = nnz * b / P;
    int lo = 0, hi = nc;
    while (lo < hi) { int mid = (lo + hi) / 2; if (ch[mid].y < t) lo = mid + 1; else hi = mid; }
    run[b] = lo;
  }
  for (int b = 1; b <= P; ++b) run[b] = std::max(run[b], run[b - 1]);
}

static Csr upload(const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<double>& v, int m, int n) {
  Csr A;
  A.m = m; A.n = n; A.nnz = (long long)ci.size();
  CK(cudaMalloc(&A.rp, (m + 1 + 4) * sizeof(int)));
  CK(cudaMalloc(&A.ci, (A.nnz + 4) * sizeof(int)));
  CK(cudaMalloc(&A.val, (A.nnz + 2) * sizeof(double)));
  CK(cudaMemcpy(A.rp, rp.data(), (m + 1) * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(A.ci, ci.data(), A.nnz * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(A.val, v.data(), A.nnz * sizeof(double), cudaMemcpyHostToDevice));
  return A;
}

template <class F>
static float timeit(F f, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

static void run(const char* name, const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<double>& v,
                int m, int n) {
  Csr A = upload(rp, ci, v, m, n);
  std::vector<double> xh(n);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& t : xh) t = nd(g);
  double *x, *y, *part, *yref;
  CK(cudaMalloc(&x, n * sizeof(double)));
  CK(cudaMalloc(&y, m * sizeof(double)));
  CK(cudaMalloc(&yref, m * sizeof(double)));
  CK(cudaMalloc(&part, 1 << 20));
  CK(cudaMemcpy(x, xh.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  const double bytes = 12.0 * A.nnz + 4.0 * (m + 1) + 8.0 * (m + n);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto report = [&](const char* v, float ms) {
    std::vector<double> a(m), b(m);
    CK(cudaMemcpy(a.data(), y, m * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), yref, m * 8, cudaMemcpyDeviceToHost));
    const bool same = !memcmp(a.data(), b.data(), m * 8);
    printf("%-6s %-28s %8.2f us %7.1f GB/s %s\n", name, v, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
           same ? "bitwise=ref" : "MISMATCH");
    CK(cudaMemset(y, 0, m * 8));
  };
  // V1 (reference output)
  {
    const int P = sms * 4;
    float ms = timeit([&] { k_warp<<<P, 256>>>(A, x, yref, part); }, 50);
    CK(cudaMemcpy(y, yref, m * 8, cudaMemcpyDeviceToDevice));
    report("warp", ms);
  }
#define PF(R, J)                                                                                   \
  {                                                                                                \
    const int P = sms * 4;                                                                         \
    float ms = timeit([&] { k_warp_pf<R, J><<<P, 256>>>(A, x, y, part); }, 50);                    \
    report("warp_pf<" #R "," #J ">", ms);                                                          \
  }
  PF(1, 8) PF(1, 6) PF(2, 8) PF(2, 12) PF(1, 12)
#define ST(CAP, ROWS, S, NB)                                                                                \
  {                                                                                                         \
    std::vector<int2> ch; std::vector<int> run;                                                             \
    const int P = sms * NB;                                                                                 \
    chunk_plan(rp, m, CAP, ROWS, P, ch, run);                                                               \
    int2* dch; int* drun;                                                                                   \
    CK(cudaMalloc(&dch, ch.size() * sizeof(int2))); CK(cudaMalloc(&drun, run.size() * sizeof(int)));       \
    CK(cudaMemcpy(dch, ch.data(), ch.size() * sizeof(int2), cudaMemcpyHostToDevice));                      \
    CK(cudaMemcpy(drun, run.data(), run.size() * sizeof(int), cudaMemcpyHostToDevice));                    \
    const int smem = S * (int)sizeof(Stage<CAP, ROWS>);                                                     \
    CK(cudaFuncSetAttribute(k_stream<CAP, ROWS, S, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    float ms = timeit([&] { k_stream<CAP, ROWS, S, NB><<<P, 256, smem>>>(A, dch, drun, x, y, part); }, 50); \
    report("stream<" #CAP "," #ROWS "," #S "," #NB ">", ms);                                               \
    cudaFree(dch); cudaFree(drun);                                                                          \
  }
  ST(1024, 256, 4, 4) ST(512, 256, 4, 4) ST(512, 128, 3, 4) ST(256, 128, 4, 4) ST(2048, 256, 3, 2)
#define WS(CAP, ROWS, S, NB)                                                                                 \
  {                                                                                                          \
    std::vector<int2> ch; std::vector<int> run;                                                              \
    const int P = sms * NB;                                                                                  \
    chunk_plan(rp, m, CAP, ROWS, P * 8, ch, run);                                                            \
    int2* dch; int* drun;                                                                                    \
    CK(cudaMalloc(&dch, ch.size() * sizeof(int2))); CK(cudaMalloc(&drun, run.size() * sizeof(int)));        \
    CK(cudaMemcpy(dch, ch.data(), ch.size() * sizeof(int2), cudaMemcpyHostToDevice));                       \
    CK(cudaMemcpy(drun, run.data(), run.size() * sizeof(int), cudaMemcpyHostToDevice));                     \
    const int smem = 8 * S * (int)sizeof(Stage<CAP, ROWS>);                                                  \
    CK(cudaFuncSetAttribute(k_wstream<CAP, ROWS, S, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    float ms = timeit([&] { k_wstream<CAP, ROWS, S, NB><<<P, 256, smem>>>(A, dch, drun, x, y, part); }, 50); \
    report("wstream<" #CAP "," #ROWS "," #S "," #NB ">", ms);                                               \
    cudaFree(dch); cudaFree(drun);                                                                           \
  }
  WS(256, 64, 3, 2) WS(256, 64, 2, 3) WS(128, 32, 4, 3) WS(384, 96, 2, 2)
  cudaFree(A.rp); cudaFree(A.ci); cudaFree(A.val); cudaFree(x); cudaFree(y); cudaFree(yref); cudaFree(part);
}

int main() {
  {  // C4-like: 5-point stencil on a 1000 x 1000 grid
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
    run("c4", rp, ci, v, m, m);
  }
  {  // C5^T-like: 1e6 rows of 10 distinct random columns in [0, 1e4)
    const int m = 1000000, n = 10000;
    std::mt19937_64 g(5);
    std::vector<int> rp(m + 1), ci;
    std::vector<double> v;
    ci.reserve(10LL * m); v.reserve(10LL * m);
    std::uniform_int_distribution<int> ui(0, n - 1);
    std::uniform_real_distribution<double> ur(0.1, 1.0);
    for (int r = 0; r < m; ++r) {
      rp[r] = (int)ci.size();
      int c[10];
      for (int i = 0; i < 10; ++i) {
        bool dup;
        do { c[i] = ui(g); dup = false; for (int j = 0; j < i; ++j) dup |= c[j] == c[i]; } while (dup);
      }
      std::sort(c, c + 10);
      for (int i = 0; i < 10; ++i) { ci.push_back(c[i]); v.push_back(ur(g)); }
    }
    rp[m] = (int)ci.size();
    run("c5T", rp, ci, v, m, n);
  }
  return 0;
}
