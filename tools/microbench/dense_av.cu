// Dense A v tile-kernel variants on C2 (5000 x 20000 fp64, 800 MB): how many
// row chunks a warp keeps in flight, where the tile's slice of v lives
// (registers vs shared memory), and the occupancy / grid trade-off.  All
// variants produce the same per-(tile,row) partials bit for bit (design study
// behind k_rows_tile; not part of the library).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/microbench/dense_av tools/microbench/dense_av.cu
#include <cstdio>
#include <cstring>
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

constexpr int TW = 512;

// V0: the library's k_rows_tile (v slice in registers, one row chunk per step)
__global__ void __launch_bounds__(256, 4) k_v0(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                              const double* __restrict__ x, double* __restrict__ part) {
  const int64_t nct = (n + TW - 1) / TW, U = nct * m, P = gridDim.x, b = blockIdx.x;
  const int64_t U0 = U * b / P, U1 = U * (b + 1) / P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t u = U0; u < U1;) {
    const int64_t ct = u / m, r0 = u - ct * m, r1 = (m < r0 + (U1 - u)) ? m : r0 + (U1 - u);
    const int64_t cb = ct * TW;
    double2 xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) xv[k] = __ldg(reinterpret_cast<const double2*>(x + cb + 64 * k + 2 * lane));
    for (int64_t r = r0 + wid; r < r1; r += 8) {
      const double* row = a + r * lda + cb + 2 * lane;
      double2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = ld_stream2(row + 64 * k);
      double a0 = 0, a1 = 0;
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        a0 = fma(v[k].x, xv[k].x, a0); a0 = fma(v[k].y, xv[k].y, a0);
        a1 = fma(v[k + 1].x, xv[k + 1].x, a1); a1 = fma(v[k + 1].y, xv[k + 1].y, a1);
      }
      const double s = warp_reduce(a0 + a1, RED_SUM);
      if (lane == 0) part[r * nct + ct] = s;
    }
    u += r1 - r0;
  }
}

// V1: v slice in shared memory, R row chunks in flight per warp
template <int R, int NB>
__global__ void __launch_bounds__(256, NB) k_v1(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                               const double* __restrict__ x, double* __restrict__ part) {
  __shared__ __align__(16) double xs[TW];
  const int64_t nct = (n + TW - 1) / TW, U = nct * m, P = gridDim.x, b = blockIdx.x;
  const int64_t U0 = U * b / P, U1 = U * (b + 1) / P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t u = U0; u < U1;) {
    const int64_t ct = u / m, r0 = u - ct * m, r1 = (m < r0 + (U1 - u)) ? m : r0 + (U1 - u);
    const int64_t cb = ct * TW;
    __syncthreads();
    xs[threadIdx.x * 2] = x[cb + threadIdx.x * 2];
    xs[threadIdx.x * 2 + 1] = x[cb + threadIdx.x * 2 + 1];
    __syncthreads();
    int64_t r = r0 + wid;
    for (; r + 8 * (R - 1) < r1; r += 8 * R) {
      double2 v[R][8];
#pragma unroll
      for (int q = 0; q < R; ++q)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[q][k] = ld_stream2(a + (r + 8 * q) * lda + cb + 2 * lane + 64 * k);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        double a0 = 0, a1 = 0;
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const double2 x0 = *reinterpret_cast<const double2*>(xs + 64 * k + 2 * lane);
          const double2 x1 = *reinterpret_cast<const double2*>(xs + 64 * (k + 1) + 2 * lane);
          a0 = fma(v[q][k].x, x0.x, a0); a0 = fma(v[q][k].y, x0.y, a0);
          a1 = fma(v[q][k + 1].x, x1.x, a1); a1 = fma(v[q][k + 1].y, x1.y, a1);
        }
        const double s = warp_reduce(a0 + a1, RED_SUM);
        if (lane == 0) part[(r + 8 * q) * nct + ct] = s;
      }
    }
    for (; r < r1; r += 8) {
      double2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = ld_stream2(a + r * lda + cb + 2 * lane + 64 * k);
      double a0 = 0, a1 = 0;
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const double2 x0 = *reinterpret_cast<const double2*>(xs + 64 * k + 2 * lane);
        const double2 x1 = *reinterpret_cast<const double2*>(xs + 64 * (k + 1) + 2 * lane);
        a0 = fma(v[k].x, x0.x, a0); a0 = fma(v[k].y, x0.y, a0);
        a1 = fma(v[k + 1].x, x1.x, a1); a1 = fma(v[k + 1].y, x1.y, a1);
      }
      const double s = warp_reduce(a0 + a1, RED_SUM);
      if (lane == 0) part[r * nct + ct] = s;
    }
    u += r1 - r0;
  }
}

// A^T v core loop (k_cols_tile<Epi,2> without the merges): RU rows in flight
// per thread, NB blocks per SM; column sums of each segment to `out`
struct XSr {  // the library's runtime input transform (identity when sp == nullptr)
  const double* sp = nullptr;
  int relu = 0;
  double s = 1.0;
  __device__ __forceinline__ double operator()(double v) const {
    if (!sp) return v;
    if (relu) v = (v >= 0.0 || v != v) ? v : 0.0;
    return __dmul_rn(s, v);
  }
};
struct XSi {
  __device__ __forceinline__ double operator()(double v) const { return v; }
};
template <int RU, int NB, class XT = XSi>
__global__ void __launch_bounds__(256, NB) k_t(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                              const double* __restrict__ x, double* __restrict__ out,
                                              XT xs = XT{}) {
  const int64_t nct = (n + TW - 1) / TW, U = nct * m, P = gridDim.x, b = blockIdx.x;
  const int64_t U0 = U * b / P, U1 = U * (b + 1) / P;
  for (int64_t u = U0; u < U1;) {
    const int64_t ct = u / m, r0 = u - ct * m, r1 = (m < r0 + (U1 - u)) ? m : r0 + (U1 - u);
    const int64_t c = ct * TW + 2 * threadIdx.x;
    double ac[2][2] = {{0, 0}, {0, 0}};
    const double* base = a + c;
    int64_t r = r0;
    for (; r + RU <= r1; r += RU) {
      double2 v[RU];
      double xr[RU];
#pragma unroll
      for (int i = 0; i < RU; ++i) v[i] = ld_stream2(base + (r + i) * lda);
#pragma unroll
      for (int i = 0; i < RU; ++i) xr[i] = xs(__ldg(x + r + i));
#pragma unroll
      for (int i = 0; i < RU; ++i) {
        ac[i & 1][0] = fma(v[i].x, xr[i], ac[i & 1][0]);
        ac[i & 1][1] = fma(v[i].y, xr[i], ac[i & 1][1]);
      }
    }
    for (; r < r1; ++r) {
      const double xr = __ldg(x + r);
      ac[0][0] = fma(base[r * lda], xr, ac[0][0]);
      ac[0][1] = fma(base[r * lda + 1], xr, ac[0][1]);
    }
    out[(b * 2 + (r0 > 0 ? 0 : 1)) * TW + 2 * threadIdx.x] = ac[0][0] + ac[1][0];
    out[(b * 2 + (r0 > 0 ? 0 : 1)) * TW + 2 * threadIdx.x + 1] = ac[0][1] + ac[1][1];
    u += r1 - r0;
  }
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

int main() {
  const int64_t m = 5000, n = 20000, lda = 20000;
  const int64_t nct = (n + TW - 1) / TW;
  std::vector<double> ah((size_t)m * lda), xh(n + TW);
  for (size_t i = 0; i < ah.size(); ++i) ah[i] = (double)((i * 2654435761u) % 1000) * 1e-3 - 0.5;
  for (size_t i = 0; i < xh.size(); ++i) xh[i] = i < (size_t)n ? 1.0 / (1.0 + i) : 0.0;
  double *a, *x, *p, *pref;
  CK(cudaMalloc(&a, ah.size() * 8));
  CK(cudaMalloc(&x, xh.size() * 8));
  CK(cudaMalloc(&p, nct * m * 8));
  CK(cudaMalloc(&pref, nct * m * 8));
  CK(cudaMemcpy(a, ah.data(), ah.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(x, xh.data(), xh.size() * 8, cudaMemcpyHostToDevice));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = 8.0 * m * n + 8.0 * (m + n);
  std::vector<double> h0(nct * m), h1(nct * m);
  auto report = [&](const char* name, float ms) {
    CK(cudaMemcpy(h1.data(), p, nct * m * 8, cudaMemcpyDeviceToHost));
    printf("%-24s %8.2f us %7.1f GB/s %s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
           memcmp(h0.data(), h1.data(), nct * m * 8) ? "MISMATCH" : "bitwise=V0");
  };
  float ms = timeit([&] { k_v0<<<sms * 4, 256>>>(a, lda, m, n, x, pref); }, 30);
  CK(cudaMemcpy(h0.data(), pref, nct * m * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(p, pref, nct * m * 8, cudaMemcpyDeviceToDevice));
  report("v0 regs R1 4blk", ms);
#define V1(R, NB)                                                                           \
  {                                                                                         \
    CK(cudaMemset(p, 0, nct * m * 8));                                                      \
    float t = timeit([&] { k_v1<R, NB><<<sms * NB, 256>>>(a, lda, m, n, x, p); }, 30);      \
    report("v1 smem R" #R " " #NB "blk", t);                                                \
  }
  V1(1, 4) V1(2, 4) V1(2, 3) V1(2, 2) V1(3, 2) V1(4, 2) V1(4, 1)
  double* tout;
  CK(cudaMalloc(&tout, (size_t)sms * 8 * 2 * TW * 8));
  std::vector<double> xm(m, 0.5);
  double* xmd;
  CK(cudaMalloc(&xmd, m * 8));
  CK(cudaMemcpy(xmd, xm.data(), m * 8, cudaMemcpyHostToDevice));
#define VT(RU, NB)                                                                             \
  {                                                                                            \
    float t = timeit([&] { k_t<RU, NB><<<sms * NB, 256>>>(a, lda, m, n, xmd, tout); }, 30);    \
    printf("%-24s %8.2f us %7.1f GB/s\n", "A^T RU" #RU " " #NB "blk", t * 1e3, bytes / (t * 1e-3) / 1e9); \
  }
  VT(8, 4) VT(12, 3)
  {
    float t = timeit([&] { k_t<12, 3, XSr><<<sms * 3, 256>>>(a, lda, m, n, xmd, tout, XSr{}); }, 30);
    printf("%-24s %8.2f us %7.1f GB/s\n", "A^T RU12 3blk runtime XS", t * 1e3, bytes / (t * 1e-3) / 1e9);
  }
  return 0;
}
