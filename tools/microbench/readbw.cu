// Streaming-read ceilings on this GPU: what fraction of the measured copy
// peak a pure read of an 800 MB fp64 array reaches with different load paths.
// (Tuning aid for the matvec passes; not part of the library.)
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void k_ldg128(const double* __restrict__ a, size_t n2, double* out) {
  const double2* p = reinterpret_cast<const double2*>(a);
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (; i + 7 * st < n2; i += 8 * st) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(p + i + u * st));
#pragma unroll
    for (int u = 0; u < 8; u += 2) { s0 += v[u].x; s1 += v[u].y; s2 += v[u + 1].x; s3 += v[u + 1].y; }
  }
  for (; i < n2; i += st) { double2 v = p[i]; s0 += v.x; s1 += v.y; }
  if (s0 + s1 + s2 + s3 == 12345.0) out[0] = 1;
}

__global__ void k_ldg256(const double* __restrict__ a, size_t n4, double* out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (; i + 3 * st < n4; i += 4 * st) {
    double v[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3]) : "l"(a + 4 * (i + u * st)));
#pragma unroll
    for (int u = 0; u < 4; ++u) { s0 += v[u][0]; s1 += v[u][1]; s2 += v[u][2]; s3 += v[u][3]; }
  }
  if (s0 + s1 + s2 + s3 == 12345.0) out[0] = 1;
}

// TMA 1-D bulk copies (cp.async.bulk) into a 4-stage smem ring per block
template <int STAGE_BYTES, int STAGES>
__global__ void __launch_bounds__(256) k_bulk(const double* __restrict__ a, size_t nbytes, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[STAGES];
  const size_t per_block = (nbytes / gridDim.x) & ~(size_t)(STAGE_BYTES - 1);
  const size_t base = (size_t)blockIdx.x * per_block;
  const int chunks = per_block / STAGE_BYTES;
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  auto issue = [&](int c) {
    const int s = c % STAGES;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(sm + s * STAGE_BYTES);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(STAGE_BYTES));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(d), "l"((const char*)a + base + (size_t)c * STAGE_BYTES), "r"(STAGE_BYTES), "r"(b) : "memory");
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < STAGES && c < chunks; ++c) issue(c);
  double s0 = 0;
  for (int c = 0; c < chunks; ++c) {
    const int s = c % STAGES;
    const unsigned phase = (c / STAGES) & 1;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(b), "r"(phase) : "memory");
    const double* src = reinterpret_cast<const double*>(sm + s * STAGE_BYTES);
    for (int k = threadIdx.x; k < STAGE_BYTES / 8; k += 256) s0 += src[k];
    __syncthreads();
    if (threadIdx.x == 0 && c + STAGES < chunks) issue(c + STAGES);
  }
  if (s0 == 12345.0) out[0] = 1;
}

// each warp streams its own contiguous region (the pass kernels' layout)
__global__ void k_blocked(const double* __restrict__ a, size_t n2, double* out) {
  const double2* p = reinterpret_cast<const double2*>(a);
  const size_t warps = (size_t)gridDim.x * (blockDim.x / 32);
  const size_t w = (size_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const size_t s = n2 * w / warps, e = n2 * (w + 1) / warps;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  size_t i = s + lane;
  for (; i + 7 * 32 < e; i += 8 * 32) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(p + i + u * 32));
#pragma unroll
    for (int u = 0; u < 8; u += 2) { s0 += v[u].x; s1 += v[u].y; s2 += v[u + 1].x; s3 += v[u + 1].y; }
  }
  for (; i < e; i += 32) { double2 v = p[i]; s0 += v.x; s1 += v.y; }
  if (s0 + s1 + s2 + s3 == 12345.0) out[0] = 1;
}
// each block streams its own contiguous region, warps interleaved inside it
__global__ void k_blocked_cta(const double* __restrict__ a, size_t n2, double* out) {
  const double2* p = reinterpret_cast<const double2*>(a);
  const size_t s = n2 * blockIdx.x / gridDim.x, e = n2 * (blockIdx.x + 1) / gridDim.x;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  size_t i = s + threadIdx.x;
  const size_t st = blockDim.x;
  for (; i + 7 * st < e; i += 8 * st) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(p + i + u * st));
#pragma unroll
    for (int u = 0; u < 8; u += 2) { s0 += v[u].x; s1 += v[u].y; s2 += v[u + 1].x; s3 += v[u + 1].y; }
  }
  for (; i < e; i += st) { double2 v = p[i]; s0 += v.x; s1 += v.y; }
  if (s0 + s1 + s2 + s3 == 12345.0) out[0] = 1;
}

int main() {
  const size_t n = 100000000;  // 800 MB
  double *a, *out;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, n * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-36s %8.2f us  %7.1f GB/s  (%s)\n", name, best * 1e3, n * 8 / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int bps : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "blocked per-warp, %d blk/SM", bps);
    run(nm, [&] { k_blocked<<<sms * bps, 256>>>(a, n / 2, out); });
    snprintf(nm, 64, "blocked per-block, %d blk/SM", bps);
    run(nm, [&] { k_blocked_cta<<<sms * bps, 256>>>(a, n / 2, out); });
    snprintf(nm, 64, "ldg128 x8 unroll, %d blk/SM", bps);
    run(nm, [&] { k_ldg128<<<sms * bps, 256>>>(a, n / 2, out); });
    snprintf(nm, 64, "ldg256 x4 unroll, %d blk/SM", bps);
    run(nm, [&] { k_ldg256<<<sms * bps, 256>>>(a, n / 4, out); });
  }
  {
    auto k = k_bulk<32768, 4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    run("bulk 32KB x4 stages, 1 blk/SM", [&] { k<<<sms, 256, 4 * 32768>>>(a, n * 8, out); });
    run("bulk 32KB x4 stages, 148*1 (again)", [&] { k<<<sms, 256, 4 * 32768>>>(a, n * 8, out); });
  }
  {
    auto k = k_bulk<16384, 6>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384);
    run("bulk 16KB x6 stages, 2 blk/SM", [&] { k<<<sms * 2, 256, 6 * 16384>>>(a, n * 8, out); });
  }
  {
    auto k = k_bulk<8192, 8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192);
    run("bulk 8KB x8 stages, 3 blk/SM", [&] { k<<<sms * 3, 256, 8 * 8192>>>(a, n * 8, out); });
  }
  return 0;
}
