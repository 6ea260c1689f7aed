// Common plumbing for the trisolve_b200 CUDA library (sm_100a).
//
// Error handling, device helpers (streaming loads, deterministic warp/block
// reductions, last-block arrival), and the per-solve reduction workspace.
// Every reduction in the library has a FIXED combination order that depends
// only on the problem shape and the launch plan, never on timing: results are
// bitwise reproducible run to run on the same GPU model (no fp64 atomics).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/trisolve_b200.h"

namespace ts {

// Allocation, freeing and device-wide synchronisation (matrix creation and
// destruction, solver-instance setup) must not run while another thread captures a
// graph: they are the "potentially unsafe" calls of stream capture, and with a pool
// of solver threads an occasional capture lost a node to them (cudaGraphAddNode:
// invalid argument).  Such code holds the structural lock SHARED (re-entrant per
// thread); a graph build holds it EXCLUSIVE.  Lock order: structural, then graph.
inline std::shared_mutex& struct_mu() {
  static std::shared_mutex mu;
  return mu;
}
struct StructShared {
  static int& depth() {
    static thread_local int d = 0;
    return d;
  }
  StructShared() {
    if (depth()++ == 0) struct_mu().lock_shared();
  }
  ~StructShared() {
    if (--depth() == 0) struct_mu().unlock_shared();
  }
  StructShared(const StructShared&) = delete;
  StructShared& operator=(const StructShared&) = delete;
};

// ---------------------------------------------------------------- errors ----
void set_error(const char* fmt, ...);
const char* last_error();

struct Err {
  int code = 0;
};

#define TS_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::ts::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e),      \
                      __FILE__, __LINE__);                                         \
      return TS_ECUDA;                                                             \
    }                                                                              \
  } while (0)

#define TS_CHECK(rc)          \
  do {                        \
    int _rc = (rc);           \
    if (_rc != 0) return _rc; \
  } while (0)

#define TS_INVAL(...)             \
  do {                            \
    ::ts::set_error(__VA_ARGS__); \
    return TS_EINVAL;             \
  } while (0)

// ------------------------------------------------------------- constants ----
constexpr int kNT = 256;          // threads per block for every pass kernel
constexpr int kMinBlocks = 4;     // __launch_bounds__ min blocks/SM (<= 64 registers)
constexpr int kWarps = kNT / 32;  // warps per block
constexpr int kKMax = 8;          // max reduction slots per pass
constexpr int kCW = 4 * kNT;      // max dense A^T tile width (columns): up to 4 per thread
constexpr int kTMax = 8;          // max CTA order supported on device
constexpr int kEpiSmem = kTMax * kTMax + 16;  // per-block scratch for Epi::prepare

enum RedOp : int { RED_SUM = 0, RED_MIN = 1 };

// ------------------------------------------------------- device helpers ----
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// 256-bit streaming load (sm_100: LDG.E.ENL2.256); p must be 32-byte aligned
__device__ __forceinline__ void ld_stream4(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void ldg4(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ int ld_stream_i(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// Epi::kPair when declared, else false (epilogues outside the EpiBase family)
template <class E>
constexpr auto pair_of(int) -> decltype(bool(E::kPair)) { return E::kPair; }
template <class E>
constexpr bool pair_of(...) { return false; }
template <class E>
constexpr bool kPairOf = pair_of<E>(0);

// Epi::kVecBlocks when declared (resident blocks per SM of its k_vec, i.e. the
// register budget of a heavy vector epilogue), else kMinBlocks
template <class E>
constexpr auto vec_blocks_of(int) -> decltype(int(E::kVecBlocks)) { return E::kVecBlocks; }
template <class E>
constexpr int vec_blocks_of(...) { return kMinBlocks; }
template <class E>
constexpr int kVecBlocksOf = vec_blocks_of<E>(0);

// plain (coherent) 128-bit load / store of an aligned element pair
__device__ __forceinline__ double2 ld_pair(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void st_pair(double* p, double2 v) {
  *reinterpret_cast<double2*>(p) = v;
}
// ---- TMA 1-D bulk copies (cp.async.bulk) + mbarrier helpers ---------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{ .reg .pred p; TS_WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; "
      "@!p bra TS_WAIT_%=; }" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both ends 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double red_combine(int op, double a, double b) {
  return op == RED_MIN ? (b < a ? b : a) : a + b;  // fixed operand order
}
__device__ __forceinline__ double red_identity(int op) {
  return op == RED_MIN ? INFINITY : 0.0;
}

// xor-butterfly warp reduction: fixed pattern, every lane ends with the value
__device__ __forceinline__ double warp_reduce(double v, int op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_combine(op, v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block reduction of K slots; result valid in thread 0.  `sm` >= kWarps*K.
template <int K, class Ops>
__device__ __forceinline__ void block_reduce(double (&v)[K], double* sm, const Ops& ops) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_reduce(v[k], ops.op(k));
  __syncthreads();  // protect sm reuse
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm[w * K + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = sm[k];
      for (int j = 1; j < kWarps; ++j) s = red_combine(ops.op(k), s, sm[j * K + k]);
      v[k] = s;
    }
  }
}

// Live kernel accounting: earliest block start (atomicMin) to the finisher.
struct KTimer {
  unsigned long long start;
  unsigned long long total_ns;
  long long count;
  long long pad;
};
__device__ __forceinline__ void ktimer_begin(KTimer* kt) {
  if (kt && threadIdx.x == 0) atomicMin(&kt->start, globaltimer());
}
// kernels that load ahead of the state word take their entry time first, so
// the hoisted work is inside the accounted interval
__device__ __forceinline__ void ktimer_begin_at(KTimer* kt, unsigned long long t_entry) {
  if (kt && threadIdx.x == 0) atomicMin(&kt->start, t_entry);
}
// `products`: matrix products the launch performed (pair / chain kernels: 2 / 2 t), so
// the class average stays a time per product
__device__ __forceinline__ void ktimer_end(KTimer* kt, int products = 1) {
  if (kt) {
    const unsigned long long now = globaltimer();
    kt->total_ns += now - kt->start;
    kt->count += products;
    kt->start = ~0ull;
  }
}

// Per-solve reduction workspace (device pointers).
struct Work {
  double* bacc;     // [pmax * kKMax] per-block partials
  double* facc;     // [pmax * kKMax] split-row / split-tile epilogue partials
  double* bpart;    // [pmax * 2] block boundary row-piece sums (first, last)
  double* tpart;    // [pmax * 2 * kCW] block boundary tile pieces
  double* npart;    // dense A v: [ntiles * m] per-(tile,row) partials, then group slots + counters
  unsigned* cnt;    // [pmax] split counters (self-resetting)
  unsigned* done;   // [4] completion counters (self-resetting)
  int pmax;
};

// All threads: returns true in every thread of the last block to arrive.
__device__ __forceinline__ bool arrive_last(unsigned* counter, unsigned total, int* sflag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    int last = (prev == total - 1);
    if (last) *counter = 0u;  // reset for the next launch (all others arrived)
    *sflag = last;
  }
  __syncthreads();
  bool last = *sflag != 0;
  if (last) __threadfence();
  return last;
}

// Final fixed-order reduction of per-block partials (+ fix partials), done by
// the whole last block; result in thread 0.
template <int K, class Ops>
__device__ __forceinline__ void reduce_partials(const double* bacc, const double* facc, int nb,
                                                double (&out)[K], double* sm, const Ops& ops) {
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = red_identity(ops.op(k));
  for (int b = threadIdx.x; b < nb; b += kNT) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double v = __ldcg(bacc + (size_t)b * kKMax + k);
      if (facc) v = red_combine(ops.op(k), v, __ldcg(facc + (size_t)b * kKMax + k));
      out[k] = red_combine(ops.op(k), out[k], v);
    }
  }
  block_reduce<K>(out, sm, ops);
}

// ---------------------------------------------------------- vector loads ----
// kCoh selects L2-coherent loads for vectors rewritten while a kernel runs;
// the pass kernels read their input vector through the read-only path.
template <bool kCoh>
__device__ __forceinline__ double ldx(const double* p) {
  if constexpr (kCoh) return __ldcg(p);
  else return __ldg(p);
}
template <bool kCoh>
__device__ __forceinline__ double2 ldx2(const double* p) {
  if constexpr (kCoh) return __ldcg(reinterpret_cast<const double2*>(p));
  else return __ldg(reinterpret_cast<const double2*>(p));
}

inline int ceil_div_i(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace ts
