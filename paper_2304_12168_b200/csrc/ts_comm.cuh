// Column sharding across GPUs: a deterministic one-shot all-reduce over
// NVLink peer memory, fused into the pass epilogues.
//
// With A split into column blocks A_p (one per rank), every m-space vector is
// replicated and every n-space vector is local (BASELINE north_star, SURVEY
// 8(e)).  Two exchange kinds exist per iteration:
//
//  * A v = sum_p A_p v_p: the local pass stores its partial m-vector straight
//    into this rank's slot of a symmetric (IPC-shared) buffer; k_ar_vec then
//    waits for every rank's epoch flag, sums the P partials in FIXED RANK
//    ORDER (so all ranks get bit-identical vectors and take identical
//    decisions) and applies the pass's own epilogue (d = v - b', phi dots,
//    residuals ...) and finisher.
//  * reductions over n-space (||c||^2, ||A^T r||^2, min x, ||x||^2): the local
//    pass's finisher parks its K partial scalars in the symmetric buffer
//    instead of finishing; k_ar_scalars combines them across ranks (slots
//    flagged replicated keep the local value) and runs the real finisher.
//
// Synchronisation: one monotonically increasing epoch per exchange (all
// ranks issue the same exchange sequence); rank p announces epoch e by a
// release store into flags[p] of every peer, then waits until its own
// flags[q] >= e for all q.  Payload slots alternate with the epoch parity:
// a rank can only reach the producer of epoch e+2 after every peer arrived at
// e+1, i.e. after they finished reading epoch e's buffers.  AR grids never
// exceed one resident wave, so block 0 (the announcer) is always running.
//
// Emulated worlds (ts_comm_create_local): W ranks of one process on ONE GPU,
// each solved by its own host thread.  Kernels that spin on each other must
// not share a GPU, so there the device barrier does not wait: every exchange
// is ordered on the host instead (LocalGroup::exchange: each rank records an
// event after its producer kernel, all ranks meet, each rank's stream waits
// on every rank's event before the consumer kernel).  Everything else — the
// symmetric slots and their epoch parity, rank-ordered sums, deferred
// scalars, halo copies, peer reads — is the same device code as across GPUs.
#pragma once

#include <chrono>
#include <condition_variable>
#include <memory>
#include <mutex>

#include "ts_state.cuh"

namespace ts {

constexpr int kMaxRanks = 16;
constexpr int kArScalars = 16;  // scalar area per slot (doubles)

struct CommDev {
  int rank = 0, world = 1;
  size_t slot = 0;                        // doubles per epoch slot (vector + scalars)
  double* const* psym = nullptr;          // [world] peer symmetric buffers (device array)
  unsigned long long* const* pflags = nullptr;  // [world] peer flag arrays
  unsigned long long* flags = nullptr;    // local flags [world]
  unsigned long long* epoch = nullptr;    // local exchange counter
  double* sym = nullptr;                  // local symmetric buffer [2 * slot]
  size_t vec_cap = 0;                     // vector capacity per slot
  int emulated = 0;                       // ranks share this GPU: exchanges are host-ordered
};

// host rendezvous of an emulated world (one process, one GPU, W host threads)
struct LocalGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;
  std::vector<cudaEvent_t> ev;  // per rank: its last producer kernel
  explicit LocalGroup(int w) : world(w), ev((size_t)w, nullptr) {}
  ~LocalGroup() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
  // false: a rank did not arrive within the timeout (the world is broken)
  bool meet() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct Comm {
  int dev = 0, rank = 0, world = 1;
  size_t vec_cap = 0;
  double* sym = nullptr;
  unsigned long long* flags = nullptr;
  unsigned long long* epoch = nullptr;
  double** psym_d = nullptr;
  unsigned long long** pflags_d = nullptr;
  std::vector<void*> opened;
  std::shared_ptr<LocalGroup> local;  // emulated world (nullptr: one rank per GPU)
  // emulated world: order this rank's next kernel after every rank's last one
  int exchange(cudaStream_t s) const {
    if (!local) return 0;
    if (cudaEventRecord(local->ev[rank], s) != cudaSuccess) {
      set_error("exchange: cudaEventRecord failed");
      return TS_ECUDA;
    }
    if (!local->meet()) {
      set_error("emulated world: a rank did not reach the exchange");
      return TS_ECUDA;
    }
    for (int q = 0; q < world; ++q)
      if (q != rank && cudaStreamWaitEvent(s, local->ev[q], 0) != cudaSuccess) {
        set_error("exchange: cudaStreamWaitEvent failed");
        return TS_ECUDA;
      }
    if (!local->meet()) {  // every rank queued its waits before any event is re-recorded
      set_error("emulated world: a rank did not reach the exchange");
      return TS_ECUDA;
    }
    return 0;
  }
  CommDev dev_view() const {
    CommDev c;
    c.rank = rank;
    c.world = world;
    c.slot = vec_cap + kArScalars;
    c.psym = psym_d;
    c.pflags = pflags_d;
    c.flags = flags;
    c.epoch = epoch;
    c.sym = sym;
    c.vec_cap = vec_cap;
    c.emulated = local ? 1 : 0;
    return c;
  }
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_peer(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// every block: announce (block 0) and wait for all ranks at epoch e (an
// emulated world is ordered by the host: nothing to wait for)
__device__ __forceinline__ void comm_barrier(const CommDev& c, unsigned long long e) {
  if (c.emulated) {
    __syncthreads();
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < c.world; ++q) st_release_sys(c.pflags[q] + c.rank, e);
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < c.world; ++q)
      while (ld_acquire_sys(c.flags + q) < e) __nanosleep(64);
  }
  __syncthreads();
}

__device__ __forceinline__ size_t slot_base(const CommDev& c, unsigned long long e) {
  return (size_t)(e & 1ull) * c.slot;
}

// local pass epilogue replacing `Epi` on a sharded A v: park the partial
// m-vector in this rank's slot (same activity predicate as the consumer)
template <class Epi>
struct EpiSymStore {
  static constexpr int K = 1;
  Epi e;
  CommDev c;
  __device__ int op(int) const { return RED_SUM; }
  __device__ bool active() const { return e.active(); }
  __device__ void idle() const {}  // k_ar_vec owns the loop condition
  __device__ KTimer* timer() const { return e.timer(); }
  __device__ void finish_block() const {}
  __device__ void count_launch() const { e.count_launch(); }
  __device__ void prepare(double* smem) { e.prepare(smem); }
  __device__ void elem(int64_t i, double v, double (&)[K]) const {
    c.sym[slot_base(c, *c.epoch + 1) + i] = v;
  }
  __device__ void finish(double (&)[K]) const {}
};

// wraps a pass epilogue: same per-element work, finisher deferred to k_ar_scalars
template <class Epi>
struct EpiDefer {
  static constexpr int K = Epi::K;
  static constexpr bool kPair = kPairOf<Epi>;
  static constexpr int kVecBlocks = kVecBlocksOf<Epi>;
  Epi e;
  CommDev c;
  __device__ int op(int k) const { return e.op(k); }
  __device__ bool active() const { return e.active(); }
  __device__ void idle() const {}  // the AR kernel owns the loop condition
  __device__ KTimer* timer() const { return e.timer(); }
  __device__ void finish_block() const {}
  __device__ void count_launch() const { e.count_launch(); }
  __device__ void prepare(double* smem) { e.prepare(smem); }
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const { e.elem(i, y, acc); }
  __device__ void elem(int64_t i, double (&acc)[K]) const { e.elem(i, acc); }
  __device__ void elem2(int64_t i, double (&acc)[K]) const {
    if constexpr (kPair) e.elem2(i, acc);
  }
  __device__ void finish(double (&red)[K]) const {
    double* s = c.sym + slot_base(c, *c.epoch + 1) + c.vec_cap;
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = red[k];
  }
};

// one block: combine the parked scalars of every rank in rank order, then the
// real finisher.  shard_mask bit k set: slot k is a per-rank partial.
template <class Epi>
__global__ void __launch_bounds__(kNT) k_ar_scalars(Epi epi, CommDev c, unsigned shard_mask) {
  constexpr int K = Epi::K;
  __shared__ int live;
  if (threadIdx.x == 0) {
    epi.count_launch();
    live = epi.active();
  }
  __syncthreads();
  if (!live) {
    if (threadIdx.x == 0) epi.idle();
    return;
  }
  const unsigned long long e = *c.epoch + 1;
  comm_barrier(c, e);
  if (threadIdx.x == 0) {
    const size_t base = slot_base(c, e) + c.vec_cap;
    double red[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (shard_mask & (1u << k)) {
        double v = ld_peer(c.psym[0] + base + k);
        for (int q = 1; q < c.world; ++q) v = red_combine(epi.op(k), v, ld_peer(c.psym[q] + base + k));
        red[k] = v;
      } else {
        red[k] = c.sym[base + k];
      }
    }
    *c.epoch = e;
    epi.finish(red);
  }
  __syncthreads();
  epi.finish_block();
}

// Row-block sharding (square A, SURVEY 8(e) for C4): every vector is split
// like the rows, and a pass over this rank's rows reads its input vector up to
// `hw` entries past either end of the local block.  k_halo publishes the
// block's first and last hw entries in this rank's symmetric slot, meets every
// rank at the epoch barrier, and copies the left neighbour's tail / right
// neighbour's head into the vector's halo padding (x[-hw, 0) and
// x[n, n + hw)).  One block; a pass whose epilogue is inactive skips it on
// every rank alike (the state is replicated), so epochs stay in step.
// phase: 1 publish, 2 barrier + copy-in, 3 both (an emulated world launches
// the two halves apart, with the host exchange between them).
template <class Epi>
__global__ void __launch_bounds__(kNT) k_halo(Epi epi, double* x, int64_t n, int64_t hw, CommDev c, int phase) {
  __shared__ int live;
  if (threadIdx.x == 0) live = epi.active();
  __syncthreads();
  if (!live) return;
  const unsigned long long e = *c.epoch + 1;
  const size_t base = slot_base(c, e);
  if (phase & 1) {
    for (int64_t i = threadIdx.x; i < hw; i += kNT) {
      c.sym[base + i] = x[i];                // head: the left neighbour's right halo
      c.sym[base + hw + i] = x[n - hw + i];  // tail: the right neighbour's left halo
    }
    __syncthreads();
  }
  if (!(phase & 2)) return;
  comm_barrier(c, e);
  for (int64_t i = threadIdx.x; i < hw; i += kNT) {
    x[-hw + i] = c.rank > 0 ? ld_peer(c.psym[c.rank - 1] + base + hw + i) : 0.0;
    x[n + i] = c.rank + 1 < c.world ? ld_peer(c.psym[c.rank + 1] + base + i) : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) *c.epoch = e;
}

// sum the ranks' partial m-vectors in rank order and run the pass epilogue
template <class Epi>
__global__ void __launch_bounds__(kNT) k_ar_vec(int64_t len, Epi epi, Work wk, CommDev c) {
  constexpr int K = Epi::K;
  __shared__ double sm[kWarps * kKMax];
  __shared__ int sflag;
  if (blockIdx.x == 0 && threadIdx.x == 0) epi.count_launch();
  if (!epi.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.idle();
    return;
  }
  const unsigned long long e = *c.epoch + 1;
  __shared__ double epi_smem[kEpiSmem];
  epi.prepare(epi_smem);
  comm_barrier(c, e);  // (its __syncthreads also publishes epi_smem)
  const size_t base = slot_base(c, e);
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = red_identity(epi.op(k));
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < len; i += stride) {
    double y = ld_peer(c.psym[0] + base + i);
    for (int q = 1; q < c.world; ++q) y += ld_peer(c.psym[q] + base + i);
    epi.elem(i, y, acc);
  }
  block_reduce<K>(acc, sm, epi);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wk.bacc[blockIdx.x * kKMax + k] = acc[k];
  }
  if (arrive_last(wk.done, gridDim.x, &sflag)) {
    double red[K];
    reduce_partials<K>(wk.bacc, nullptr, (int)gridDim.x, red, sm, epi);
    if (threadIdx.x == 0) {
      *c.epoch = e;
      epi.finish(red);
    }
    __syncthreads();
    epi.finish_block();
  }
}

}  // namespace ts
