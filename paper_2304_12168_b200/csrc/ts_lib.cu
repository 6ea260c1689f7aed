// trisolve_b200: C ABI entry points, matrix creation, and the solve drivers.
//
// A solve = init kernels, then a CUDA graph whose single WHILE node runs one
// device-resident iteration per trip (see ts_state.cuh) until the state
// leaves RUNNING, needs host maintenance (CTA residual recheck every 250
// iterations, TA b' revalidation every 512 pivots — both are cadences of the
// reference, centering.py:344-352 / triangle.py:239-242), or the device trace
// ring (seg_cap rows) needs flushing.  The host synchronises only at those
// points, never inside an iteration.
#include <execinfo.h>
#include <fcntl.h>
#include <signal.h>
#include <unistd.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "ts_cta.cuh"
#include "ts_comm.cuh"
#include "ts_mmio.cuh"

namespace ts {

// ---------------------------------------------------------------- errors ----
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

static thread_local long long g_launches = 0;  // kernels enqueued by this thread

// TS_BACKTRACE=<file>: append the native stack to <file> on SIGSEGV / SIGABRT
// (addresses resolve against this library with addr2line; built with -lineinfo)
static char g_bt_path[512] = "";
static void segv_backtrace(int sig) {
  void* bt[64];
  const int n = backtrace(bt, 64);
  const int fd = open(g_bt_path, O_WRONLY | O_CREAT | O_APPEND, 0644);
  if (fd >= 0) {
    const char* hdr = sig == SIGSEGV ? "SIGSEGV\n" : "SIGABRT\n";
    ssize_t w = write(fd, hdr, 8);
    (void)w;
    backtrace_symbols_fd(bt, n, fd);
    close(fd);
  }
  _exit(128 + sig);
}
static struct SegvInit {
  SegvInit() {
    const char* e = getenv("TS_BACKTRACE");
    if (e && *e) {
      snprintf(g_bt_path, sizeof(g_bt_path), "%s", e);
      signal(SIGSEGV, segv_backtrace);
      signal(SIGABRT, segv_backtrace);
    }
  }
} g_segv_init;

// ------------------------------------------------------- device guards ----
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

static std::once_flag g_pool_once[64];
static void setup_pool(int dev) {
  if (dev < 0 || dev >= 64) return;
  std::call_once(g_pool_once[dev], [dev]() {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

static int sm_count(int dev) {
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

// ------------------------------------------------------ storage pools ----
// Retired matrices: ts_matrix_destroy parks an unsharded handle here (device
// storage, launch plans and its cached solver instances with their
// instantiated graphs) instead of freeing it; a later create of the same
// kind and shape on the same device takes it back, uploads the new entries
// into the same buffers and rebuilds only what depends on them (Frobenius
// norm; for CSR the transpose and the plan tables).  cudaMalloc / cudaFree
// of hundreds of MB and graph instantiation then leave the per-call path of
// a stream of same-shaped solves.  TS_MATRIX_POOL=0 disables it;
// ts_pool_trim() (and any failing allocation) releases it.
static std::mutex g_retire_mu;
static std::vector<Mat*> g_retired;
constexpr size_t kRetireMax = 2;  // handles kept per process

static bool matrix_pool_enabled() {
  static const bool on = [] {
    const char* e = getenv("TS_MATRIX_POOL");
    return !(e && !strcmp(e, "0"));
  }();
  return on;
}

static void free_matrix(Mat* A);

static Mat* retire_take(int dev, int kind, int64_t m, int64_t n, int64_t nnz) {
  if (!matrix_pool_enabled()) return nullptr;
  std::lock_guard<std::mutex> g(g_retire_mu);
  for (size_t i = 0; i < g_retired.size(); ++i) {
    Mat* A = g_retired[i];
    if (A->dev == dev && A->kind == kind && A->m == m && A->n == n && A->nnz == nnz) {
      g_retired.erase(g_retired.begin() + i);
      return A;
    }
  }
  return nullptr;
}

static int pool_trim_device(int dev) {  // dev < 0: all devices
  std::vector<Mat*> drop;
  {
    std::lock_guard<std::mutex> g(g_retire_mu);
    for (size_t i = 0; i < g_retired.size();) {
      if (dev < 0 || g_retired[i]->dev == dev) {
        drop.push_back(g_retired[i]);
        g_retired.erase(g_retired.begin() + i);
      } else {
        ++i;
      }
    }
  }
  for (Mat* A : drop) free_matrix(A);
  return (int)drop.size();
}

// cudaMalloc that releases retired storage and retries once on failure
static cudaError_t dev_malloc(void** p, size_t bytes, int dev) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess && pool_trim_device(dev) > 0) {
    cudaGetLastError();
    e = cudaMalloc(p, bytes);
  }
  return e;
}
template <class T>
static cudaError_t dev_malloc(T** p, size_t bytes, int dev) {
  return dev_malloc(reinterpret_cast<void**>(p), bytes, dev);
}

static void free_plan(RowPlan& p) {
  if (p.wrow) cudaFree(p.wrow);
  if (!p.sell_borrowed)
    for (void* q : {(void*)p.sell_sp, (void*)p.sell_ci, (void*)p.sell_val})
      if (q) cudaFree(q);
  if (!p.slab_borrowed)
    for (void* q : {(void*)p.slab_cb, (void*)p.slab_sp, (void*)p.slab_wr, (void*)p.slab_pos,
                    (void*)p.slab_col, (void*)p.slab_val})
      if (q) cudaFree(q);
  p.sell_borrowed = 0;
  p.slab_borrowed = 0;
  p.slab_cb = p.slab_sp = p.slab_pos = nullptr;
  p.slab_wr = nullptr;
  p.slab_col = nullptr;
  p.slab_val = nullptr;
  p.wrow = nullptr;
  p.sell_sp = nullptr;
  p.sell_ci = nullptr;
  p.sell_val = nullptr;
  p.sell_slots = 0;
}

// Dense upload: one linear copy when both sides are contiguous, else row slabs
// of ~16 MB (one copy-engine command per slab, so
// the small host<->device copies of a solve running concurrently on another
// stream (state, b, x) are not queued behind a whole 800 MB transfer
// (double-buffered pipelines of same-shaped problems).
static cudaError_t upload_rows(double* dst, int64_t dld, const double* src, int64_t sld, int64_t m,
                               int64_t n, cudaStream_t st) {
  if (dld == n && sld == n)  // contiguous both sides: one linear copy
    return cudaMemcpyAsync(dst, src, (size_t)m * n * sizeof(double), cudaMemcpyDefault, st);
  const int64_t slab = std::max<int64_t>(1, ((int64_t)16 << 20) / std::max<int64_t>(1, n * 8));
  for (int64_t r = 0; r < m; r += slab) {
    const int64_t rows = std::min(slab, m - r);
    cudaError_t e = cudaMemcpy2DAsync(dst + r * dld, dld * sizeof(double), src + r * sld,
                                      sld * sizeof(double), n * sizeof(double), rows,
                                      cudaMemcpyDefault, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// a new plan replaces `old` in place when the geometry is unchanged (cached
// graphs bake the grid and the plan-table pointer); false: geometry changed
static bool adopt_plan(RowPlan& old, RowPlan& nw, int64_t rows, cudaStream_t st) {
  const bool same = old.kind == nw.kind && old.P == nw.P && (old.wrow != nullptr) == (nw.wrow != nullptr) &&
                    old.sell_slots == nw.sell_slots && (old.sell_sp != nullptr) == (nw.sell_sp != nullptr) &&
                    old.slab_slots == nw.slab_slots && old.slab_nsl == nw.slab_nsl &&
                    old.slab_maxw == nw.slab_maxw;
  if (same) {
    if (nw.wrow)
      cudaMemcpyAsync(old.wrow, nw.wrow, (size_t)nw.P * kWarps * sizeof(int),
                      cudaMemcpyDeviceToDevice, st);
    if (nw.sell_sp && !nw.sell_borrowed) {
      cudaMemcpyAsync(old.sell_sp, nw.sell_sp, (size_t)((rows + 31) / 32 + 1) * sizeof(int),
                      cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(old.sell_ci, nw.sell_ci, (size_t)nw.sell_slots * sizeof(int), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(old.sell_val, nw.sell_val, (size_t)nw.sell_slots * sizeof(double),
                      cudaMemcpyDeviceToDevice, st);
    }
    if (nw.slab_sp && !nw.slab_borrowed) {
      const size_t nsp = (size_t)nw.P * nw.slab_nsl + 1, npos = (size_t)nw.P * nw.slab_rows;
      cudaMemcpyAsync(old.slab_cb, nw.slab_cb, (nw.P + 1) * sizeof(int), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(old.slab_sp, nw.slab_sp, nsp * sizeof(int), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(old.slab_wr, nw.slab_wr, (size_t)nw.P * 33 * sizeof(int2), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(old.slab_pos, nw.slab_pos, npos * sizeof(int), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(old.slab_col, nw.slab_col, nw.slab_slots * sizeof(uint16_t), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(old.slab_val, nw.slab_val, nw.slab_slots * sizeof(double), cudaMemcpyDeviceToDevice, st);
    }
    cudaStreamSynchronize(st);
    free_plan(nw);
  } else {
    if (nw.sell_borrowed) {  // nw refilled old's tables: they change owner, not freed
      old.sell_sp = nullptr;
      old.sell_ci = nullptr;
      old.sell_val = nullptr;
      nw.sell_borrowed = 0;
    }
    if (nw.slab_borrowed) {
      old.slab_cb = old.slab_sp = old.slab_pos = nullptr;
      old.slab_wr = nullptr;
      old.slab_col = nullptr;
      old.slab_val = nullptr;
      nw.slab_borrowed = 0;
    }
    free_plan(old);
    old = nw;
  }
  nw = RowPlan();
  return same;
}

// Device -> host reads of the creation path land in pinned scratch first: a
// copy into pageable memory is synchronous inside the driver and stalls the
// kernels of solves running concurrently on other streams.
static cudaError_t d2h_pinned(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  static thread_local void* buf = nullptr;
  static thread_local size_t cap = 0;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, src) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  }
  if (cap < bytes) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    cudaError_t e = cudaHostAlloc(&buf, bytes, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    cap = bytes;
  }
  cudaError_t e = cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) memcpy(dst, buf, bytes);
  return e;
}

// Pinned host blocks for solver outputs (x, b', r): the device->host copy of
// a result then runs at full PCIe rate instead of through the driver's
// pageable staging.  Freed blocks are cached by exact size.
static std::mutex g_host_mu;
static std::vector<std::pair<size_t, void*>> g_host_free;
static size_t g_host_cached = 0;
constexpr size_t kHostCacheMax = (size_t)1 << 31;

// ------------------------------------------------------------ workspace ----
// Owns stream-ordered allocations for one call.
struct Arena {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Arena(cudaStream_t s) : st(s) {}
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <class T>
  int get(T** out, size_t count) {
    void* p = nullptr;
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    if (e != cudaSuccess) {
      set_error("cudaMallocAsync(%zu) failed: %s", bytes, cudaGetErrorString(e));
      return TS_ENOMEM;
    }
    ptrs.push_back(p);
    *out = static_cast<T*>(p);
    return 0;
  }
};

static int make_work(Arena& ar, int pmax, Work* w, int64_t npart = 0) {
  w->pmax = pmax;
  TS_CHECK(ar.get(&w->npart, (size_t)std::max<int64_t>(npart, 1)));
  TS_CHECK(ar.get(&w->bacc, (size_t)pmax * kKMax));
  TS_CHECK(ar.get(&w->facc, (size_t)pmax * kKMax));
  TS_CHECK(ar.get(&w->bpart, (size_t)pmax * 2));
  TS_CHECK(ar.get(&w->tpart, (size_t)pmax * 2 * kCW));
  TS_CHECK(ar.get(&w->cnt, (size_t)pmax));
  TS_CHECK(ar.get(&w->done, 4));
  TS_CUDA(cudaMemsetAsync(w->npart, 0, sizeof(double) * std::max<int64_t>(npart, 1), ar.st));
  TS_CUDA(cudaMemsetAsync(w->cnt, 0, sizeof(unsigned) * pmax, ar.st));
  TS_CUDA(cudaMemsetAsync(w->done, 0, sizeof(unsigned) * 4, ar.st));
  return 0;
}

// copy `count` doubles from any pointer (host or device) into a fresh buffer
static int stage_in(Arena& ar, const double* src, size_t count, double** out) {
  TS_CHECK(ar.get(out, count));
  if (count) TS_CUDA(cudaMemcpyAsync(*out, src, count * sizeof(double), cudaMemcpyDefault, ar.st));
  return 0;
}

// ----------------------------------------------------------------- plans ----
static void flat_ranges(int64_t E, int64_t P, int64_t b, int wid, int64_t* s, int64_t* e) {
  const int64_t S0 = E * b / P, S1 = E * (b + 1) / P, L = S1 - S0;
  *s = S0 + L * wid / kWarps;
  *e = S0 + L * (wid + 1) / kWarps;
}

int plan_rows_csr(const int* rp, int64_t rows, int64_t nnz, int sms, RowPlan* out,
                  cudaStream_t st) {
  RowPlan p;
  const int64_t pmax = resident_blocks(sms);
  const bool long_rows = rows > 0 && nnz / rows >= 32 && nnz >= (int64_t)kWarps * 256;
  if (!long_rows) {
    // thread-per-row CSR for small (L2-resident, latency-bound) matrices, the
    // sliced-ELL copy (coalesced, no row-pointer chase) once the pass is
    // HBM-bound; TS_CSR_SHORT=thread|sell forces one (kernel comparisons).
    // The SELL tables are built by build_sell() on the device arrays.
    const char* force = getenv("TS_CSR_SHORT");
    bool thread_rows = nnz < ((int64_t)1 << 21);
    if (force && !strcmp(force, "thread")) thread_rows = true;
    if (force && !strcmp(force, "sell")) thread_rows = false;
    p.kind = thread_rows ? PLAN_SHORT : PLAN_SELL;
    const int64_t g = thread_rows ? (rows + kNT - 1) / kNT : ((rows + 31) / 32 + kWarps - 1) / kWarps;
    p.P = (int)std::max<int64_t>(1, std::min(g, pmax));
    *out = p;
    return 0;
  }
  // long rows of near-uniform length (no row above twice the mean): one warp per
  // row with prefetched chunks (k_rows_wrow); else the load-balanced flat split.
  // TS_CSR_LONG=flat forces the flat split.
  {
    const char* lf = getenv("TS_CSR_LONG");
    int64_t maxlen = 0;
    for (int64_t r = 0; r < rows; ++r) maxlen = std::max<int64_t>(maxlen, rp[r + 1] - rp[r]);
    if (!(lf && !strcmp(lf, "flat")) && maxlen * rows <= 2 * nnz) {
      p.kind = PLAN_WROW;
      p.P = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * kWrowBlocks, (rows + kWarps - 1) / kWarps));
      *out = p;
      return 0;
    }
  }
  p.kind = PLAN_FLAT;
  p.P = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * kFlatBlocks, nnz / ((int64_t)kWarps * 256)));
  std::vector<int> wr((size_t)p.P * kWarps);
  for (int64_t b = 0; b < p.P; ++b)
    for (int w = 0; w < kWarps; ++w) {
      int64_t s, e;
      flat_ranges(nnz, p.P, b, w, &s, &e);
      wr[b * kWarps + w] = (int)first_row_at(rp, rows, s);
    }
  TS_CUDA(cudaMalloc(&p.wrow, wr.size() * sizeof(int)));
  TS_CUDA(cudaMemcpyAsync(p.wrow, wr.data(), wr.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  TS_CUDA(cudaStreamSynchronize(st));
  *out = p;
  return 0;
}

int plan_rows_dense(int64_t m, int64_t n, int sms, RowPlan* out, cudaStream_t) {
  RowPlan p;
  if (n < 128 || m * n < (int64_t)kWarps * 256) {
    p.kind = PLAN_SHORT;
    p.P = (int)std::max<int64_t>(1, std::min((m + kNT - 1) / kNT, (int64_t)resident_blocks(sms)));
  } else {
    p.kind = PLAN_TILE;
    p.P = tile_grid(m, n, sms, kTileNBlocks);
    // small and L2-resident: one warp per row (TS_DENSE_SMALL=tile keeps the tile kernel)
    const char* e = getenv("TS_DENSE_SMALL");
    if (wdense_fits(m, n) && !(e && !strcmp(e, "tile"))) {
      p.wdense = 1;
      p.P = wdense_grid(m, sms);
    }
  }
  *out = p;
  return 0;
}

// ------------------------------------------------------ small kernels ----
struct EpiFroDense {
  static constexpr int K = 1;
  const double* a;
  int64_t lda, n;
  double* out;
  __device__ int op(int) const { return RED_SUM; }
  __device__ bool active() const { return true; }
  __device__ void idle() const {}
  __device__ KTimer* timer() const { return nullptr; }
  __device__ void finish_block() const {}
  __device__ void count_launch() const {}
  __device__ void prepare(double*) {}
  __device__ void elem(int64_t i, double (&acc)[K]) const {
    const double v = a[(i / n) * lda + (i % n)];
    acc[0] = fma(v, v, acc[0]);
  }
  __device__ void finish(double (&r)[K]) const { *out = sqrt(r[0]); }
};
struct EpiFroVals {
  static constexpr int K = 1;
  const double* v;
  double* out;
  __device__ int op(int) const { return RED_SUM; }
  __device__ bool active() const { return true; }
  __device__ void idle() const {}
  __device__ KTimer* timer() const { return nullptr; }
  __device__ void finish_block() const {}
  __device__ void count_launch() const {}
  __device__ void prepare(double*) {}
  __device__ void elem(int64_t i, double (&acc)[K]) const { acc[0] = fma(v[i], v[i], acc[0]); }
  __device__ void finish(double (&r)[K]) const { *out = sqrt(r[0]); }
};
// min / max of column indices (validation)
struct EpiIdxRange {
  static constexpr int K = 2;
  const int* ci;
  double* out;
  __device__ int op(int k) const { return RED_MIN; }
  __device__ bool active() const { return true; }
  __device__ void idle() const {}
  __device__ KTimer* timer() const { return nullptr; }
  __device__ void finish_block() const {}
  __device__ void count_launch() const {}
  __device__ void prepare(double*) {}
  __device__ void elem(int64_t i, double (&acc)[K]) const {
    const double v = (double)ci[i];
    acc[0] = py_min(acc[0], v);
    acc[1] = py_min(acc[1], -v);
  }
  __device__ void finish(double (&r)[K]) const {
    out[0] = r[0];
    out[1] = -r[1];
  }
};

// max |row - column| over the stored entries (the bandwidth of a square matrix)
__global__ void k_csr_band(const int* rowid, const int* ci, int64_t nnz, int* out) {
  int mx = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int d = rowid[k] - ci[k];
    mx = max(mx, d < 0 ? -d : d);
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0) atomicMax(out, mx);
}

__global__ void k_expand_rows(const int* rp, int64_t rows, int* rowid) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    for (int k = rp[r]; k < rp[r + 1]; ++k) rowid[k] = (int)r;
}
// exact transposed copy (32 x 32 tiles through shared memory)
__global__ void k_transpose(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                            double* __restrict__ t, int64_t ldt) {
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < m && c < n) tile[j][threadIdx.x] = a[r * lda + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t c = c0 + j, r = r0 + threadIdx.x;
    if (r < m && c < n) t[c * ldt + r] = tile[threadIdx.x][j];
  }
}
__global__ void k_iota(int* v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int)i;
}
__global__ void k_gather_T(const int* perm, const int* rowid, const double* val, int* ciT,
                           double* valT, int64_t nnz) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int k = perm[j];
    ciT[j] = rowid[k];
    valT[j] = val[k];
  }
}
__global__ void k_rowptr_from_keys(const int* keys, int64_t nnz, int64_t ncols, int* rpT) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kc = (j < nnz) ? keys[j] : ncols;
    const int64_t kp = (j > 0) ? keys[j - 1] : -1;
    for (int64_t c = kp + 1; c <= kc; ++c) rpT[c] = (int)j;
  }
}

// sliced-ELL copy (k_rows_sell): 32 x the longest row of each 32-row slice
__global__ void k_sell_width(const int* rp, int64_t rows, int64_t nsl, int* w32) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= nsl; q += (int64_t)gridDim.x * blockDim.x) {
    int w = 0;
    if (q < nsl)
      for (int64_t r = q * 32; r < rows && r < q * 32 + 32; ++r) w = max(w, rp[r + 1] - rp[r]);
    w32[q] = 32 * w;
  }
}
// slot (slice q, entry k, lane l) = sp[q] + 32 k + l <- entry k of row 32 q + l
__global__ void k_sell_fill(const int* rp, const int* ci, const double* val, int64_t rows, int64_t nsl,
                            const int* sp, int* sci, double* sval) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nsl * 32; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = t >> 5, r = t;
    const int l = (int)(t & 31);
    const int b0 = sp[q], w = (sp[q + 1] - b0) >> 5;
    const int k0 = r < rows ? rp[r] : 0, len = r < rows ? rp[r + 1] - k0 : 0;
    for (int k = 0; k < w; ++k) {
      const int64_t d = (int64_t)b0 + 32 * k + l;
      sci[d] = k < len ? ci[k0 + k] : kSellPad;
      sval[d] = k < len ? val[k0 + k] : 0.0;
    }
  }
}

// column-slab copy (k_slab_av): per (slab, row) the row's run of entries
// inside the slab (CSR rows sorted by column: contiguous); flags unsorted rows
__global__ void k_slab_runs(const int* rp, const int* ci, int64_t m, const int* cb, int P, int* cnt, int* start,
                            int* unsorted) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    int e = rp[r];
    const int e1 = rp[r + 1];
    for (int k = e + 1; k < e1; ++k)
      if (ci[k] < ci[k - 1]) *unsorted = 1;
    for (int s = 0; s < P; ++s) {
      const int st = e, lim = cb[s + 1];
      while (e < e1 && ci[e] < lim) ++e;
      cnt[(int64_t)s * m + r] = e - st;
      start[(int64_t)s * m + r] = st;
    }
  }
}
__global__ void k_slab_iota(int64_t m, int P, int* rows, int* offs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)P * m; i += (int64_t)gridDim.x * blockDim.x)
    rows[i] = (int)(i % m);
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= P; s += (int64_t)gridDim.x * blockDim.x)
    offs[s] = (int)(s * m);
}
// slice widths (the first, longest row of each sorted slice) and the position
// (slice * 32 + lane) of every row in its slab's order
__global__ void k_slab_tables(const int* slen, const int* srow, int64_t m, int P, int nsl, int* width, int* pos) {
  const int64_t tot = (int64_t)P * nsl * 32;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / ((int64_t)nsl * 32), i = t - s * nsl * 32;  // i = q * 32 + lane
    const int row = i < m ? srow[s * m + i] : -1;
    if (row >= 0) pos[s * m + row] = (int)i;
    if ((i & 31) == 0) width[s * nsl + (i >> 5)] = i < m ? slen[s * m + i] : 0;
  }
}
__global__ void k_slab_fill(const int* ci, const double* val, int64_t m, int P, int nsl, const int* cb,
                            const int* cnt, const int* start, const int* pos, const int* sp, uint16_t* scol,
                            double* sval) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)P * m; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / m;
    const int i = pos[t];
    const int64_t base = (int64_t)sp[s * nsl + (i >> 5)] + (i & 31);
    const int k0 = start[t], c0 = cb[s];
    for (int k = 0; k < cnt[t]; ++k) {
      scol[base + 32 * k] = (uint16_t)(ci[k0 + k] - c0);
      sval[base + 32 * k] = val[k0 + k];
    }
  }
}

static int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 4096));
}

// The sliced-ELL tables of a PLAN_SELL orientation, from its CSR on the
// device (no-op for other plans): slice widths on the device, the offsets
// scanned on the host in 64 bits (a padded size past the int32 slot range
// falls back to the thread-per-row kernel), then the fill on the device.
static int build_sell(RowPlan& p, const int* rp, const int* ci, const double* val, int64_t rows, int sms, int dev,
                      cudaStream_t st, RowPlan* reuse = nullptr) {
  if (p.kind != PLAN_SELL) return 0;
  const int64_t nsl = (rows + 31) / 32;
  std::vector<int> w((size_t)nsl + 1);
  {
    Arena ar(st);
    int* w32;
    TS_CHECK(ar.get(&w32, (size_t)nsl + 1));
    k_sell_width<<<grid_for(nsl + 1), 256, 0, st>>>(rp, rows, nsl, w32);
    TS_CUDA(cudaGetLastError());
    TS_CUDA(d2h_pinned(w.data(), w32, ((size_t)nsl + 1) * sizeof(int), st));
  }
  int64_t total = 0;
  for (int64_t q = 0; q <= nsl; ++q) {
    const int64_t wq = w[q];
    w[q] = (int)std::min<int64_t>(total, INT32_MAX);
    total += wq;
  }
  if (total >= (int64_t)INT32_MAX) {  // slot offsets are int: keep the CSR kernel
    p.kind = PLAN_SHORT;
    p.P = (int)std::max<int64_t>(1, std::min<int64_t>((rows + kNT - 1) / kNT, resident_blocks(sms)));
    return 0;
  }
  const size_t slots = (size_t)std::max<int64_t>(total, 1);
  if (reuse && reuse->kind == PLAN_SELL && reuse->sell_slots == total && reuse->sell_sp) {
    // a recycled handle of the same shape and padded size: refill its tables
    // in place (no cudaMalloc / cudaFree: both synchronise the device and
    // would stall solves running on other streams)
    p.sell_sp = reuse->sell_sp;
    p.sell_ci = reuse->sell_ci;
    p.sell_val = reuse->sell_val;
    p.sell_borrowed = 1;
  } else if (dev_malloc(&p.sell_sp, ((size_t)nsl + 1) * sizeof(int), dev) != cudaSuccess ||
             dev_malloc(&p.sell_ci, slots * sizeof(int), dev) != cudaSuccess ||
             dev_malloc(&p.sell_val, slots * sizeof(double), dev) != cudaSuccess) {
    set_error("cudaMalloc for the sliced-ELL copy (%lld slots) failed", (long long)total);
    return TS_ENOMEM;
  }
  p.sell_slots = total;
  TS_CUDA(cudaMemcpyAsync(p.sell_sp, w.data(), ((size_t)nsl + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
  k_sell_fill<<<grid_for(nsl * 32), 256, 0, st>>>(rp, ci, val, rows, nsl, p.sell_sp, p.sell_ci, p.sell_val);
  TS_CUDA(cudaGetLastError());
  TS_CUDA(cudaStreamSynchronize(st));  // the host offsets leave scope
  return 0;
}

// The column-slab tables of a long-row CSR A v over a wide matrix (PLAN_SLAB,
// k_slab_av): P = #SM slabs of equal nnz (column boundaries from the CSC
// column pointers).  Kept only when it pays and fits: n >= 65536 (x beyond
// any L1), every slab <= kSlabMaxW columns, the per-(slab, row) partials at
// most a quarter of the matrix bytes, sorted row indices.  Otherwise `p`
// stays the row kernel's plan.
static int build_slab(RowPlan& p, const int* rp, const int* ci, const double* val, int64_t m, int64_t n,
                      int64_t nnz, const std::vector<int>& colptr, int sms, int dev, cudaStream_t st,
                      RowPlan* reuse = nullptr) {
  if (!(p.kind == PLAN_WROW || p.kind == PLAN_FLAT) || n < 65536 || m > (int64_t)INT32_MAX / 64) return 0;
  const int P = sms;
  if ((double)m * P * 16.0 > 0.25 * 12.0 * (double)nnz) return 0;
  std::vector<int> cb(P + 1);
  int maxw = 0;
  for (int s = 0; s <= P; ++s) {
    const int64_t target = nnz * s / P;
    cb[s] = s == 0 ? 0 : s == P ? (int)n
                   : (int)(std::lower_bound(colptr.begin(), colptr.end(), (int)target) - colptr.begin());
    if (s > 0) {
      cb[s] = std::max(cb[s], cb[s - 1]);
      maxw = std::max(maxw, cb[s] - cb[s - 1]);
    }
  }
  const int nsl = (int)((m + 31) / 32);
  if (maxw > kSlabMaxW || maxw < 1 || slab_smem(maxw, nsl) > (size_t)kSlabSmemMax) return 0;
  const int64_t Pm = (int64_t)P * m, Pn32 = (int64_t)P * nsl * 32;
  Arena ar(st);
  int *dcb, *cnt, *start, *unsorted, *rows_in, *offs, *slen, *srow, *width, *pos;
  TS_CHECK(ar.get(&dcb, P + 1));
  TS_CHECK(ar.get(&cnt, Pm));
  TS_CHECK(ar.get(&start, Pm));
  TS_CHECK(ar.get(&unsorted, 1));
  TS_CHECK(ar.get(&rows_in, Pm));
  TS_CHECK(ar.get(&offs, P + 1));
  TS_CHECK(ar.get(&slen, Pm));
  TS_CHECK(ar.get(&srow, Pm));
  TS_CHECK(ar.get(&width, (size_t)P * nsl));
  TS_CHECK(ar.get(&pos, Pm));
  TS_CUDA(cudaMemcpyAsync(dcb, cb.data(), (P + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
  TS_CUDA(cudaMemsetAsync(unsorted, 0, sizeof(int), st));
  k_slab_runs<<<grid_for(m), 256, 0, st>>>(rp, ci, m, dcb, P, cnt, start, unsorted);
  k_slab_iota<<<grid_for(Pm), 256, 0, st>>>(m, P, rows_in, offs);
  // rows of every slab by in-slab length, descending, stable
  int end_bit = 1;
  while (end_bit < 31 && (1ll << end_bit) <= (int64_t)nnz) ++end_bit;
  size_t tb = 0;
  cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, tb, cnt, slen, rows_in, srow, (int)Pm, P, offs,
                                                     offs + 1, 0, end_bit, st);
  char* tmp;
  TS_CHECK(ar.get(&tmp, std::max<size_t>(tb, 16)));
  if (cub::DeviceSegmentedRadixSort::SortPairsDescending(tmp, tb, cnt, slen, rows_in, srow, (int)Pm, P, offs,
                                                         offs + 1, 0, end_bit, st) != cudaSuccess) {
    set_error("segmented sort for the column-slab copy failed");
    return TS_ECUDA;
  }
  k_slab_tables<<<grid_for(Pn32), 256, 0, st>>>(slen, srow, m, P, nsl, width, pos);
  TS_CUDA(cudaGetLastError());
  std::vector<int> w((size_t)P * nsl);
  int hun = 0;
  TS_CUDA(d2h_pinned(w.data(), width, w.size() * sizeof(int), st));
  TS_CUDA(d2h_pinned(&hun, unsorted, sizeof(int), st));
  if (hun) return 0;  // unsorted column indices: keep the row kernel
  // slice offsets (64-bit scan) and the warp runs of every slab (equal slots)
  std::vector<int> sp((size_t)P * nsl + 1), wr((size_t)P * 33);
  int64_t tot = 0;
  for (int s = 0; s < P; ++s) {
    const int64_t s0 = tot;
    for (int q = 0; q < nsl; ++q) {
      sp[(size_t)s * nsl + q] = (int)std::min<int64_t>(tot, INT32_MAX);
      tot += 32ll * w[(size_t)s * nsl + q];
    }
    const int64_t stot = tot - s0;
    int64_t acc = 0;
    int q = 0;
    for (int ww = 0; ww <= 32; ++ww) {
      const int64_t target = stot * ww / 32;
      while (q < nsl && acc + 16ll * w[(size_t)s * nsl + q] < target) acc += 32ll * w[(size_t)s * nsl + q++];
      wr[(size_t)s * 33 + ww] = ww == 32 ? nsl : std::max(q, ww ? wr[(size_t)s * 33 + ww - 1] : 0);
    }
  }
  if (tot >= (int64_t)INT32_MAX) return 0;
  sp[(size_t)P * nsl] = (int)tot;
  // every warp run with its slot offset: one load instead of the wr -> sp chain
  std::vector<int2> wre((size_t)P * 33);
  for (int s = 0; s < P; ++s)
    for (int ww = 0; ww <= 32; ++ww) {
      const int q = wr[(size_t)s * 33 + ww];
      wre[(size_t)s * 33 + ww] = make_int2(q, sp[(size_t)s * nsl + q]);
    }
  const size_t slots = (size_t)std::max<int64_t>(tot, 1);
  if (reuse && reuse->kind == PLAN_SLAB && reuse->slab_slots == tot && reuse->P == P && reuse->slab_nsl == nsl &&
      reuse->slab_rows == m) {
    // a recycled handle of the same shape and size: refill its tables in place
    p.slab_cb = reuse->slab_cb;
    p.slab_sp = reuse->slab_sp;
    p.slab_wr = reuse->slab_wr;
    p.slab_pos = reuse->slab_pos;
    p.slab_col = reuse->slab_col;
    p.slab_val = reuse->slab_val;
    p.slab_borrowed = 1;
  } else if (dev_malloc(&p.slab_cb, (P + 1) * sizeof(int), dev) != cudaSuccess ||
             dev_malloc(&p.slab_sp, sp.size() * sizeof(int), dev) != cudaSuccess ||
             dev_malloc(&p.slab_wr, wre.size() * sizeof(int2), dev) != cudaSuccess ||
             dev_malloc(&p.slab_pos, Pm * sizeof(int), dev) != cudaSuccess ||
             dev_malloc(&p.slab_col, slots * sizeof(uint16_t), dev) != cudaSuccess ||
             dev_malloc(&p.slab_val, slots * sizeof(double), dev) != cudaSuccess) {
    set_error("cudaMalloc for the column-slab copy (%lld slots) failed", (long long)tot);
    return TS_ENOMEM;
  }
  TS_CUDA(cudaMemcpyAsync(p.slab_cb, cb.data(), (P + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
  TS_CUDA(cudaMemcpyAsync(p.slab_sp, sp.data(), sp.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  TS_CUDA(cudaMemcpyAsync(p.slab_wr, wre.data(), wre.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  TS_CUDA(cudaMemcpyAsync(p.slab_pos, pos, Pm * sizeof(int), cudaMemcpyDeviceToDevice, st));
  TS_CUDA(cudaMemsetAsync(p.slab_col, 0xFF, slots * sizeof(uint16_t), st));  // padding: kSlabPad
  TS_CUDA(cudaMemsetAsync(p.slab_val, 0, slots * sizeof(double), st));
  k_slab_fill<<<grid_for(Pm), 256, 0, st>>>(ci, val, m, P, nsl, p.slab_cb, cnt, start, pos, p.slab_sp,
                                            p.slab_col, p.slab_val);
  TS_CUDA(cudaGetLastError());
  TS_CUDA(cudaStreamSynchronize(st));  // the host tables leave scope
  p.kind = PLAN_SLAB;
  p.P = P;
  p.slab_nsl = nsl;
  p.slab_rows = m;
  p.slab_maxw = maxw;
  p.slab_slots = tot;
  return 0;
}
}  // namespace ts

using namespace ts;

struct ts_matrix : public ts::Mat {};

namespace ts {
static void free_matrix(Mat* A) {
  DeviceGuard g(A->dev);
  cudaDeviceSynchronize();
  destroy_instances(A);
  void* ps[] = {A->a,   A->aT,  A->rp,  A->ci,  A->val, A->rpT, A->ciT, A->valT,
                nullptr};
  for (void* p : ps)
    if (p) cudaFree(p);
  free_plan(A->planN);
  free_plan(A->planT);
  delete static_cast<ts_matrix*>(A);
}
}  // namespace ts

// ======================================================================= ABI
extern "C" {

int ts_abi_version(void) { return TS_ABI_VERSION; }
const char* ts_last_error(void) { return ts::last_error(); }
int ts_device_count(int* count) {
  TS_CUDA(cudaGetDeviceCount(count));
  return 0;
}


// A fully built, unsharded, non-column-tiled handle is retired into the
// storage pool (see retire_take); everything else is freed.
static int matrix_release(ts_matrix* A, bool complete) {
  StructShared structural;
  if (!A) return 0;
  if (complete && matrix_pool_enabled() && !A->comm && A->halo == 0) {
    {
      DeviceGuard g(A->dev);
      cudaDeviceSynchronize();  // no solve may still read the storage
    }
    Mat* evict = nullptr;
    {
      std::lock_guard<std::mutex> g(g_retire_mu);
      g_retired.push_back(A);
      if (g_retired.size() > kRetireMax) {
        evict = g_retired.front();
        g_retired.erase(g_retired.begin());
      }
    }
    if (evict) free_matrix(evict);
    return 0;
  }
  free_matrix(A);
  return 0;
}

int ts_matrix_destroy(ts_matrix* A) { return matrix_release(A, true); }

int ts_pool_trim(int device) {
  StructShared structural;
  pool_trim_device(device);
  std::vector<std::pair<size_t, void*>> drop;
  {
    std::lock_guard<std::mutex> g(g_host_mu);
    drop.swap(g_host_free);
    g_host_cached = 0;
  }
  for (auto& kv : drop) cudaFreeHost(static_cast<char*>(kv.second) - 64);
  return 0;
}

int ts_host_alloc(size_t bytes, void** out) {
  StructShared structural;
  if (!out) TS_INVAL("null output pointer");
  *out = nullptr;
  bytes = std::max<size_t>(bytes, 64);
  {
    std::lock_guard<std::mutex> g(g_host_mu);
    for (size_t i = g_host_free.size(); i-- > 0;)  // most recently freed first
      if (g_host_free[i].first == bytes) {
        *out = g_host_free[i].second;
        g_host_cached -= bytes;
        g_host_free.erase(g_host_free.begin() + i);
        return 0;
      }
  }
  // pinned blocks carry their size in a 64-byte header
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, bytes + 64, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    set_error("cudaHostAlloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    return TS_ENOMEM;
  }
  *reinterpret_cast<size_t*>(p) = bytes;
  *out = static_cast<char*>(p) + 64;
  return 0;
}

int ts_host_free(void* ptr) {
  StructShared structural;
  if (!ptr) return 0;
  void* base = static_cast<char*>(ptr) - 64;
  const size_t bytes = *reinterpret_cast<size_t*>(base);
  {
    std::lock_guard<std::mutex> g(g_host_mu);
    if (g_host_cached + bytes <= kHostCacheMax) {
      g_host_free.emplace_back(bytes, ptr);
      g_host_cached += bytes;
      return 0;
    }
  }
  cudaFreeHost(base);
  return 0;
}

int ts_matrix_plans(const ts_matrix* A, int32_t* plan_av, int32_t* plan_atv) {
  if (!A) TS_INVAL("null matrix handle");
  if (plan_av) *plan_av = A->planN.kind;
  if (plan_atv) *plan_atv = A->planT.kind;
  return 0;
}

int ts_matrix_info(const ts_matrix* A, int64_t* m, int64_t* n, int64_t* nnz, int32_t* kind,
                   double* fro) {
  if (!A) TS_INVAL("null matrix handle");
  if (m) *m = A->m;
  if (n) *n = A->n;
  if (nnz) *nnz = A->nnz;
  if (kind) *kind = A->kind;
  if (fro) *fro = A->fro;
  return 0;
}

static int finish_create(ts_matrix* A, cudaStream_t st, Arena& ar) {
  if (A->kind == 0 && A->aT) {  // PLAN_TRANS: the transposed copy of the new entries
    dim3 grid((unsigned)((A->n + 31) / 32), (unsigned)((A->m + 31) / 32));
    k_transpose<<<grid, dim3(32, 8), 0, st>>>(A->a, A->lda, A->m, A->n, A->aT, A->ldaT);
    TS_CUDA(cudaGetLastError());
  }
  // Frobenius norm once (linalg.py:64-69); cached on the immutable handle
  Work wk;
  TS_CHECK(make_work(ar, work_blocks(A->sms), &wk, A->npart));
  double* dfro;
  TS_CHECK(ar.get(&dfro, 1));
  if (A->kind == 0) {
    EpiFroDense e{A->a, A->lda, A->n, dfro};
    TS_CHECK(launch_vec(A->m * A->n, A->sms, e, wk, st));
  } else {
    EpiFroVals e{A->val, dfro};
    TS_CHECK(launch_vec(A->nnz, A->sms, e, wk, st));
  }
  // read back through pinned memory: a device->pageable copy is synchronous in
  // the driver and stalled concurrent solves on other streams
  static thread_local double* hfro = nullptr;
  if (!hfro) TS_CUDA(cudaHostAlloc(&hfro, sizeof(double), cudaHostAllocDefault));
  TS_CUDA(cudaMemcpyAsync(hfro, dfro, sizeof(double), cudaMemcpyDeviceToHost, st));
  TS_CUDA(cudaStreamSynchronize(st));
  A->fro = *hfro;
  return 0;
}

int ts_matrix_create_dense(const double* a, int64_t m, int64_t n, int64_t lda, int device,
                           void* stream, ts_matrix** out) {
  StructShared structural;
  if (!out) TS_INVAL("null output handle");
  *out = nullptr;
  if (m < 1 || n < 1) TS_INVAL("matrix must have at least one row and one column (got %lld x %lld)",
                               (long long)m, (long long)n);
  if (lda < n) TS_INVAL("lda (%lld) < n (%lld)", (long long)lda, (long long)n);
  if (!a) TS_INVAL("null matrix data");
  DeviceGuard g(device);
  setup_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  if (ts_matrix* R = static_cast<ts_matrix*>(retire_take(device, 0, m, n, m * n))) {
    // same shape: plans, instances and graphs stay valid; new entries only
    int rc = 0;
    {
      Arena ar(st);
      cudaError_t e = upload_rows(R->a, R->lda, a, lda, m, n, st);
      if (e != cudaSuccess) {
        set_error("dense upload failed: %s", cudaGetErrorString(e));
        rc = TS_ECUDA;
      }
      if (!rc) rc = finish_create(R, st, ar);
    }
    if (rc) {
      matrix_release(R, false);
      return rc;
    }
    *out = R;
    return 0;
  }
  ts_matrix* A = new ts_matrix();
  A->dev = device;
  A->sms = sm_count(device);
  A->kind = 0;
  A->m = m;
  A->n = n;
  A->nnz = m * n;
  A->lda = n >= 64 ? (n + 15) / 16 * 16 : (n + 3) / 4 * 4;
  int rc = 0;
  {
    Arena ar(st);
    cudaError_t e = dev_malloc(&A->a, (size_t)A->lda * m * sizeof(double), device);
    if (e != cudaSuccess) {
      set_error("cudaMalloc(dense %lld x %lld) failed: %s", (long long)m, (long long)A->lda,
                cudaGetErrorString(e));
      rc = TS_ENOMEM;
    }
    if (!rc && A->lda != n) e = cudaMemsetAsync(A->a, 0, (size_t)A->lda * m * sizeof(double), st);
    if (!rc && e == cudaSuccess) e = upload_rows(A->a, A->lda, a, lda, m, n, st);
    if (!rc && e != cudaSuccess) {
      set_error("dense upload failed: %s", cudaGetErrorString(e));
      rc = TS_ECUDA;
    }
    A->npart = npart_elems(m, n);
    if (!rc) rc = plan_rows_dense(m, n, A->sms, &A->planN, st);
    if (!rc) {
      A->planT.kind = PLAN_TILE;
      A->planT.P = tile_grid(m, n, A->sms, kTileTBlocks, kTileMinRowsT);
      // small dense A (<= kTransBytes, L2-sized): A^T v as the fused row-tile
      // kernel over a transposed copy (C1: 7.3 vs 9.4 us per pass: no split-
      // tile merges); TS_DENSE_T=cols keeps the column-tile kernel
      const char* te = getenv("TS_DENSE_T");
      if (m >= 128 && n >= 128 && 8 * m * n <= kTransBytes && !(te && !strcmp(te, "cols"))) {
        A->ldaT = m >= 64 ? (m + 15) / 16 * 16 : (m + 3) / 4 * 4;
        if (dev_malloc(&A->aT, (size_t)A->ldaT * n * sizeof(double), device) != cudaSuccess) {
          set_error("cudaMalloc(transposed dense %lld x %lld) failed", (long long)n, (long long)m);
          rc = TS_ENOMEM;
        } else {
          if (A->ldaT != m) cudaMemsetAsync(A->aT, 0, (size_t)A->ldaT * n * sizeof(double), st);
          A->planT.kind = PLAN_TRANS;
          A->planT.P = tile_grid(n, m, A->sms, kTileNBlocks);
          const char* se = getenv("TS_DENSE_SMALL");
          if (wdense_fits(n, m) && !(se && !strcmp(se, "tile"))) {
            A->planT.wdense = 1;
            A->planT.P = wdense_grid(n, A->sms);
          }
          A->npart = npart_elems(m, n) + npart_elems(n, m);  // disjoint A v / A^T v layouts
        }
      }
      // HBM-sized dense A: a transposed copy for A v on the column-tile kernel
      // (TS_DENSE_AV=rows keeps the row-tile kernel and saves the copy)
      const char* ae = getenv("TS_DENSE_AV");
      if (!rc && !A->aT && m >= 1024 && n >= 1024 && 8 * m * n >= kNcolsBytes && A->planN.kind == PLAN_TILE &&
          !A->planN.wdense && !(ae && !strcmp(ae, "rows"))) {
        A->ldaT = (m + 15) / 16 * 16;
        if (dev_malloc(&A->aT, (size_t)A->ldaT * n * sizeof(double), device) == cudaSuccess) {
          if (A->ldaT != m) cudaMemsetAsync(A->aT, 0, (size_t)A->ldaT * n * sizeof(double), st);
          A->planN.kind = PLAN_NCOLS;
          A->planN.P = tile_grid(n, m, A->sms, kTileTBlocks, kTileMinRowsT);
        } else {
          cudaGetLastError();  // no room for the copy: the row-tile kernel stays
          A->aT = nullptr;
        }
      }
    }
    if (!rc) rc = finish_create(A, st, ar);
  }
  if (rc) {
    matrix_release(A, false);
    return rc;
  }
  *out = A;
  return 0;
}

int ts_matrix_create_csr(const int32_t* indptr, const int32_t* indices, const double* data,
                         int64_t m, int64_t n, int64_t nnz, int device, void* stream,
                         ts_matrix** out) {
  StructShared structural;
  if (!out) TS_INVAL("null output handle");
  *out = nullptr;
  if (m < 1 || n < 1) TS_INVAL("matrix must have at least one row and one column (got %lld x %lld)",
                               (long long)m, (long long)n);
  if (nnz < 0 || nnz >= (int64_t)INT32_MAX) TS_INVAL("nnz %lld outside the int32 index range", (long long)nnz);
  if (!indptr || (nnz > 0 && (!indices || !data))) TS_INVAL("null CSR array");
  DeviceGuard g(device);
  setup_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  // host copy of the row pointer for validation and planning
  std::vector<int> rp_h((size_t)m + 1);
  TS_CUDA(d2h_pinned(rp_h.data(), indptr, (m + 1) * sizeof(int), st));
  if (rp_h[0] != 0 || rp_h[m] != nnz) TS_INVAL("CSR indptr must start at 0 and end at nnz");
  for (int64_t r = 0; r < m; ++r)
    if (rp_h[r + 1] < rp_h[r]) TS_INVAL("CSR indptr is not nondecreasing at row %lld", (long long)r);

  ts_matrix* A = static_cast<ts_matrix*>(retire_take(device, 1, m, n, nnz));
  const bool reuse = A != nullptr;  // same shape: storage, plans and instances recycled
  if (!A) A = new ts_matrix();
  A->dev = device;
  A->sms = sm_count(device);
  A->kind = 1;
  A->m = m;
  A->n = n;
  A->nnz = nnz;
  int rc = 0;
  auto fail = [&](int code) {
    matrix_release(A, false);
    return code;
  };
  {
    Arena ar(st);
    const size_t nz = (size_t)std::max<int64_t>(nnz, 1);
    // +16 B tails: k_rows_stream's bulk copies round their ranges to 16 bytes
    if (!reuse && (dev_malloc(&A->rp, (m + 1 + 4) * sizeof(int), device) != cudaSuccess ||
                   dev_malloc(&A->ci, (nz + 4) * sizeof(int), device) != cudaSuccess ||
                   dev_malloc(&A->val, (nz + 2) * sizeof(double), device) != cudaSuccess ||
                   dev_malloc(&A->rpT, (n + 1 + 4) * sizeof(int), device) != cudaSuccess ||
                   dev_malloc(&A->ciT, (nz + 4) * sizeof(int), device) != cudaSuccess ||
                   dev_malloc(&A->valT, (nz + 2) * sizeof(double), device) != cudaSuccess)) {
      set_error("cudaMalloc for CSR storage failed (nnz=%lld)", (long long)nnz);
      return fail(TS_ENOMEM);
    }
    if (cudaMemcpyAsync(A->rp, rp_h.data(), (m + 1) * sizeof(int), cudaMemcpyHostToDevice, st) ||
        (nnz && cudaMemcpyAsync(A->ci, indices, nnz * sizeof(int), cudaMemcpyDefault, st)) ||
        (nnz && cudaMemcpyAsync(A->val, data, nnz * sizeof(double), cudaMemcpyDefault, st))) {
      set_error("CSR upload failed");
      return fail(TS_ECUDA);
    }
    int* dband = nullptr;
    if (nnz > 0) {
      // validate column indices on the device
      Work wk;
      if ((rc = make_work(ar, work_blocks(A->sms), &wk))) return fail(rc);
      double* rng;
      if ((rc = ar.get(&rng, 2))) return fail(rc);
      EpiIdxRange er{A->ci, rng};
      if ((rc = launch_vec(nnz, A->sms, er, wk, st))) return fail(rc);
      double hr[2] = {0.0, 0.0};
      if (d2h_pinned(hr, rng, sizeof(hr), st) != cudaSuccess) {
        set_error("CSR index range read-back failed: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(TS_ECUDA);
      }
      if (hr[0] < 0 || hr[1] >= (double)n) {
        set_error("CSR column index out of range [0, %lld)", (long long)n);
        return fail(TS_EINVAL);
      }
      // transposed CSR: stable radix sort of (column, position)
      int *rowid, *keys_out, *perm_in, *perm_out;
      if ((rc = ar.get(&rowid, nz)) || (rc = ar.get(&keys_out, nz)) || (rc = ar.get(&perm_in, nz)) ||
          (rc = ar.get(&perm_out, nz)))
        return fail(rc);
      k_expand_rows<<<grid_for(m), 256, 0, st>>>(A->rp, m, rowid);
      if ((rc = ar.get(&dband, 1))) return fail(rc);
      cudaMemsetAsync(dband, 0, sizeof(int), st);
      k_csr_band<<<grid_for(nnz), 256, 0, st>>>(rowid, A->ci, nnz, dband);
      k_iota<<<grid_for(nnz), 256, 0, st>>>(perm_in, nnz);
      int end_bit = 1;
      while (end_bit < 31 && ((int64_t)1 << end_bit) < n) ++end_bit;
      size_t tmp_bytes = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, A->ci, keys_out, perm_in, perm_out,
                                      (int)nnz, 0, end_bit, st);
      void* tmp;
      if ((rc = ar.get((char**)&tmp, tmp_bytes))) return fail(rc);
      if (cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, A->ci, keys_out, perm_in, perm_out,
                                          (int)nnz, 0, end_bit, st) != cudaSuccess) {
        set_error("radix sort for the transposed CSR failed");
        return fail(TS_ECUDA);
      }
      k_gather_T<<<grid_for(nnz), 256, 0, st>>>(perm_out, rowid, A->val, A->ciT, A->valT, nnz);
      k_rowptr_from_keys<<<grid_for(nnz + 1), 256, 0, st>>>(keys_out, nnz, n, A->rpT);
    } else {
      cudaMemsetAsync(A->rpT, 0, (n + 1) * sizeof(int), st);
    }
    if (cudaGetLastError() != cudaSuccess) {
      set_error("CSR transpose kernels failed");
      return fail(TS_ECUDA);
    }
    std::vector<int> rpT_h((size_t)n + 1);
    if (d2h_pinned(rpT_h.data(), A->rpT, (n + 1) * sizeof(int), st) != cudaSuccess) {
      set_error("CSR transpose failed: %s", cudaGetErrorString(cudaGetLastError()));
      return fail(TS_ECUDA);
    }
    A->band = -1;
    if (dband) {
      int hb = 0;
      if (d2h_pinned(&hb, dband, sizeof(int), st) == cudaSuccess) A->band = hb;
    } else if (nnz == 0) {
      A->band = 0;
    }
    {
      RowPlan pN, pT;
      if ((rc = plan_rows_csr(rp_h.data(), m, nnz, A->sms, &pN, st))) return fail(rc);
      if ((rc = plan_rows_csr(rpT_h.data(), n, nnz, A->sms, &pT, st))) {
        free_plan(pN);
        return fail(rc);
      }
      if ((rc = build_sell(pN, A->rp, A->ci, A->val, m, A->sms, device, st, reuse ? &A->planN : nullptr)) ||
          (rc = build_sell(pT, A->rpT, A->ciT, A->valT, n, A->sms, device, st, reuse ? &A->planT : nullptr)) ||
          (rc = build_slab(pN, A->rp, A->ci, A->val, m, n, nnz, rpT_h, A->sms, device, st,
                           reuse ? &A->planN : nullptr))) {
        free_plan(pN);
        free_plan(pT);
        return fail(rc);
      }
      const bool keepN = adopt_plan(A->planN, pN, m, st);
      const bool keepT = adopt_plan(A->planT, pT, n, st);
      A->npart = A->planN.kind == PLAN_SLAB ? (int64_t)A->planN.P * m : 0;  // the slab partials
      // a recycled handle's instances bake the old launch geometry
      if (reuse && !(keepN && keepT)) destroy_instances(A);
    }
    if (nnz > 0) {
      if ((rc = finish_create(A, st, ar))) return fail(rc);
    } else {
      A->fro = 0.0;
    }
  }
  *out = A;
  return 0;
}

// A row block of a square matrix with both orientations given by the caller
// (the rank's rows of A and the rank's columns of A as rows of A^T), column /
// row indices local to the block and reaching `halo` entries past either end.
int ts_matrix_create_csr_pair(const int32_t* indptr, const int32_t* indices, const double* data,
                              int64_t nnz, const int32_t* indptr_t, const int32_t* indices_t,
                              const double* data_t, int64_t nnz_t, int64_t m, int64_t halo,
                              int device, void* stream, ts_matrix** out) {
  StructShared structural;
  if (!out) TS_INVAL("null output handle");
  *out = nullptr;
  if (m < 1) TS_INVAL("row block must have at least one row");
  if (halo < 0 || halo > m) TS_INVAL("halo %lld outside 0..%lld", (long long)halo, (long long)m);
  if (nnz < 0 || nnz >= (int64_t)INT32_MAX || nnz_t < 0 || nnz_t >= (int64_t)INT32_MAX)
    TS_INVAL("nnz outside the int32 index range");
  if (!indptr || !indptr_t || (nnz && (!indices || !data)) || (nnz_t && (!indices_t || !data_t)))
    TS_INVAL("null CSR array");
  DeviceGuard g(device);
  setup_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> rp_h((size_t)m + 1), rpT_h((size_t)m + 1);
  TS_CUDA(cudaMemcpyAsync(rp_h.data(), indptr, (m + 1) * sizeof(int), cudaMemcpyDefault, st));
  TS_CUDA(cudaMemcpyAsync(rpT_h.data(), indptr_t, (m + 1) * sizeof(int), cudaMemcpyDefault, st));
  TS_CUDA(cudaStreamSynchronize(st));
  if (rp_h[0] != 0 || rp_h[m] != nnz || rpT_h[0] != 0 || rpT_h[m] != nnz_t)
    TS_INVAL("CSR indptr must start at 0 and end at nnz");
  for (int64_t r = 0; r < m; ++r)
    if (rp_h[r + 1] < rp_h[r] || rpT_h[r + 1] < rpT_h[r])
      TS_INVAL("CSR indptr is not nondecreasing at row %lld", (long long)r);
  ts_matrix* A = new ts_matrix();
  A->dev = device;
  A->sms = sm_count(device);
  A->kind = 1;
  A->m = m;
  A->n = m;
  A->nnz = nnz;
  A->halo = halo;
  int rc = 0;
  auto fail = [&](int code) {
    matrix_release(A, false);
    return code;
  };
  {
    Arena ar(st);
    const size_t nz = (size_t)std::max<int64_t>(nnz, 1), nzt = (size_t)std::max<int64_t>(nnz_t, 1);
    if (dev_malloc(&A->rp, (m + 1 + 4) * sizeof(int), device) != cudaSuccess ||
        dev_malloc(&A->ci, (nz + 4) * sizeof(int), device) != cudaSuccess ||
        dev_malloc(&A->val, (nz + 2) * sizeof(double), device) != cudaSuccess ||
        dev_malloc(&A->rpT, (m + 1 + 4) * sizeof(int), device) != cudaSuccess ||
        dev_malloc(&A->ciT, (nzt + 4) * sizeof(int), device) != cudaSuccess ||
        dev_malloc(&A->valT, (nzt + 2) * sizeof(double), device) != cudaSuccess) {
      set_error("cudaMalloc for the row-block CSR failed");
      return fail(TS_ENOMEM);
    }
    if (cudaMemcpyAsync(A->rp, rp_h.data(), (m + 1) * sizeof(int), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(A->rpT, rpT_h.data(), (m + 1) * sizeof(int), cudaMemcpyHostToDevice, st) ||
        (nnz && cudaMemcpyAsync(A->ci, indices, nnz * sizeof(int), cudaMemcpyDefault, st)) ||
        (nnz && cudaMemcpyAsync(A->val, data, nnz * sizeof(double), cudaMemcpyDefault, st)) ||
        (nnz_t && cudaMemcpyAsync(A->ciT, indices_t, nnz_t * sizeof(int), cudaMemcpyDefault, st)) ||
        (nnz_t && cudaMemcpyAsync(A->valT, data_t, nnz_t * sizeof(double), cudaMemcpyDefault, st))) {
      set_error("row-block CSR upload failed");
      return fail(TS_ECUDA);
    }
    // local indices must stay inside [-halo, m + halo)
    Work wk;
    double* rng;
    if ((rc = make_work(ar, work_blocks(A->sms), &wk)) || (rc = ar.get(&rng, 2))) return fail(rc);
    double hr[4] = {0, 0, 0, 0};
    if (nnz) {
      EpiIdxRange er{A->ci, rng};
      if ((rc = launch_vec(nnz, A->sms, er, wk, st))) return fail(rc);
      cudaMemcpyAsync(hr, rng, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    }
    if (nnz_t) {
      EpiIdxRange er{A->ciT, rng};
      if ((rc = launch_vec(nnz_t, A->sms, er, wk, st))) return fail(rc);
      cudaMemcpyAsync(hr + 2, rng, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    }
    if ((nnz && (hr[0] < -(double)halo || hr[1] >= (double)(m + halo))) ||
        (nnz_t && (hr[2] < -(double)halo || hr[3] >= (double)(m + halo)))) {
      set_error("row-block index outside [-%lld, %lld)", (long long)halo, (long long)(m + halo));
      return fail(TS_EINVAL);
    }
    RowPlan pN, pT;
    if ((rc = plan_rows_csr(rp_h.data(), m, nnz, A->sms, &pN, st))) return fail(rc);
    if ((rc = plan_rows_csr(rpT_h.data(), m, nnz_t, A->sms, &pT, st))) {
      free_plan(pN);
      return fail(rc);
    }
    if ((rc = build_sell(pN, A->rp, A->ci, A->val, m, A->sms, device, st)) ||
        (rc = build_sell(pT, A->rpT, A->ciT, A->valT, m, A->sms, device, st))) {
      free_plan(pN);
      free_plan(pT);
      return fail(rc);
    }
    adopt_plan(A->planN, pN, m, st);
    adopt_plan(A->planT, pT, m, st);
    if (nnz > 0) {
      if ((rc = finish_create(A, st, ar))) return fail(rc);
    } else {
      A->fro = 0.0;
    }
  }
  *out = A;
  return 0;
}

// ------------------------------------------------------ device gallery ----
// Deterministic sparse families generated straight into device CSR
// (reference gallery.py:64-71, 118-191); the coefficients arrive computed on
// the host with the reference's own expressions, so values are bit-identical.
namespace ts {
__global__ void k_stencil5_count(int64_t g, int* cnt) {
  const int64_t n = g * g;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ix = k % g, iy = k / g;
    cnt[k] = 1 + (ix > 0) + (ix < g - 1) + (iy > 0) + (iy < g - 1);
  }
}
// entries in ascending column order: south, west, centre, east, north
__global__ void k_stencil5_fill(int64_t g, double c, double w, double e, double s, double nn, int mode,
                                const int* rp, int* ci, double* val) {
  const int64_t n = g * g;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ix = k % g, iy = k / g;
    int q = rp[k];
    const int nb = (ix > 0) + (ix < g - 1) + (iy > 0) + (iy < g - 1);
    if (iy > 0) { ci[q] = (int)(k - g); val[q++] = s; }
    if (ix > 0) { ci[q] = (int)(k - 1); val[q++] = w; }
    ci[q] = (int)k;
    val[q++] = mode ? (double)nb : c;
    if (ix < g - 1) { ci[q] = (int)(k + 1); val[q++] = e; }
    if (iy < g - 1) { ci[q] = (int)(k + g); val[q++] = nn; }
  }
}
// Clement: A[i, i-1] = sqrt(i (n - i)), A[i, i+1] = sqrt((i + 1) (n - i - 1))
__global__ void k_clement_fill(int64_t n, int* rp, int* ci, double* val) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    rp[i] = (int)(i == 0 ? 0 : (i == n ? 2 * n - 2 : 2 * i - 1));
    if (i == n) continue;
    int q = i == 0 ? 0 : (int)(2 * i - 1);
    if (i > 0) {
      const double k = (double)i;
      ci[q] = (int)(i - 1);
      val[q++] = sqrt(__dmul_rn(k, __dsub_rn((double)n, k)));
    }
    if (i < n - 1) {
      const double k = (double)(i + 1);
      ci[q] = (int)(i + 1);
      val[q] = sqrt(__dmul_rn(k, __dsub_rn((double)n, k)));
    }
  }
}
}  // namespace ts

int ts_matrix_gen_stencil5(int64_t grid, double center, double west, double east, double south,
                           double north, int32_t center_mode, int device, void* stream, ts_matrix** out) {
  StructShared structural;
  if (!out) TS_INVAL("null output handle");
  *out = nullptr;
  if (grid < 2) TS_INVAL("grid must be at least 2");
  const int64_t n = grid * grid, nnz = 5 * n - 4 * grid;
  if (nnz >= (int64_t)INT32_MAX) TS_INVAL("nnz outside the int32 index range");
  DeviceGuard g(device);
  setup_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = 0;
  {
    Arena ar(st);
    int *cnt, *rp, *ci;
    double* val;
    if ((rc = ar.get(&cnt, n + 1)) || (rc = ar.get(&rp, n + 1)) || (rc = ar.get(&ci, nnz)) ||
        (rc = ar.get(&val, nnz)))
      return rc;
    TS_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(int), st));
    k_stencil5_count<<<grid_for(n), 256, 0, st>>>(grid, cnt);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, rp, (int)(n + 1), st);
    char* tmp;
    if ((rc = ar.get(&tmp, std::max<size_t>(tb, 16)))) return rc;
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, rp, (int)(n + 1), st);
    k_stencil5_fill<<<grid_for(n), 256, 0, st>>>(grid, center, west, east, south, north, center_mode,
                                                  rp, ci, val);
    TS_CUDA(cudaGetLastError());
    rc = ts_matrix_create_csr(rp, ci, val, n, n, nnz, device, stream, out);
  }
  return rc;
}

int ts_matrix_gen_clement(int64_t n, int device, void* stream, ts_matrix** out) {
  StructShared structural;
  if (!out) TS_INVAL("null output handle");
  *out = nullptr;
  if (n < 2) TS_INVAL("n must be at least 2");
  const int64_t nnz = 2 * n - 2;
  if (nnz >= (int64_t)INT32_MAX) TS_INVAL("nnz outside the int32 index range");
  DeviceGuard g(device);
  setup_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = 0;
  {
    Arena ar(st);
    int *rp, *ci;
    double* val;
    if ((rc = ar.get(&rp, n + 1)) || (rc = ar.get(&ci, nnz)) || (rc = ar.get(&val, nnz))) return rc;
    k_clement_fill<<<grid_for(n + 1), 256, 0, st>>>(n, rp, ci, val);
    TS_CUDA(cudaGetLastError());
    rc = ts_matrix_create_csr(rp, ci, val, n, n, nnz, device, stream, out);
  }
  return rc;
}

// ---------------------------------------------------------- Matrix Market
struct ts_mm : public ts::MmParsed {};

int ts_mm_parse(const char* data, int64_t len, int32_t is_path, ts_mm** out, ts_mm_info* info) {
  if (!out || !data) TS_INVAL("null argument");
  *out = nullptr;
  std::vector<char> buf;
  const char* p = data;
  size_t n = (size_t)std::max<int64_t>(len, 0);
  if (is_path) {
    FILE* fh = fopen(data, "rb");
    if (!fh) TS_INVAL("cannot open %s", data);
    fseek(fh, 0, SEEK_END);
    const long sz = ftell(fh);
    fseek(fh, 0, SEEK_SET);
    buf.resize((size_t)std::max(sz, 0L));
    const size_t got = sz > 0 ? fread(buf.data(), 1, (size_t)sz, fh) : 0;
    fclose(fh);
    p = buf.data();
    n = got;
  }
  ts_mm* P = new ts_mm();
  const int rc = ts::mm_parse(p, n, P);
  if (rc) {
    delete P;
    return rc;
  }
  if (info) {
    info->format = P->fmt;
    info->field = P->field;
    info->symmetry = P->sym;
    info->rows = P->m;
    info->cols = P->n;
    info->entries = P->entries;
    info->stored = P->fmt == 0 ? ts::mm_expanded_count(*P) : (int64_t)P->vals.size();
  }
  *out = P;
  return 0;
}

int ts_mm_coo(const ts_mm* P, int32_t* rows, int32_t* cols, double* vals) {
  if (!P || P->fmt != 0) TS_INVAL("not a coordinate Matrix Market object");
  int64_t c = 0;
  for (size_t k = 0; k < P->ri.size(); ++k) {
    rows[c] = P->ri[k];
    cols[c] = P->ci[k];
    vals[c] = P->v[k];
    ++c;
    if (P->sym != 0 && P->ri[k] != P->ci[k]) {
      rows[c] = P->ci[k];
      cols[c] = P->ri[k];
      vals[c] = P->sym == 2 ? -P->v[k] : P->v[k];
      ++c;
    }
  }
  return 0;
}

int ts_mm_dense(const ts_mm* P, double* a) {
  if (!P || P->fmt != 1) TS_INVAL("not an array Matrix Market object");
  const int64_t m = P->m, n = P->n;
  std::fill(a, a + m * n, 0.0);
  int64_t k = 0;
  for (int64_t j = 0; j < n; ++j) {  // column-major per the exchange format (mmio.py:142-155)
    const int64_t i0 = P->sym == 0 ? 0 : (P->sym == 1 ? j : j + 1);
    for (int64_t i = i0; i < m; ++i) {
      const double v = P->vals[k++];
      a[i * n + j] = v;
      if (P->sym == 1 && i != j) a[j * n + i] = v;
      else if (P->sym == 2) a[j * n + i] = -v;
    }
  }
  return 0;
}

int ts_mm_free(ts_mm* P) {
  delete P;
  return 0;
}

// Coordinate file -> device CSR handle: triplets uploaded once, mirrored,
// sorted, de-duplicated and compressed on the device.
int ts_mm_to_device(const ts_mm* P, int device, void* stream, ts_matrix** out, int64_t* duplicates) {
  StructShared structural;
  if (!P || !out) TS_INVAL("null argument");
  *out = nullptr;
  if (P->fmt != 0) TS_INVAL("array files are dense: build them with ts_matrix_create_dense");
  DeviceGuard g(device);
  setup_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ne = (int64_t)P->ri.size(), m = P->m, n = P->n;
  std::vector<int64_t> off((size_t)ne + 1);
  off[0] = 0;
  for (int64_t k = 0; k < ne; ++k) off[k + 1] = off[k] + ((P->sym != 0 && P->ri[k] != P->ci[k]) ? 2 : 1);
  const int64_t cnt = off[ne];
  if (cnt >= (int64_t)INT32_MAX) TS_INVAL("nnz %lld outside the int32 index range", (long long)cnt);
  int rc = 0;
  ts_matrix* A = nullptr;
  int64_t uniq = 0;
  {
    Arena ar(st);
    const size_t c1 = (size_t)std::max<int64_t>(cnt, 1), e1 = (size_t)std::max<int64_t>(ne, 1);
    int32_t *dri, *dci;
    double *dv, *val, *vout;
    int64_t *doff, *pos, *perm;
    unsigned long long *key, *key_s;
    int *head, *uidx, *rowcnt, *rp, *ciout;
    if ((rc = ar.get(&dri, e1)) || (rc = ar.get(&dci, e1)) || (rc = ar.get(&dv, e1)) ||
        (rc = ar.get(&doff, e1 + 1)) || (rc = ar.get(&key, c1)) || (rc = ar.get(&key_s, c1)) ||
        (rc = ar.get(&pos, c1)) || (rc = ar.get(&perm, c1)) || (rc = ar.get(&val, c1)) ||
        (rc = ar.get(&head, c1)) || (rc = ar.get(&uidx, c1)) || (rc = ar.get(&vout, c1)) ||
        (rc = ar.get(&ciout, c1)) || (rc = ar.get(&rowcnt, (size_t)m + 1)) || (rc = ar.get(&rp, (size_t)m + 1)))
      return rc;
    if (ne) {
      TS_CUDA(cudaMemcpyAsync(dri, P->ri.data(), ne * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      TS_CUDA(cudaMemcpyAsync(dci, P->ci.data(), ne * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      TS_CUDA(cudaMemcpyAsync(dv, P->v.data(), ne * sizeof(double), cudaMemcpyHostToDevice, st));
      TS_CUDA(cudaMemcpyAsync(doff, off.data(), ne * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      k_mm_expand<<<grid_for(ne), 256, 0, st>>>(dri, dci, dv, doff, ne, P->sym, n, key, pos, val);
      int end_bit = 1;
      while (end_bit < 63 && (1ull << end_bit) < (unsigned long long)(m * n)) ++end_bit;
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key_s, pos, perm, (int)cnt, 0, end_bit, st);
      char* tmp;
      if ((rc = ar.get(&tmp, tb))) return rc;
      if (cub::DeviceRadixSort::SortPairs(tmp, tb, key, key_s, pos, perm, (int)cnt, 0, end_bit, st) !=
          cudaSuccess) {
        set_error("radix sort of the Matrix Market coordinates failed");
        return TS_ECUDA;
      }
      k_mm_heads<<<grid_for(cnt), 256, 0, st>>>(key_s, cnt, head);
      size_t sb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, sb, head, uidx, (int)cnt, st);
      char* tmp2;
      if ((rc = ar.get(&tmp2, std::max(sb, (size_t)16)))) return rc;
      cub::DeviceScan::ExclusiveSum(tmp2, sb, head, uidx, (int)cnt, st);
      TS_CUDA(cudaMemsetAsync(rowcnt, 0, (m + 1) * sizeof(int), st));
      k_mm_unique<<<grid_for(cnt), 256, 0, st>>>(key_s, perm, val, head, uidx, cnt, n, ciout, vout, rowcnt);
      int last[2];
      TS_CUDA(cudaMemcpyAsync(&last[0], uidx + cnt - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
      TS_CUDA(cudaMemcpyAsync(&last[1], head + cnt - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
      size_t sb2 = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, sb2, rowcnt, rp, (int)(m + 1), st);
      char* tmp3;
      if ((rc = ar.get(&tmp3, std::max(sb2, (size_t)16)))) return rc;
      cub::DeviceScan::ExclusiveSum(tmp3, sb2, rowcnt, rp, (int)(m + 1), st);
      TS_CUDA(cudaStreamSynchronize(st));
      uniq = (int64_t)last[0] + last[1];
    } else {
      TS_CUDA(cudaMemsetAsync(rp, 0, (m + 1) * sizeof(int), st));
      TS_CUDA(cudaStreamSynchronize(st));
    }
    rc = ts_matrix_create_csr(rp, ciout, vout, m, n, uniq, device, stream, &A);
  }
  if (rc) return rc;
  if (duplicates) *duplicates = cnt - uniq;
  *out = A;
  return 0;
}

}  // extern "C"

#include "ts_drivers.cuh"
