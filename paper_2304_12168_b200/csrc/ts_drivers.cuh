// Solve drivers (host side of the device state machines) and the operator /
// CTA-piece ABI entry points.  Included once, from ts_lib.cu.
#pragma once

#include <functional>
#include <type_traits>

namespace ts {

// direct (non-graph) iteration: every kernel predicated on device state
using BodyFn = std::function<int(cudaStream_t)>;
// graph iteration: populate the WHILE body graph (captures + conditional nodes)
using GraphFn = std::function<int(cudaGraph_t body, cudaGraphConditionalHandle hwhile, cudaStream_t cap)>;

// add a SWITCH node at the current point of an ongoing capture on `cap`
static int capture_switch(cudaStream_t cap, cudaGraphConditionalHandle h, int ncases,
                          cudaGraph_t** cases) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  TS_CUDA(cudaStreamGetCaptureInfo(cap, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeSwitch;
  np.conditional.size = ncases;
  cudaGraphNode_t node;
  TS_CUDA(cudaGraphAddNode(&node, g, deps, nd, &np));
  TS_CUDA(cudaStreamUpdateCaptureDependencies(cap, &node, 1, cudaStreamSetCaptureDependencies));
  *cases = np.conditional.phGraph_out;
  return 0;
}

static int capture_into(cudaStream_t cap, cudaGraph_t g, const std::function<int(cudaStream_t)>& f) {
  // relaxed: the capture holds kernel launches on a private stream only, and
  // nothing another solver thread does (allocations, module loads, its own
  // captures) may invalidate it
  TS_CUDA(cudaStreamBeginCaptureToGraph(cap, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  const int rc = f(cap);
  cudaGraph_t out = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cap, &out);
  if (rc) return rc;
  if (ce != cudaSuccess) {
    set_error("graph capture failed: %s", cudaGetErrorString(ce));
    return TS_ECUDA;
  }
  return 0;
}

// ---- solve inputs without the copy engines -------------------------------
// A solve's host->device traffic (its state, b, x0) goes through kernels that
// read pinned / mapped host memory over PCIe instead of cudaMemcpy: the H2D
// copy engine may be busy for tens of milliseconds with another stream's
// matrix upload (the double-buffered pipeline of same-shaped problems), and a
// small cudaMemcpy queued behind it would stall the whole solve.
__global__ void k_put_state(SolveState* ds, const SolveState s) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *ds = s;
}
__global__ void k_put_ll(long long* p, long long v) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *p = v;
}
__global__ void k_copy_in(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

static SolveState* pinned_state() {
  static thread_local SolveState* hs = nullptr;
  if (!hs) {
    StructShared structural;
    if (cudaHostAlloc(&hs, sizeof(SolveState) + 64, cudaHostAllocDefault) != cudaSuccess) {
      hs = nullptr;
    }
  }
  return hs;
}

// Sharded passes.  Every launch we enqueue is counted.  The exchange step of
// a pass follows its layout:
//  * column blocks (wide A): A v = [local partial -> symmetric slot] +
//    [k_ar_vec: rank-ordered m-vector sum + the real epilogue]; A^T v is local
//    with its finisher deferred to k_ar_scalars;
//  * tall row blocks: the mirror image — A^T v sums an n-vector over ranks,
//    A v is local with its scalars summed;
//  * square banded row blocks: k_halo brings the neighbours' edges into the
//    input vector's padding, the pass is local, every scalar is summed.
// In an emulated world (ranks sharing one GPU) the host orders each exchange
// (Comm::exchange) between producer and consumer kernels.
inline int ar_grid(int64_t len, int sms) {
  int64_t g = (len + kNT * 4 - 1) / (kNT * 4);
  const int64_t cap = (int64_t)sms * 2;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}
template <int K>
constexpr unsigned all_slots() { return (K >= 32) ? ~0u : ((1u << K) - 1u); }

template <class Epi>
static int pass(const Mat& M, int trans, const double* x, XS xs, const Epi& e, const Work& w,
                cudaStream_t s) {
  ++g_launches;
  Epi e2 = e;
  if constexpr (std::is_base_of<EpiBase, Epi>::value) e2.tclass = trans ? 1 : 0;
  if (!M.comm) return launch_pass(M, trans, x, xs, e2, w, s);
  const Comm& C = *M.comm;
  const CommDev cd = C.dev_view();
  ++g_launches;
  if (M.row_shard) {  // halo in, local pass, every reduction slot summed over ranks
    double* xm = const_cast<double*>(x);
    if (C.local) {
      g_launches += 2;
      k_halo<Epi><<<1, kNT, 0, s>>>(e2, xm, M.m, M.halo, cd, 1);
      TS_CHECK(C.exchange(s));
      k_halo<Epi><<<1, kNT, 0, s>>>(e2, xm, M.m, M.halo, cd, 2);
    } else {
      g_launches += 1;
      k_halo<Epi><<<1, kNT, 0, s>>>(e2, xm, M.m, M.halo, cd, 3);
    }
    EpiDefer<Epi> d{e2, cd};
    TS_CHECK(launch_pass(M, trans, x, xs, d, w, s));
    TS_CHECK(C.exchange(s));
    k_ar_scalars<Epi><<<1, kNT, 0, s>>>(e2, cd, all_slots<Epi::K>());
    TS_CUDA(cudaGetLastError());
    return 0;
  }
  const bool vec_sum = M.tall_shard ? trans != 0 : trans == 0;
  if (vec_sum) {
    const int64_t len = trans ? M.n : M.m;
    if (len > (int64_t)cd.vec_cap) TS_INVAL("communicator vector capacity too small");
    EpiSymStore<Epi> ps{e2, cd};
    TS_CHECK(launch_pass(M, trans, x, xs, ps, w, s));
    TS_CHECK(C.exchange(s));
    k_ar_vec<Epi><<<ar_grid(len, M.sms), kNT, 0, s>>>(len, e2, w, cd);
  } else {
    EpiDefer<Epi> d{e2, cd};
    TS_CHECK(launch_pass(M, trans, x, xs, d, w, s));
    TS_CHECK(C.exchange(s));
    k_ar_scalars<Epi><<<1, kNT, 0, s>>>(e2, cd, all_slots<Epi::K>());
  }
  TS_CUDA(cudaGetLastError());
  return 0;
}
// vector passes: Epi::kShardMask marks the slots that reduce over n-space;
// they are per-rank partials on column blocks, the other (m-space) slots on
// tall row blocks, every slot on square row blocks
template <class Epi>
static int vecpass(const Mat& M, int64_t len, const Epi& e, const Work& w, cudaStream_t s) {
  ++g_launches;
  Epi e2 = e;
  unsigned mask = 0;
  if constexpr (std::is_base_of<EpiBase, Epi>::value) {
    e2.tclass = 2;
    mask = Epi::kShardMask;
  }
  if (M.comm && M.row_shard) mask = all_slots<Epi::K>();
  else if (M.comm && M.tall_shard) mask = all_slots<Epi::K>() & ~mask;
  if (!M.comm || !mask) return launch_vec(len, M.sms, e2, w, s);
  const CommDev cd = M.comm->dev_view();
  ++g_launches;
  EpiDefer<Epi> d{e2, cd};
  TS_CHECK(launch_vec(len, M.sms, d, w, s));
  TS_CHECK(M.comm->exchange(s));
  k_ar_scalars<Epi><<<1, kNT, 0, s>>>(e2, cd, mask);
  TS_CUDA(cudaGetLastError());
  return 0;
}

// ----------------------------------------------------------- instances ----
// A solver instance owns everything a solve touches on the device — state,
// reduction workspace, trace ring, vectors — plus the instantiated CUDA graph
// whose kernel nodes bake those addresses in.  Instances are cached on the
// (immutable) matrix handle per solver shape, so a repeated solve is just
// memcpy-in, init kernels, graph launches, final kernels, memcpy-out.
// Conditional graphs are built, run and destroyed under one process-wide lock:
// with a pool of solver threads (TRISOLVE_WORKERS), building or destroying one
// thread's graph while another thread's WHILE graph was executing made
// cudaGraphAddNode fail now and then, and once crashed inside the destroy (one
// run in ~20-40 of tests/test_gpu_cli.py::test_bench_rows).  The lock is held
// from the graph launch to the state read-back that follows it, so the solves
// of one process take turns on the device they would share anyway; direct
// launches (TS_NO_GRAPH, emulated worlds) are not affected.
inline std::mutex& graph_mu() {
  static std::mutex mu;
  return mu;
}

struct Instance {
  int key[4] = {0, 0, 0, 0};
  bool in_use = false;
  std::vector<void*> allocs;
  SolveState* ds = nullptr;
  Work wk;
  ts_trace_row* dtrace = nullptr;
  int seg_cap = 8192;
  // TA family vectors
  double *b = nullptr, *bp = nullptr, *gap = nullptr, *d = nullptr, *x = nullptr, *cv = nullptr,
         *fr = nullptr, *t1 = nullptr, *x0 = nullptr;
  // CTA vectors
  double *xs = nullptr;
  KrylovPtrs kp;
  ProbePtrs pp = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // graph
  cudaGraph_t graph = nullptr;
  cudaGraphNode_t wnode = nullptr;  // the WHILE node of `graph`
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  bool no_graph = false;  // the graph could not be built: iterations are launched directly
  cudaStream_t out = nullptr;  // result read-back, concurrent with the final residual passes
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  int64_t pad = 0;  // row-block shards: halo entries before and after every vector
  double* hstage = nullptr;  // pinned staging of pageable host inputs (lazily sized)
  size_t hstage_n = 0;
  // dst (device, n) <- src (device, pinned host, or pageable host), copy-engine free
  int stage_in(double* dst, const double* src, int64_t n, cudaStream_t st) {
    if (n <= 0) return 0;
    cudaPointerAttributes at;
    const double* from = src;
    if (cudaPointerGetAttributes(&at, src) != cudaSuccess) {
      cudaGetLastError();
      at.type = cudaMemoryTypeUnregistered;
    }
    if (at.type == cudaMemoryTypeHost && at.devicePointer) {
      from = static_cast<const double*>(at.devicePointer);
    } else if (at.type == cudaMemoryTypeUnregistered) {  // pageable: through pinned staging
      if (hstage_n < (size_t)n) {
        TS_CUDA(cudaStreamSynchronize(st));
        if (hstage) cudaFreeHost(hstage);
        hstage = nullptr;
        hstage_n = 0;
        TS_CUDA(cudaHostAlloc(&hstage, (size_t)n * sizeof(double), cudaHostAllocMapped));
        hstage_n = (size_t)n;
      }
      TS_CUDA(cudaStreamSynchronize(st));  // the previous staged input was consumed
      memcpy(hstage, src, (size_t)n * sizeof(double));
      double* dp = nullptr;
      TS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), hstage, 0));
      from = dp;
    }
    const int64_t g = std::min<int64_t>((n + 255) / 256, 1024);
    k_copy_in<<<(int)g, 256, 0, st>>>(dst, from, n);
    TS_CUDA(cudaGetLastError());
    return 0;
  }
  template <class T>
  int alloc(T** out, size_t count) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>((count + 2 * pad) * sizeof(T), 16);
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      set_error("cudaMalloc(%zu) for a solver instance failed", bytes);
      return TS_ENOMEM;
    }
    if (pad) cudaMemset(p, 0, bytes);
    allocs.push_back(p);
    *out = static_cast<T*>(p) + pad;
    return 0;
  }
  int init_common(const Mat& M) {
    const int pmax = work_blocks(M.sms);
    TS_CHECK(alloc(&wk.bacc, (size_t)pmax * kKMax));
    TS_CHECK(alloc(&wk.facc, (size_t)pmax * kKMax));
    TS_CHECK(alloc(&wk.bpart, (size_t)pmax * 2));
    TS_CHECK(alloc(&wk.tpart, (size_t)pmax * 2 * kCW));
    TS_CHECK(alloc(&wk.npart, (size_t)std::max<int64_t>(M.npart, 1)));
    TS_CUDA(cudaMemset(wk.npart, 0, sizeof(double) * std::max<int64_t>(M.npart, 1)));
    TS_CHECK(alloc(&wk.cnt, (size_t)pmax));
    TS_CHECK(alloc(&wk.done, 4));
    wk.pmax = pmax;
    TS_CUDA(cudaMemset(wk.cnt, 0, sizeof(unsigned) * pmax));
    TS_CUDA(cudaMemset(wk.done, 0, sizeof(unsigned) * 4));
    TS_CHECK(alloc(&ds, 1));
    TS_CHECK(alloc(&dtrace, (size_t)seg_cap));
    TS_CUDA(cudaEventCreate(&ev0));
    TS_CUDA(cudaEventCreate(&ev1));
    return 0;
  }
  // drop a (partially) built graph: the next solve rebuilds it or runs without
  void drop_graph() {
    std::lock_guard<std::mutex> lk(graph_mu());
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (cap) cudaStreamDestroy(cap);
    exec = nullptr;
    graph = nullptr;
    cap = nullptr;
    wnode = nullptr;
  }
  // a build failed: the half-built graph is abandoned, not destroyed (the driver
  // crashed in cuGraphDestroy on such a graph); happens, if ever, once per instance
  void abandon_graph() {
    cudaGetLastError();
    exec = nullptr;
    graph = nullptr;
    cap = nullptr;
    wnode = nullptr;
  }
  ~Instance() {
    if (hstage) cudaFreeHost(hstage);
    drop_graph();
    if (out) cudaStreamDestroy(out);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (void* p : allocs) cudaFree(p);
  }

  // The loop has stopped and the host has read the state (a synchronisation
  // point), so x is final: its device->host copy runs on a second stream while
  // the final residual passes (which only read x) run on the solve's stream.
  int read_back(void* dst, const void* src, size_t bytes) {
    if (!out) TS_CUDA(cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking));
    TS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, out));
    return 0;
  }
  int read_back_done() {
    if (out) TS_CUDA(cudaStreamSynchronize(out));
    return 0;
  }

  int build(const GraphFn& gbody) {
    std::unique_lock<std::shared_mutex> sl(struct_mu());  // no allocation / free / device sync meanwhile
    std::lock_guard<std::mutex> lk(graph_mu());
    TS_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    TS_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    TS_CUDA(cudaGraphAddNode(&wnode, graph, nullptr, 0, &np));
    cudaGraph_t bodyg = np.conditional.phGraph_out[0];
    TS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    TS_CHECK(gbody(bodyg, h, cap));
    TS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    return 0;
  }
};

void destroy_instances(Mat* M) {
  std::lock_guard<std::mutex> g(M->cache_mu);
  for (Instance* I : M->cache) delete I;
  M->cache.clear();
}

// Take a free cached instance with this key, or make one with `setup`.
static int acquire(const Mat& Mc, const int key[4], const std::function<int(Instance*)>& setup,
                   Instance** out) {
  Mat& M = const_cast<Mat&>(Mc);  // the cache is the handle's only mutable part
  {
    std::lock_guard<std::mutex> g(M.cache_mu);
    for (Instance* I : M.cache) {
      if (!I->in_use && memcmp(I->key, key, sizeof(I->key)) == 0) {
        I->in_use = true;
        *out = I;
        return 0;
      }
    }
  }
  StructShared structural;  // the instance's allocations
  Instance* I = new Instance();
  memcpy(I->key, key, sizeof(I->key));
  I->pad = M.row_shard ? M.halo : 0;
  int rc = I->init_common(M);
  if (!rc) rc = setup(I);
  if (rc) {
    delete I;
    return rc;
  }
  I->in_use = true;
  {
    std::lock_guard<std::mutex> g(M.cache_mu);
    if (M.cache.size() < 16) M.cache.push_back(I);
    else I->key[3] = -1;  // uncached: released by delete
  }
  *out = I;
  return 0;
}
static void release(const Mat& Mc, Instance* I) {
  Mat& M = const_cast<Mat&>(Mc);
  if (I->key[3] == -1) {
    delete I;
    return;
  }
  std::lock_guard<std::mutex> g(M.cache_mu);
  I->in_use = false;
}
struct InstanceLease {
  const Mat& M;
  Instance* I = nullptr;
  explicit InstanceLease(const Mat& m) : M(m) {}
  ~InstanceLease() {
    if (I) release(M, I);
  }
};

// Per-call driver state around an instance.
struct SolveCtx {
  const Mat& M;
  cudaStream_t st;
  Instance* I;
  SolveState* hs = nullptr;
  long long* hflushed = nullptr;
  ts_trace_row* utrace = nullptr;
  int64_t ucap = 0;
  long long flushed = 0;

  SolveCtx(const Mat& m, cudaStream_t s, Instance* inst) : M(m), st(s), I(inst) {}

  int init(SolveState& init_state, ts_trace_row* trace, int64_t trace_cap) {
    hs = pinned_state();
    if (!hs) {
      set_error("cudaHostAlloc for the solve state failed");
      return TS_ENOMEM;
    }
    hflushed = reinterpret_cast<long long*>(reinterpret_cast<char*>(hs) + sizeof(SolveState));
    utrace = trace;
    ucap = trace ? trace_cap : 0;
    init_state.trace = I->dtrace;
    init_state.seg_cap = I->seg_cap;
    for (int i = 0; i < 4; ++i) init_state.kt[i] = KTimer{~0ull, 0ull, 0, 0};
    *hs = init_state;
    TS_CUDA(cudaEventRecord(I->ev0, st));
    k_put_state<<<1, 32, 0, st>>>(I->ds, init_state);
    TS_CUDA(cudaGetLastError());
    return 0;
  }

  int read_state() {
    TS_CUDA(cudaMemcpyAsync(hs, I->ds, sizeof(SolveState), cudaMemcpyDeviceToHost, st));
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("device failure during solve: %s", cudaGetErrorString(e));
      return TS_ECUDA;
    }
    return 0;
  }

  int flush() {
    const long long upto = hs->trace_count;
    if (upto == flushed) return 0;
    const int seg_cap = I->seg_cap;
    while (flushed < upto) {
      const long long ring = flushed % seg_cap;
      long long chunk = std::min<long long>(upto - flushed, seg_cap - ring);
      if (flushed < ucap) {
        const long long n = std::min<long long>(chunk, ucap - flushed);
        TS_CUDA(cudaMemcpyAsync(utrace + flushed, I->dtrace + ring, n * sizeof(ts_trace_row),
                                cudaMemcpyDefault, st));
      }
      flushed += chunk;
    }
    *hflushed = flushed;
    k_put_ll<<<1, 32, 0, st>>>(&I->ds->trace_flushed, flushed);
    TS_CUDA(cudaGetLastError());
    TS_CUDA(cudaStreamSynchronize(st));  // ring reuse
    return 0;
  }

  int run(const BodyFn& body, const GraphFn& gbody, const std::function<int(cudaStream_t)>& maint) {
    TS_CHECK(read_state());
    TS_CHECK(flush());
    static const bool no_graph = getenv("TS_NO_GRAPH") != nullptr;
    // an emulated world's exchanges are host-ordered: one iteration per launch
    const bool direct = no_graph || (M.comm && M.comm->local);
    while (hs->status == TS_RUNNING) {
      if (hs->maint != MAINT_NONE) {
        // graph mode services revalidation / recheck inside the loop; the host
        // path runs in direct mode, for the probe, and after a trace-ring flush
        static const bool dbg = getenv("TS_DEBUG_MAINT") != nullptr;
        if (dbg) fprintf(stderr, "[trisolve] host maintenance %d at iteration %lld\n", hs->maint, hs->iterations);
        TS_CHECK(maint(st));
      } else if (!direct && !I->no_graph) {
        if (!I->exec) {
          // a failed build is retried once; after that this instance launches
          // its iterations directly (same kernels, same results)
          int brc = I->build(gbody);
          if (brc) {
            I->abandon_graph();
            brc = I->build(gbody);
          }
          if (brc) {
            I->abandon_graph();
            I->no_graph = true;
            continue;
          }
        }
        std::lock_guard<std::mutex> lk(graph_mu());
        TS_CUDA(cudaGraphLaunch(I->exec, st));
        TS_CHECK(read_state());  // the graph has left the device before the lock is released
        TS_CHECK(flush());
        continue;
      } else {
        TS_CHECK(body(st));
      }
      TS_CHECK(read_state());
      TS_CHECK(flush());
    }
    return 0;
  }

  int finish_timing(ts_result* res) {
    TS_CUDA(cudaEventRecord(I->ev1, st));
    TS_CUDA(cudaEventSynchronize(I->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, I->ev0, I->ev1);
    res->elapsed_ms = ms;
    res->kernel_launches = hs->launches;  // every solver kernel bumps it on the device
    return 0;
  }
};

static void fill_result(const SolveState& s, ts_result* r) {
  r->status = s.status;
  r->detail = s.detail;
  r->iterations = s.iterations;
  r->residual_norm = s.residual_norm;
  r->normal_residual_norm = s.normal_residual_norm;
  r->rho = s.rho;
  r->lower_bound = s.lower_bound;
  r->has_lower_bound = s.has_lb;
  r->min_x_entry = s.x_min;
  r->detail_value = s.detail_value;
  r->trace_rows = s.trace_count;
  r->trivial = s.trivial;
  for (int i = 0; i < 4; ++i) {
    r->kernel_ms[i] = s.kt[i].total_ns * 1e-6;
    r->kernel_count[i] = s.kt[i].count;
  }
  r->gap_norm = s.gap_norm;
  r->x_norm = s.x_norm;
}

// ================================================================== TA ====
struct TaArgs {
  int mode = MODE_ADAPTIVE;
  int gram = 0;
  double eps = 0, eps_prime = -1, rho_cap = -1, rho_max = -1, rho = 0;
  long long max_iters = 100000;
  int halvings = 0;
  const double* x0 = nullptr;
};

// kernels of the TA family bound to one instance
struct TaKernels {
  const Mat& M;
  Instance* I;
  int gram, relu;
  int64_t mo, no, mx;

  // y = Op v with a fused epilogue (Op = A, or A^T A for the Gram pair)
  template <class Epi>
  int op_apply(cudaStream_t s, const double* v, XS xs, const Epi& epi, int pred) const {
    if (!gram) return pass(M, 0, v, xs, epi, I->wk, s);
    EpiStore es;
    es.st = I->ds; es.y = I->t1; es.pred = pred;
    TS_CHECK(pass(M, 0, v, xs, es, I->wk, s));
    return pass(M, 1, I->t1, XS{}, epi, I->wk, s);
  }
  template <class Epi>
  int op_apply_t(cudaStream_t s, const double* v, const Epi& epi, int pred) const {
    if (!gram) return pass(M, 1, v, XS{}, epi, I->wk, s);
    EpiStore es;
    es.st = I->ds; es.y = I->t1; es.pred = pred;
    TS_CHECK(pass(M, 0, v, XS{}, es, I->wk, s));
    return pass(M, 1, I->t1, XS{}, epi, I->wk, s);
  }
  // c = Op^T gap; the finisher decides pivot / expand / stop
  int c_pass(cudaStream_t s, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hsw,
             int use) const {
    EpiTaC ec;
    ec.st = I->ds; ec.c = I->cv; ec.cond = hw; ec.use_cond = use; ec.sw = hsw; ec.use_sw = use;
    return op_apply_t(s, I->gap, ec, 1);
  }
  // pivot: v = Op pre (fused d.d, gap.d), then the convex-combination update
  int pivot(cudaStream_t s, cudaGraphConditionalHandle hw, int use) const {
    EpiTaV ev;
    ev.st = I->ds; ev.bp = I->bp; ev.gap = I->gap; ev.d = I->d;
    XS xs;
    xs.sp = &I->ds->scale;
    xs.relu = relu;
    TS_CHECK(op_apply(s, I->cv, xs, ev, 2));
    EpiTaUpd eu;
    eu.st = I->ds; eu.cond = hw; eu.use_cond = use;
    eu.b = I->b; eu.d = I->d; eu.c = I->cv; eu.bp = I->bp; eu.gap = I->gap; eu.x = I->x;
    eu.m = mo; eu.n = no; eu.relu = relu;
    return vecpass(M, mx, eu, I->wk, s);
  }
  // b' = A x, gap = b - b' (every 512 pivots, triangle.py:239-242)
  int revalidate(cudaStream_t s, cudaGraphConditionalHandle hw, int use) const {
    EpiTaBp eb;
    eb.st = I->ds; eb.b = I->b; eb.bp = I->bp; eb.gap = I->gap; eb.kind = 1;
    eb.cond = hw; eb.use_cond = use;
    return op_apply(s, I->x, XS{}, eb, 0);
  }
  // graph body: [c pass] -> SWITCH{0: pivot, 1: revalidate}  (expand / stop
  // select no case; a due revalidation idles the c pass, which selects case 1)
  int graph(cudaGraph_t bodyg, cudaGraphConditionalHandle hw, cudaStream_t cap) const {
    cudaGraphConditionalHandle hsw;
    TS_CUDA(cudaGraphConditionalHandleCreate(&hsw, bodyg, 0, 0));
    cudaGraph_t* cases = nullptr;
    TS_CHECK(capture_into(cap, bodyg, [&](cudaStream_t s) -> int {
      TS_CHECK(c_pass(s, hw, hsw, 1));
      return capture_switch(s, hsw, 2, &cases);
    }));
    TS_CHECK(capture_into(cap, cases[0], [&](cudaStream_t s) -> int { return pivot(s, hw, 1); }));
    return capture_into(cap, cases[1], [&](cudaStream_t s) -> int { return revalidate(s, hw, 1); });
  }
};

static int ta_solve(const Mat& M, const double* b_in, const TaArgs& a, double* x_out,
                    double* bp_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                    cudaStream_t st) {
  const int64_t mo = a.gram ? M.n : M.m;  // operator rows (TA's b-space)
  const int64_t no = M.n;                 // operator cols (x-space)
  const int64_t mx = std::max(mo, no);
  const int relu = a.mode == MODE_LP;
  const int key[4] = {1, a.gram, relu, 0};
  InstanceLease lease(M);
  TS_CHECK(acquire(M, key, [&](Instance* I) -> int {
    TS_CHECK(I->alloc(&I->b, mo));
    TS_CHECK(I->alloc(&I->bp, mo));
    TS_CHECK(I->alloc(&I->gap, mo));
    TS_CHECK(I->alloc(&I->d, mo));
    TS_CHECK(I->alloc(&I->fr, mo));
    TS_CHECK(I->alloc(&I->x, no));
    TS_CHECK(I->alloc(&I->cv, no));
    TS_CHECK(I->alloc(&I->x0, no));
    if (a.gram) TS_CHECK(I->alloc(&I->t1, M.m));
    return 0;
  }, &lease.I));
  Instance* I = lease.I;
  SolveCtx c(M, st, I);
  SolveState s0;
  memset(&s0, 0, sizeof(s0));
  s0.mode = a.mode;
  s0.gram = a.gram;
  s0.eps = a.eps;
  s0.eps_prime = a.eps_prime;
  s0.rho_cap = a.rho_cap;
  s0.rho_max = a.rho_max;
  s0.rho = a.mode == MODE_BALL ? a.rho : 0.0;
  s0.max_iters = a.max_iters;
  s0.halvings_left = std::max(0, a.halvings);
  s0.a_fro = a.gram ? M.fro * M.fro : M.fro;
  s0.m_rows = M.comm ? (a.gram ? M.n_global : M.m_global) : mo;
  s0.n_cols = M.comm ? M.n_global : no;
  TS_CHECK(c.init(s0, trace, trace_cap));
  SolveState* ds = I->ds;
  const Work& wk = I->wk;
  TaKernels K{M, I, a.gram, relu, mo, no, mx};
  TS_CHECK(I->stage_in(I->b, b_in, mo, st));

  // ---- init (triangle.py:197-204, feasibility.py:77-79)
  if (a.x0) {
    TS_CHECK(I->stage_in(I->x0, a.x0, no, st));
    EpiNormTo en;
    en.st = ds; en.v = I->x0; en.len = no; en.what = 0;
    TS_CHECK(vecpass(M, no, en, wk, st));
    EpiCopyWarm ec;
    ec.st = ds; ec.src = I->x0; ec.dst = I->x;
    TS_CHECK(vecpass(M, no, ec, wk, st));
    EpiTaBp eb;
    eb.st = ds; eb.b = I->b; eb.bp = I->bp; eb.gap = I->gap; eb.kind = 0;
    TS_CHECK(K.op_apply(st, I->x, XS{}, eb, 0));
  } else {
    EpiTaInitZero ez;
    ez.st = ds; ez.b = I->b; ez.bp = I->bp; ez.gap = I->gap; ez.x = I->x; ez.m = mo; ez.n = no;
    TS_CHECK(vecpass(M, mx, ez, wk, st));
  }
  BodyFn body = [&](cudaStream_t s) -> int {
    TS_CHECK(K.c_pass(s, 0, 0, 0));
    return K.pivot(s, 0, 0);
  };
  GraphFn gbody = [&](cudaGraph_t bodyg, cudaGraphConditionalHandle hw, cudaStream_t cap) -> int {
    return K.graph(bodyg, hw, cap);
  };
  auto maint = [&](cudaStream_t s) -> int { return K.revalidate(s, 0, 0); };
  TS_CHECK(c.run(body, gbody, maint));
  if (c.hs->error == TS_EDEGENERATE) {
    set_error("degenerate pivot: v coincides with the iterate");
    return TS_EDEGENERATE;
  }
  bool early = false;  // x (and b') on their way to the host during the final passes
  if (c.hs->trivial) {
    TS_CUDA(cudaMemsetAsync(I->x, 0, no * sizeof(double), st));
  } else {
    early = true;
    if (x_out) TS_CHECK(I->read_back(x_out, I->x, no * sizeof(double)));
    if (bp_out) TS_CHECK(I->read_back(bp_out, I->bp, mo * sizeof(double)));
    EpiFinalR efr;
    efr.st = ds; efr.b = I->b; efr.fr = I->fr;
    TS_CHECK(K.op_apply(st, I->x, XS{}, efr, 0));
    EpiFinalNR enr;
    enr.st = ds; enr.out = nullptr;
    TS_CHECK(K.op_apply_t(st, I->fr, enr, 0));
    EpiXNorm en;  // ||x|| for the min-norm bisection (triangle.py:306)
    en.st = ds; en.v = I->x;
    TS_CHECK(vecpass(M, no, en, wk, st));
  }
  TS_CHECK(c.read_state());
  if (!early) {
    if (x_out) TS_CUDA(cudaMemcpyAsync(x_out, I->x, no * sizeof(double), cudaMemcpyDefault, st));
    if (bp_out) TS_CUDA(cudaMemcpyAsync(bp_out, I->bp, mo * sizeof(double), cudaMemcpyDefault, st));
  } else {
    TS_CHECK(I->read_back_done());
  }
  fill_result(*c.hs, res);
  TS_CHECK(c.finish_timing(res));
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// ================================================================= CTA ====
struct CtaArgs {
  double epsilon = 1e-15;
  int t_max = 5;
  int gram = 1;
  long long max_iters = 100000;
  int known_solvable = 0;
  long long recheck_every = 250;
  double rcond = 1e-13;
  int accelerate = 0;
  int accel_patience = 3;
  double accel_ratio = 0.95;
  const double* x_start = nullptr;
  int enhanced = 0;
  int normal = 0;  // operator = A^T A of the handle (GramProduct)
};

// The pass that applies an operand of the CTA: A itself, or the implicit
// normal matrix G = A^T A (the reference's GramProduct, linalg.py:93-114),
// applied as A v -> t1, then A^T t1 with the real epilogue; G is symmetric,
// so G^T v = G v.  The store pass carries the outer epilogue's activity
// predicate, so an inactive pair skips both halves alike.
template <class Epi>
struct EpiTmpFor : EpiBase {
  static constexpr int K = 1;
  Epi e;
  double* y = nullptr;
  __device__ bool active() const { return e.active(); }
  __device__ void idle() const {}
  __device__ void elem(int64_t i, double v, double (&)[K]) const { y[i] = v; }
  __device__ void finish(double (&)[K]) const {}
};

struct CtaOp {
  const Mat& M;
  const Instance* I;
  int normal;
  int64_t mo() const { return normal ? M.n : M.m; }  // operator rows (b-space)
  int64_t no() const { return M.n; }                 // operator columns (x-space)
  template <class Epi>
  int apply(int trans, const double* v, const Epi& e, cudaStream_t s) const {
    if (!normal) return pass(M, trans, v, XS{}, e, I->wk, s);
    EpiTmpFor<Epi> t;
    t.st = e.st;
    t.e = e;
    t.y = I->t1;
    TS_CHECK(pass(M, 0, v, XS{}, t, I->wk, s));
    return pass(M, 1, I->t1, XS{}, e, I->wk, s);
  }
  template <class Epi>
  int N(const double* v, const Epi& e, cudaStream_t s) const { return apply(0, v, e, s); }
  template <class Epi>
  int T(const double* v, const Epi& e, cudaStream_t s) const { return apply(1, v, e, s); }
};

static int cta_alloc(Instance* I, const Mat& M, int t_max, int gram, int enhanced = 0, int normal = 0) {
  const int64_t mo = normal ? M.n : M.m, no = M.n;
  memset(&I->kp, 0, sizeof(I->kp));
  for (int i = 0; i <= t_max; ++i) TS_CHECK(I->alloc(&I->kp.p[i], mo));
  if (gram)
    for (int i = 0; i < t_max; ++i) TS_CHECK(I->alloc(&I->kp.q[i], no));
  TS_CHECK(I->alloc(&I->b, mo));
  TS_CHECK(I->alloc(&I->x, no));
  TS_CHECK(I->alloc(&I->xs, no));
  TS_CHECK(I->alloc(&I->fr, mo));
  if (normal) TS_CHECK(I->alloc(&I->t1, M.m));
  if (enhanced) {
    TS_CHECK(I->alloc(&I->pp.y, mo));
    TS_CHECK(I->alloc(&I->pp.hy, mo));
    TS_CHECK(I->alloc(&I->pp.aty, no));
    TS_CHECK(I->alloc(&I->pp.xh, no));
    TS_CHECK(I->alloc(&I->pp.fr2, mo));
  }
  return 0;
}

// enhanced probe steps 1..npairs-1 (centering.py:240-250), after the moments
static int cta_probe_kernels(const CtaOp& op, const Instance* I, int npairs, int gram, cudaStream_t s) {
  const Mat& M = op.M;
  for (int j = 1; j < npairs; ++j) {
    EpiProbeUpd eu;
    eu.st = I->ds; eu.kp = I->kp; eu.pp = I->pp; eu.x = I->x; eu.m = op.mo(); eu.n = op.no();
    eu.gram = gram; eu.j = j;
    TS_CHECK(vecpass(M, std::max(op.mo(), op.no()), eu, I->wk, s));
    EpiProbeN en;
    en.st = I->ds; en.y = I->pp.y; en.hy = I->pp.hy; en.j = j;
    if (gram) {
      EpiProbeT et;
      et.st = I->ds; et.aty = I->pp.aty; et.j = j;
      TS_CHECK(op.T(I->pp.y, et, s));
      TS_CHECK(op.N(I->pp.aty, en, s));
    } else {
      TS_CHECK(op.N(I->pp.y, en, s));
    }
  }
  return 0;
}

// stepped vs refined normal residual, adopt x_hat if it wins (centering.py:335-343)
static int cta_probe_finish(const CtaOp& op, const Instance* I, cudaStream_t s) {
  EpiProbeR r1;
  r1.st = I->ds; r1.b = I->b; r1.fr = I->fr;
  TS_CHECK(op.N(I->x, r1, s));
  EpiProbeNR n1;
  n1.st = I->ds; n1.which = 0;
  TS_CHECK(op.T(I->fr, n1, s));
  EpiProbeR r2;
  r2.st = I->ds; r2.b = I->b; r2.fr = I->pp.fr2;
  TS_CHECK(op.N(I->pp.xh, r2, s));
  EpiProbeNR n2;
  n2.st = I->ds; n2.which = 1;
  TS_CHECK(op.T(I->pp.fr2, n2, s));
  EpiProbeTake et;
  et.st = I->ds; et.xh = I->pp.xh; et.fr2 = I->pp.fr2; et.x = I->x; et.r = I->kp.p[0];
  et.m = op.mo(); et.n = op.no();
  return vecpass(op.M, std::max(op.mo(), op.no()), et, I->wk, s);
}

// moments pairs for orders 1..npairs (predicated on state t); `solve_last`
// makes the pair that equals the state's t run the Hankel solves
static int cta_pairs(const CtaOp& op, const Instance* I, int npairs, int gram, int solve_last,
                     cudaStream_t s, int slot = -1) {
  const bool pair = gram && !op.normal && band_pair_ok(op.M);
  bool dpair = gram && !op.normal && dense_pair_ok(op.M);
  // (kNoCoop from a launch helper: the cooperative grid would not be co-resident
  // on this device; the barrier-free kernels below take over)
  if (dpair && solve_last && dense_chain_ok(op.M, npairs)) {  // every pair of the iteration in one kernel
    const int rc = launch_chain_wdense(op.M, I->kp, I->ds, npairs, slot, I->wk, s);
    if (rc != kNoCoop) {
      ++g_launches;
      return rc;
    }
    dpair = false;
  }
  if (gram && !op.normal && solve_last && csr_chain_ok(op.M, npairs)) {  // L2-resident short-row CSR: the same
    const int rc = launch_chain_csr(op.M, I->kp, I->ds, npairs, slot, I->wk, s);
    if (rc != kNoCoop) {
      ++g_launches;
      return rc;
    }
  }
  for (int i = 1; i <= npairs; ++i) {
    if (dpair) {  // small dense: both passes in one cooperative kernel
      EpiCtaQ eq;
      eq.st = I->ds; eq.q = I->kp.q[i - 1]; eq.i = i; eq.tclass = 1; eq.slot = slot;
      EpiCtaP ep;
      ep.st = I->ds; ep.pprev = I->kp.p[i - 1]; ep.p = I->kp.p[i]; ep.i = i;
      ep.with_solve = solve_last; ep.tclass = 0; ep.slot = slot;
      const int rc = launch_pair_wdense(op.M, I->kp.p[i - 1], I->kp.q[i - 1], eq, ep, I->wk, s);
      if (rc == kNoCoop) {
        dpair = false;
        --i;  // this pair again, as two passes
        continue;
      }
      ++g_launches;
      TS_CHECK(rc);
    } else if (pair) {  // q_i = A^T p_{i-1} and p_i = A q_i in one kernel (square banded, L2-resident)
      EpiCtaQ eq;
      eq.st = I->ds; eq.q = I->kp.q[i - 1]; eq.i = i; eq.tclass = 1; eq.slot = slot;
      EpiCtaP ep;
      ep.st = I->ds; ep.pprev = I->kp.p[i - 1]; ep.p = I->kp.p[i]; ep.i = i;
      ep.with_solve = solve_last; ep.tclass = 0; ep.slot = slot;
      ++g_launches;
      TS_CHECK(launch_pair_band(op.M, I->kp.p[i - 1], eq, ep, I->wk, s));
    } else if (gram) {
      EpiCtaQ eq;
      eq.st = I->ds; eq.q = I->kp.q[i - 1]; eq.i = i; eq.slot = slot;
      TS_CHECK(op.T(I->kp.p[i - 1], eq, s));
      EpiCtaP ep;
      ep.st = I->ds; ep.pprev = I->kp.p[i - 1]; ep.p = I->kp.p[i]; ep.i = i;
      ep.with_solve = solve_last; ep.slot = slot;
      TS_CHECK(op.N(I->kp.q[i - 1], ep, s));
    } else {
      EpiCtaP ep;
      ep.st = I->ds; ep.pprev = I->kp.p[i - 1]; ep.p = I->kp.p[i]; ep.i = i;
      ep.with_solve = solve_last; ep.slot = slot;
      TS_CHECK(op.N(I->kp.p[i - 1], ep, s));
    }
  }
  return 0;
}

// one CTA step of at most `npairs` pairs: moments (+ Hankel in the last pair's
// finisher), candidate norms / retry rule, fused r / x update (tail)
static int cta_step_kernels(const CtaOp& op, const Instance* I, int npairs, int gram, cudaStream_t s,
                            cudaGraphConditionalHandle h, int use, int enhanced = 0,
                            cudaGraphConditionalHandle hsw = 0, int ncases = 0, int slot = -1) {
  const int64_t mo = op.mo(), no = op.no();
  EpiCtaCand ecd;
  ecd.st = I->ds; ecd.kp = I->kp; ecd.m = mo; ecd.slot = slot;
  EpiCtaUpd eu;
  eu.st = I->ds; eu.cond = h; eu.use_cond = use; eu.kp = I->kp; eu.x = I->x; eu.m = mo;
  eu.n = no; eu.gram = gram;
  eu.sw = hsw; eu.use_sw = ncases > 0; eu.ncases = ncases; eu.slot = slot;
  // both vector passes single-block (<= 1024 unknowns, unsharded): one kernel for the two
  static const bool vec_fuse_off = [] {
    const char* e = getenv("TS_VEC_FUSE");
    return e && e[0] == '0';
  }();
  const bool fuse = !vec_fuse_off && !op.M.comm && vec_grid(std::max(mo, no), op.M.sms) == 1;
  // ... and behind a chained small dense matrix, the whole iteration is one kernel
  static const bool tail_off = [] {
    const char* e = getenv("TS_CHAIN_TAIL");
    return e && e[0] == '0';
  }();
  if (fuse && !tail_off && !enhanced && gram && !op.normal && dense_pair_ok(op.M) && dense_chain_ok(op.M, npairs)) {
    ChainTail tl;
    tl.cand = ecd; tl.cand.tclass = 2;
    tl.upd = eu; tl.upd.tclass = 2;
    tl.len_cand = mo; tl.len_upd = std::max(mo, no);
    const int rc = launch_chain_wdense(op.M, I->kp, I->ds, npairs, slot, I->wk, s, &tl);
    if (rc != kNoCoop) {
      ++g_launches;
      return rc;
    }
  }
  TS_CHECK(cta_pairs(op, I, npairs, gram, 1, s, slot));
  if (enhanced) TS_CHECK(cta_probe_kernels(op, I, npairs, gram, s));
  if (!fuse) TS_CHECK(vecpass(op.M, mo, ecd, I->wk, s));
  if (fuse) {
    ++g_launches;
    ecd.tclass = 2;
    eu.tclass = 2;
    k_vec2<EpiCtaCand, EpiCtaUpd><<<1, kNT, 0, s>>>(mo, ecd, std::max(mo, no), eu, I->wk);
    TS_CUDA(cudaGetLastError());
    return 0;
  }
  return vecpass(op.M, std::max(mo, no), eu, I->wk, s);
}

static int cta_solve(const Mat& M, const double* b_in, const CtaArgs& a, double* x_out,
                     ts_trace_row* trace, int64_t trace_cap, ts_result* res, cudaStream_t st) {
  const int key[4] = {2 + 16 * a.normal, a.gram, a.t_max, a.enhanced};
  InstanceLease lease(M);
  TS_CHECK(acquire(M, key, [&](Instance* I) {
    return cta_alloc(I, M, a.t_max, a.gram, a.enhanced, a.normal);
  }, &lease.I));
  Instance* I = lease.I;
  const CtaOp op{M, I, a.normal};
  const int64_t mo = op.mo(), no = op.no();
  SolveCtx c(M, st, I);
  SolveState s0;
  memset(&s0, 0, sizeof(s0));
  s0.mode = MODE_CTA;
  s0.gram = a.gram;
  s0.epsilon = a.epsilon;
  s0.t_max = a.t_max;
  s0.max_iters = a.max_iters;
  s0.recheck_every = a.recheck_every;
  s0.known_solvable = a.known_solvable;
  s0.accelerate = a.accelerate;
  s0.accel_patience = a.accel_patience;
  s0.accel_ratio = a.accel_ratio;
  s0.rcond = a.rcond;
  s0.a_fro = a.normal ? M.fro * M.fro : M.fro;  // ||A^T A||_F as the reference's GramProduct reports it
  s0.m_rows = M.comm ? M.m_global : mo;
  s0.n_cols = M.comm ? M.n_global : no;
  s0.warm = 1;
  s0.enhanced = a.enhanced;
  s0.probe_done = 1;
  TS_CHECK(c.init(s0, trace, trace_cap));
  SolveState* ds = I->ds;
  const Work& wk = I->wk;
  TS_CHECK(I->stage_in(I->b, b_in, mo, st));
  if (a.x_start) {
    TS_CHECK(I->stage_in(I->xs, a.x_start, no, st));
    EpiCopyWarm ec;
    ec.st = ds; ec.src = I->xs; ec.dst = I->x;
    TS_CHECK(vecpass(M, no, ec, wk, st));
    EpiCtaInitR ei;
    ei.st = ds; ei.b = I->b; ei.r = I->kp.p[0];
    TS_CHECK(op.N(I->x, ei, st));
  } else {
    EpiCtaInit ei;
    ei.st = ds; ei.b = I->b; ei.r = I->kp.p[0]; ei.x = I->x; ei.m = mo; ei.n = no;
    TS_CHECK(vecpass(M, std::max(mo, no), ei, wk, st));
  }
  BodyFn body = [&](cudaStream_t s) -> int {
    return cta_step_kernels(op, I, a.t_max, a.gram, s, 0, 0, a.enhanced);
  };
  // ||x||, then r = b - A x against the maintained residual
  auto recheck = [&](cudaStream_t s, cudaGraphConditionalHandle hw, int use, cudaGraphConditionalHandle hsw,
                     int nocase, int need_maint = 0) -> int {
    EpiNormTo en;
    en.st = ds; en.v = I->x; en.len = no; en.what = 1; en.need_maint = need_maint;
    TS_CHECK(vecpass(M, no, en, wk, s));
    EpiCtaRecheck er;
    er.st = ds; er.b = I->b; er.r = I->kp.p[0]; er.need_maint = need_maint;
    er.cond = hw; er.use_cond = use; er.sw = hsw; er.use_sw = use && nocase > 0; er.nocase = nocase;
    return op.N(I->x, er, s);
  };
  // graph: [head: switch = t - 1] -> WHILE{ SWITCH{order 1 .. t_max} }: each case
  // launches exactly its t pairs + candidate + update, and the update's
  // finisher — which takes the next order from the schedule — selects the
  // next trip's case itself, so the head runs once per graph launch, not once
  // per iteration (tools/microbench/cond_handle.cu: a case kernel may set the
  // value the next trip's SWITCH reads; the first value may come from a
  // kernel node in the outer graph)
  // Default (plain CTA): no SWITCH at all.  One WHILE trip is one PERIOD of
  // the triangle-wave order schedule (2 t_max - 2 iterations); every
  // iteration's kernels are baked in with their schedule slot and run when the
  // state stands at that slot, so the conditional nodes cost one WHILE
  // evaluation per period instead of a WHILE and a SWITCH evaluation per
  // iteration (tools/microbench/lat_chain.cu: 3.5 + 3 us).  The recheck
  // kernels open every trip and idle unless it is due.  A solve that stops,
  // or re-enters, in mid-period idles through the rest of that trip.
  static const bool force_switch = getenv("TS_CTA_SWITCH") != nullptr;
  const int period = a.t_max == 1 ? 1 : 2 * a.t_max - 2;
  GraphFn gperiod = [&](cudaGraph_t bodyg, cudaGraphConditionalHandle hw, cudaStream_t cap) -> int {
    return capture_into(cap, bodyg, [&](cudaStream_t s) -> int {
      TS_CHECK(recheck(s, 0, 0, 0, 0, MAINT_RECHECK));
      for (int slot = 0; slot < period; ++slot) {
        const int t = a.t_max == 1 ? 1 : (slot < a.t_max ? slot + 1 : 2 * a.t_max - 1 - slot);
        TS_CHECK(cta_step_kernels(op, I, t, a.gram, s, hw, 1, 0, 0, 0, slot));
      }
      return 0;
    });
  };
  GraphFn gbody = [&](cudaGraph_t bodyg, cudaGraphConditionalHandle hw, cudaStream_t cap) -> int {
    if (!a.enhanced && !force_switch && period <= 16) return gperiod(bodyg, hw, cap);
    cudaGraphConditionalHandle hsw;
    TS_CUDA(cudaGraphConditionalHandleCreate(&hsw, bodyg, 0, 0));
    {
      cudaGraphNodeParams kp = {};
      kp.type = cudaGraphNodeTypeKernel;
      SolveState* dsp = ds;
      int nocase = a.t_max + 1;
      void* args[4] = {&dsp, &hsw, &hw, &nocase};
      kp.kernel.func = (void*)k_cta_head;
      kp.kernel.gridDim = dim3(1);
      kp.kernel.blockDim = dim3(32);
      kp.kernel.kernelParams = args;
      cudaGraphNode_t first;
      TS_CUDA(cudaGraphAddNode(&first, I->graph, nullptr, 0, &kp));
      TS_CUDA(cudaGraphAddDependencies(I->graph, &first, &I->wnode, 1));
    }
    cudaGraph_t* cases = nullptr;
    TS_CHECK(capture_into(cap, bodyg, [&](cudaStream_t s) -> int {
      return capture_switch(s, hsw, a.t_max + 1, &cases);
    }));
    for (int k = 0; k < a.t_max; ++k)
      TS_CHECK(capture_into(cap, cases[k], [&](cudaStream_t s) -> int {
        return cta_step_kernels(op, I, k + 1, a.gram, s, hw, 1, a.enhanced, hsw, a.t_max);
      }));
    // case t_max: the residual recheck every `recheck_every` iterations (centering.py:345-352)
    return capture_into(cap, cases[a.t_max], [&](cudaStream_t s) -> int {
      return recheck(s, hw, 1, hsw, a.t_max + 1);
    });
  };
  auto maint = [&](cudaStream_t s) -> int {
    if (c.hs->maint == MAINT_PROBE) return cta_probe_finish(op, I, s);
    return recheck(s, 0, 0, 0, 0);
  };
  TS_CHECK(c.run(body, gbody, maint));
  const bool early = !c.hs->trivial;  // x on its way to the host during the final passes
  if (early && x_out) TS_CHECK(I->read_back(x_out, I->x, no * sizeof(double)));
  if (!c.hs->trivial) {
    EpiFinalR efr;
    efr.st = ds; efr.b = I->b; efr.fr = I->fr;
    TS_CHECK(op.N(I->x, efr, st));
    EpiFinalNR enr;
    enr.st = ds; enr.out = nullptr;
    TS_CHECK(op.T(I->fr, enr, st));
  }
  TS_CHECK(c.read_state());
  if (!early) {
    if (x_out) TS_CUDA(cudaMemcpyAsync(x_out, I->x, no * sizeof(double), cudaMemcpyDefault, st));
  } else {
    TS_CHECK(I->read_back_done());
  }
  fill_result(*c.hs, res);
  TS_CHECK(c.finish_timing(res));
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

__global__ void k_hankel_one(const double* phi, int order, double rcond, double* alpha, int* ok) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *ok = hankel_min_norm(phi, order, rcond, alpha) ? 1 : 0;
}

}  // namespace ts

// ======================================================================= ABI
extern "C" {

#define TS_CHECK_HANDLE(A)                   \
  do {                                       \
    if (!(A)) TS_INVAL("null matrix handle"); \
  } while (0)
// the one-shot operator calls stage x into unpadded scratch and run one
// rank's pass alone: a shard handle (halo padding, collective exchanges)
// must go through the collective solvers instead
#define TS_CHECK_UNSHARDED(A)                                                              \
  do {                                                                                     \
    if ((A)->comm) TS_INVAL("operator calls are not supported on a sharded matrix handle"); \
  } while (0)

int ts_matvec(const ts_matrix* A, const double* x, double* y, void* stream) {
  TS_CHECK_HANDLE(A);
  TS_CHECK_UNSHARDED(A);
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk, A->npart));
    double *dx, *dy;
    TS_CHECK(stage_in(ar, x, A->n, &dx));
    TS_CHECK(ar.get(&dy, A->m));
    EpiStore e;
    e.y = dy;
    TS_CHECK(pass(*A, 0, dx, XS{}, e, wk, st));
    TS_CUDA(cudaMemcpyAsync(y, dy, A->m * sizeof(double), cudaMemcpyDefault, st));
  }
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int ts_rmatvec(const ts_matrix* A, const double* x, double* y, void* stream) {
  TS_CHECK_HANDLE(A);
  TS_CHECK_UNSHARDED(A);
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk, A->npart));
    double *dx, *dy;
    TS_CHECK(stage_in(ar, x, A->m, &dx));
    TS_CHECK(ar.get(&dy, A->n));
    EpiStore e;
    e.y = dy;
    TS_CHECK(pass(*A, 1, dx, XS{}, e, wk, st));
    TS_CUDA(cudaMemcpyAsync(y, dy, A->n * sizeof(double), cudaMemcpyDefault, st));
  }
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int ts_gram_matvec(const ts_matrix* A, const double* x, double* y, void* stream) {
  TS_CHECK_HANDLE(A);
  TS_CHECK_UNSHARDED(A);
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk, A->npart));
    double *dx, *dt, *dy;
    TS_CHECK(stage_in(ar, x, A->n, &dx));
    TS_CHECK(ar.get(&dt, A->m));
    TS_CHECK(ar.get(&dy, A->n));
    EpiStore e1;
    e1.y = dt;
    TS_CHECK(pass(*A, 0, dx, XS{}, e1, wk, st));
    EpiStore e2;
    e2.y = dy;
    TS_CHECK(pass(*A, 1, dt, XS{}, e2, wk, st));
    TS_CUDA(cudaMemcpyAsync(y, dy, A->n * sizeof(double), cudaMemcpyDefault, st));
  }
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

struct EpiResid {
  static constexpr int K = 1;
  const double* b;
  double* r;
  double* out;
  __device__ int op(int) const { return RED_SUM; }
  __device__ bool active() const { return true; }
  __device__ void idle() const {}
  __device__ KTimer* timer() const { return nullptr; }
  __device__ void finish_block() const {}
  __device__ void count_launch() const {}
  __device__ void prepare(double*) {}
  __device__ void elem(int64_t i, double y, double (&acc)[K]) const {
    const double f = __dsub_rn(b[i], y);
    r[i] = f;
    acc[0] = fma(f, f, acc[0]);
  }
  __device__ void finish(double (&red)[K]) const { *out = sqrt(red[0]); }
};

// r = b - Op x, ||r||, ||Op^T r|| for Op = A (normal = 0) or the implicit
// normal matrix A^T A (normal = 1; symmetric, so Op^T r = A^T (A r))
static int residual_impl(const ts_matrix* A, int normal, const double* x, const double* b, double* r_out,
                         double* r_norm, double* atr_norm, void* stream) {
  TS_CHECK_HANDLE(A);
  if (!x || !b) TS_INVAL("null argument");
  if (A->comm) TS_INVAL("not supported on a column-sharded matrix");
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t mo = normal ? A->n : A->m, no = A->n;
  double hn[2] = {0.0, 0.0};
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk, A->npart));
    double *dx, *db, *dr, *dn, *dt, *dm = nullptr;
    TS_CHECK(stage_in(ar, x, no, &dx));
    TS_CHECK(stage_in(ar, b, mo, &db));
    TS_CHECK(ar.get(&dr, mo));
    TS_CHECK(ar.get(&dt, no));
    TS_CHECK(ar.get(&dn, 2));
    if (normal) TS_CHECK(ar.get(&dm, A->m));
    auto apply = [&](int trans, const double* v, auto epi) -> int {
      if (!normal) return pass(*A, trans, v, XS{}, epi, wk, st);
      EpiStore es;
      es.y = dm;
      TS_CHECK(pass(*A, 0, v, XS{}, es, wk, st));
      return pass(*A, 1, dm, XS{}, epi, wk, st);
    };
    EpiResid er{db, dr, dn};
    TS_CHECK(apply(0, dx, er));
    if (atr_norm) {
      EpiStore es;
      es.y = dt;
      es.sq = dn + 1;
      TS_CHECK(apply(1, dr, es));
    }
    if (r_out) TS_CUDA(cudaMemcpyAsync(r_out, dr, mo * sizeof(double), cudaMemcpyDefault, st));
    TS_CUDA(cudaMemcpyAsync(hn, dn, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    TS_CUDA(cudaStreamSynchronize(st));
  }
  if (r_norm) *r_norm = hn[0];
  if (atr_norm) *atr_norm = sqrt(hn[1]);
  return 0;
}

int ts_residual(const ts_matrix* A, const double* x, const double* b, double* r_out,
                double* r_norm, double* atr_norm, void* stream) {
  return residual_impl(A, 0, x, b, r_out, r_norm, atr_norm, stream);
}

int ts_gram_residual(const ts_matrix* A, const double* x, const double* b, double* r_out,
                     double* r_norm, double* gr_norm, void* stream) {
  return residual_impl(A, 1, x, b, r_out, r_norm, gr_norm, stream);
}

static int dot_impl(const double* u, const double* v, int64_t len, double* out, int sq,
                    cudaStream_t st) {
  if (len < 0) TS_INVAL("negative length");
  int dev = 0;
  cudaGetDevice(&dev);
  Mat dummy;
  dummy.sms = sm_count(dev);
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(dummy.sms), &wk));
    double *du, *dv, *dout;
    TS_CHECK(stage_in(ar, u, (size_t)len, &du));
    dv = du;
    if (!sq) TS_CHECK(stage_in(ar, v, (size_t)len, &dv));
    TS_CHECK(ar.get(&dout, 1));
    if (len == 0) {
      TS_CUDA(cudaMemsetAsync(dout, 0, sizeof(double), st));
    } else {
      EpiDot e{du, dv, dout, sq};
      TS_CHECK(vecpass(dummy, len, e, wk, st));
    }
    TS_CUDA(cudaMemcpyAsync(out, dout, sizeof(double), cudaMemcpyDefault, st));
  }
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int ts_norm2(const double* v, int64_t len, double* out, void* stream) {
  return dot_impl(v, v, len, out, 1, (cudaStream_t)stream);
}
int ts_dot(const double* u, const double* v, int64_t len, double* out, void* stream) {
  return dot_impl(u, v, len, out, 0, (cudaStream_t)stream);
}

int ts_hankel_min_norm(const double* phi, int32_t t, int32_t order, double rcond, double* alpha,
                       void* stream) {
  if (t < 1 || t > kTMax) TS_INVAL("order t=%d outside 1..%d", t, kTMax);
  if (order < 1 || order > t) TS_INVAL("order %d outside 1..%d", order, t);
  cudaStream_t st = (cudaStream_t)stream;
  int ok = 0;
  {
    Arena ar(st);
    double *dphi, *dal;
    int* dok;
    TS_CHECK(stage_in(ar, phi, 2 * (size_t)t, &dphi));
    TS_CHECK(ar.get(&dal, (size_t)order));
    TS_CHECK(ar.get(&dok, 1));
    ++g_launches;
    k_hankel_one<<<1, 32, 0, st>>>(dphi, order, rcond, dal, dok);
    TS_CUDA(cudaGetLastError());
    TS_CUDA(cudaMemcpyAsync(alpha, dal, order * sizeof(double), cudaMemcpyDefault, st));
    TS_CUDA(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, st));
  }
  TS_CUDA(cudaStreamSynchronize(st));
  if (!ok) {
    set_error("SVD did not converge in Linear Least Squares");
    return TS_EINVAL;
  }
  return 0;
}

int ts_moments(const ts_matrix* A, int32_t h_mode, const double* r, int32_t t, double* phi,
               double* krylov, double* transposed, void* stream) {
  TS_CHECK_HANDLE(A);
  if (t < 1 || t > kTMax || t > A->m)
    TS_INVAL("order t=%d outside 1..%lld", t, (long long)std::min<int64_t>(A->m, kTMax));
  if (h_mode == 1 && A->m != A->n) TS_INVAL("symmetric mode requires a square matrix");
  if (A->comm) TS_INVAL("not supported on a column-sharded matrix");
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int gram = h_mode == 0;
  const int key[4] = {3, gram, kTMax, 0};
  InstanceLease lease(*A);
  TS_CHECK(acquire(*A, key, [&](Instance* I) { return cta_alloc(I, *A, kTMax, gram); }, &lease.I));
  Instance* I = lease.I;
  SolveCtx c(*A, st, I);
  SolveState s0;
  memset(&s0, 0, sizeof(s0));
  s0.mode = MODE_CTA;
  s0.t = t;
  s0.gram = gram;
  TS_CHECK(c.init(s0, nullptr, 0));
  TS_CUDA(cudaMemcpyAsync(I->kp.p[0], r, A->m * sizeof(double), cudaMemcpyDefault, st));
  TS_CHECK(cta_pairs(CtaOp{*A, I, 0}, I, t, gram, 0, st));
  TS_CHECK(c.read_state());
  memcpy(phi, c.hs->phi, 2 * t * sizeof(double));
  if (krylov)
    for (int i = 0; i <= t; ++i)
      TS_CUDA(cudaMemcpyAsync(krylov + (size_t)i * A->m, I->kp.p[i], A->m * sizeof(double),
                              cudaMemcpyDefault, st));
  if (transposed && gram)
    for (int i = 0; i < t; ++i)
      TS_CUDA(cudaMemcpyAsync(transposed + (size_t)i * A->n, I->kp.q[i], A->n * sizeof(double),
                              cudaMemcpyDefault, st));
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int ts_cta_step(const ts_matrix* A, int32_t h_mode, const double* x, const double* r, int32_t t,
                double rcond, double* x_out, double* r_out, int32_t* order_out,
                double* atr_norm_out, int32_t* status_out, void* stream) {
  TS_CHECK_HANDLE(A);
  if (t < 1 || t > kTMax || t > A->m)
    TS_INVAL("order t=%d outside 1..%lld", t, (long long)std::min<int64_t>(A->m, kTMax));
  if (h_mode == 1 && A->m != A->n) TS_INVAL("symmetric mode requires a square matrix");
  if (A->comm) TS_INVAL("not supported on a column-sharded matrix");
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int gram = h_mode == 0;
  const int key[4] = {3, gram, kTMax, 0};
  InstanceLease lease(*A);
  TS_CHECK(acquire(*A, key, [&](Instance* I) { return cta_alloc(I, *A, kTMax, gram); }, &lease.I));
  Instance* I = lease.I;
  SolveCtx c(*A, st, I);
  SolveState s0;
  memset(&s0, 0, sizeof(s0));
  s0.mode = MODE_CTA;
  s0.t = t;
  s0.t_max = t;
  s0.gram = gram;
  s0.known_solvable = 1;
  s0.max_iters = (long long)1 << 60;
  s0.rcond = rcond;
  s0.eps_abs = -1.0;
  TS_CHECK(c.init(s0, nullptr, 0));
  TS_CUDA(cudaMemcpyAsync(I->kp.p[0], r, A->m * sizeof(double), cudaMemcpyDefault, st));
  TS_CUDA(cudaMemcpyAsync(I->x, x, A->n * sizeof(double), cudaMemcpyDefault, st));
  EpiDot e{I->kp.p[0], I->kp.p[0], &I->ds->r_norm, 1};  // ||r|| for the monotone test
  TS_CHECK(vecpass(*A, A->m, e, I->wk, st));
  TS_CHECK(cta_step_kernels(CtaOp{*A, I, 0}, I, t, gram, st, 0, 0));
  TS_CHECK(c.read_state());
  if (c.hs->status == TS_NUMERICAL_FAILURE) {
    set_error("moment solve failed: SVD did not converge in Linear Least Squares");
    return TS_EINVAL;
  }
  const int nestatus = (c.hs->status == TS_NORMAL_EQ_SOLUTION) ? TS_NORMAL_EQ_SOLUTION : 0;
  if (status_out) *status_out = nestatus;
  if (!nestatus) {
    if (order_out) *order_out = c.hs->sel_order;
    if (atr_norm_out) *atr_norm_out = c.hs->atr_norm;
    if (x_out) TS_CUDA(cudaMemcpyAsync(x_out, I->x, A->n * sizeof(double), cudaMemcpyDefault, st));
    if (r_out)
      TS_CUDA(cudaMemcpyAsync(r_out, I->kp.p[0], A->m * sizeof(double), cudaMemcpyDefault, st));
  }
  TS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// ------------------------------------------------------- column sharding --
int ts_comm_create(int device, int rank, int world, int64_t vec_capacity, ts_comm** out,
                   void* ipc_handles_out) {
  StructShared structural;
  if (!out || !ipc_handles_out) TS_INVAL("null argument");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    TS_INVAL("rank %d / world %d outside 0..%d", rank, world, kMaxRanks);
  if (vec_capacity < 1) TS_INVAL("vector capacity must be positive");
  DeviceGuard g(device);
  Comm* c = new Comm();
  c->dev = device;
  c->rank = rank;
  c->world = world;
  c->vec_cap = (size_t)vec_capacity;
  const size_t slot = c->vec_cap + kArScalars;
  auto fail = [&](const char* what, cudaError_t e) {
    set_error("%s failed: %s", what, cudaGetErrorString(e));
    if (c->sym) cudaFree(c->sym);
    if (c->flags) cudaFree(c->flags);
    if (c->epoch) cudaFree(c->epoch);
    delete c;
    return TS_ECUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&c->sym, 2 * slot * sizeof(double))) != cudaSuccess) return fail("cudaMalloc(sym)", e);
  if ((e = cudaMalloc(&c->flags, 256)) != cudaSuccess) return fail("cudaMalloc(flags)", e);
  if ((e = cudaMalloc(&c->epoch, sizeof(unsigned long long))) != cudaSuccess) return fail("cudaMalloc(epoch)", e);
  cudaMemset(c->sym, 0, 2 * slot * sizeof(double));
  cudaMemset(c->flags, 0, 256);
  cudaMemset(c->epoch, 0, sizeof(unsigned long long));
  cudaIpcMemHandle_t hs, hf;
  if ((e = cudaIpcGetMemHandle(&hs, c->sym)) != cudaSuccess) return fail("cudaIpcGetMemHandle(sym)", e);
  if ((e = cudaIpcGetMemHandle(&hf, c->flags)) != cudaSuccess) return fail("cudaIpcGetMemHandle(flags)", e);
  memcpy(ipc_handles_out, &hs, sizeof(hs));
  memcpy(static_cast<char*>(ipc_handles_out) + 64, &hf, sizeof(hf));
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail("comm init", e);
  *out = reinterpret_cast<ts_comm*>(c);
  return 0;
}

// An emulated world: `world` ranks of this process on one device, each with
// its own symmetric slots, flags and epoch; peers are plain device pointers
// and every exchange is ordered on the host (LocalGroup, csrc/ts_comm.cuh).
// Each rank's solves must run on their own host thread.
int ts_comm_create_local(int device, int world, int64_t vec_capacity, const int32_t* devices,
                         ts_comm** out) {
  StructShared structural;
  if (!out) TS_INVAL("null argument");
  if (world < 1 || world > kMaxRanks) TS_INVAL("world %d outside 1..%d", world, kMaxRanks);
  if (vec_capacity < 1) TS_INVAL("vector capacity must be positive");
  std::vector<int> dev(world, device);
  if (devices)
    for (int r = 0; r < world; ++r) dev[r] = devices[r];
  // ranks on different GPUs read each other's slots over NVLink: peer access
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) {
      if (dev[r] == dev[q]) continue;
      int ok = 0;
      TS_CUDA(cudaDeviceCanAccessPeer(&ok, dev[r], dev[q]));
      if (!ok) TS_INVAL("device %d cannot access device %d (no peer path)", dev[r], dev[q]);
      DeviceGuard pg(dev[r]);
      const cudaError_t pe = cudaDeviceEnablePeerAccess(dev[q], 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) TS_CUDA(pe);
      cudaGetLastError();
    }
  DeviceGuard g(device);
  auto grp = std::make_shared<LocalGroup>(world);
  std::vector<Comm*> cs;
  auto fail = [&](const char* what, cudaError_t e) {
    set_error("%s failed: %s", what, cudaGetErrorString(e));
    for (Comm* c : cs) {
      for (void* p : {(void*)c->sym, (void*)c->flags, (void*)c->epoch, (void*)c->psym_d, (void*)c->pflags_d})
        if (p) cudaFree(p);
      delete c;
    }
    return TS_ECUDA;
  };
  const size_t slot = (size_t)vec_capacity + kArScalars;
  cudaError_t e;
  for (int r = 0; r < world; ++r) {
    DeviceGuard rg(dev[r]);
    Comm* c = new Comm();
    cs.push_back(c);
    c->dev = dev[r];
    c->rank = r;
    c->world = world;
    c->vec_cap = (size_t)vec_capacity;
    c->local = grp;
    if ((e = cudaMalloc(&c->sym, 2 * slot * sizeof(double))) != cudaSuccess) return fail("cudaMalloc(sym)", e);
    if ((e = cudaMalloc(&c->flags, 256)) != cudaSuccess) return fail("cudaMalloc(flags)", e);
    if ((e = cudaMalloc(&c->epoch, sizeof(unsigned long long))) != cudaSuccess) return fail("cudaMalloc(epoch)", e);
    cudaMemset(c->sym, 0, 2 * slot * sizeof(double));
    cudaMemset(c->flags, 0, 256);
    cudaMemset(c->epoch, 0, sizeof(unsigned long long));
    if ((e = cudaEventCreateWithFlags(&grp->ev[r], cudaEventDisableTiming)) != cudaSuccess)
      return fail("cudaEventCreate", e);
  }
  std::vector<double*> psym(world);
  std::vector<unsigned long long*> pflags(world);
  for (int r = 0; r < world; ++r) {
    psym[r] = cs[r]->sym;
    pflags[r] = cs[r]->flags;
  }
  for (Comm* c : cs) {
    DeviceGuard rg(c->dev);
    if ((e = cudaMalloc(&c->psym_d, world * sizeof(double*))) != cudaSuccess) return fail("cudaMalloc", e);
    if ((e = cudaMalloc(&c->pflags_d, world * sizeof(unsigned long long*))) != cudaSuccess)
      return fail("cudaMalloc", e);
    cudaMemcpy(c->psym_d, psym.data(), world * sizeof(double*), cudaMemcpyHostToDevice);
    cudaMemcpy(c->pflags_d, pflags.data(), world * sizeof(unsigned long long*), cudaMemcpyHostToDevice);
  }
  for (Comm* c : cs) {
    DeviceGuard rg(c->dev);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail("comm init", e);
  }
  for (int r = 0; r < world; ++r) out[r] = reinterpret_cast<ts_comm*>(cs[r]);
  return 0;
}

int ts_comm_connect(ts_comm* h, const void* all_handles) {
  StructShared structural;
  Comm* c = reinterpret_cast<Comm*>(h);
  if (!c || !all_handles) TS_INVAL("null argument");
  DeviceGuard g(c->dev);
  std::vector<double*> psym(c->world);
  std::vector<unsigned long long*> pflags(c->world);
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) {
      psym[q] = c->sym;
      pflags[q] = c->flags;
      continue;
    }
    cudaIpcMemHandle_t hs, hf;
    memcpy(&hs, static_cast<const char*>(all_handles) + 128 * q, sizeof(hs));
    memcpy(&hf, static_cast<const char*>(all_handles) + 128 * q + 64, sizeof(hf));
    void *ps = nullptr, *pf = nullptr;
    TS_CUDA(cudaIpcOpenMemHandle(&ps, hs, cudaIpcMemLazyEnablePeerAccess));
    c->opened.push_back(ps);
    TS_CUDA(cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess));
    c->opened.push_back(pf);
    psym[q] = static_cast<double*>(ps);
    pflags[q] = static_cast<unsigned long long*>(pf);
  }
  TS_CUDA(cudaMalloc(&c->psym_d, c->world * sizeof(double*)));
  TS_CUDA(cudaMalloc(&c->pflags_d, c->world * sizeof(unsigned long long*)));
  TS_CUDA(cudaMemcpy(c->psym_d, psym.data(), c->world * sizeof(double*), cudaMemcpyHostToDevice));
  TS_CUDA(cudaMemcpy(c->pflags_d, pflags.data(), c->world * sizeof(unsigned long long*),
                     cudaMemcpyHostToDevice));
  return 0;
}

int ts_comm_destroy(ts_comm* h) {
  StructShared structural;
  Comm* c = reinterpret_cast<Comm*>(h);
  if (!c) return 0;
  DeviceGuard g(c->dev);
  cudaDeviceSynchronize();
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  for (void* p : {(void*)c->sym, (void*)c->flags, (void*)c->epoch, (void*)c->psym_d,
                  (void*)c->pflags_d})
    if (p) cudaFree(p);
  delete c;
  return 0;
}

int ts_matrix_set_shard(ts_matrix* A, ts_comm* h, int64_t n_global, int64_t col_offset,
                        double fro_global) {
  TS_CHECK_HANDLE(A);
  Comm* c = reinterpret_cast<Comm*>(h);
  if (c && c->dev != A->dev) TS_INVAL("communicator and matrix live on different devices");
  if (c && (col_offset < 0 || col_offset + A->n > n_global))
    TS_INVAL("shard columns [%lld, %lld) outside 0..%lld", (long long)col_offset,
             (long long)(col_offset + A->n), (long long)n_global);
  if (c && A->m > (int64_t)c->vec_cap) TS_INVAL("communicator vector capacity below m");
  destroy_instances(A);  // instances bake the (un)sharded kernel sequence
  A->comm = c;
  A->n_global = c ? n_global : A->n;
  A->m_global = A->m;
  A->col_off = c ? col_offset : 0;
  A->row_off = 0;
  A->row_shard = 0;
  A->tall_shard = 0;
  if (c) A->fro = fro_global;
  return 0;
}

int ts_matrix_set_tall_shard(ts_matrix* A, ts_comm* h, int64_t m_global, int64_t row_offset,
                             double fro_global) {
  TS_CHECK_HANDLE(A);
  Comm* c = reinterpret_cast<Comm*>(h);
  if (!c) TS_INVAL("row sharding needs a communicator");
  if (c->dev != A->dev) TS_INVAL("communicator and matrix live on different devices");
  if (A->halo) TS_INVAL("a halo (banded) row block takes ts_matrix_set_row_shard");
  if (row_offset < 0 || row_offset + A->m > m_global)
    TS_INVAL("shard rows [%lld, %lld) outside 0..%lld", (long long)row_offset,
             (long long)(row_offset + A->m), (long long)m_global);
  if (A->n > (int64_t)c->vec_cap) TS_INVAL("communicator vector capacity below n");
  destroy_instances(A);
  A->comm = c;
  A->tall_shard = 1;
  A->row_shard = 0;
  A->m_global = m_global;
  A->n_global = A->n;
  A->row_off = row_offset;
  A->col_off = 0;
  A->fro = fro_global;
  return 0;
}

int ts_matrix_set_row_shard(ts_matrix* A, ts_comm* h, int64_t n_global, int64_t row_offset,
                            double fro_global) {
  TS_CHECK_HANDLE(A);
  Comm* c = reinterpret_cast<Comm*>(h);
  if (!c) TS_INVAL("row sharding needs a communicator");
  if (c->dev != A->dev) TS_INVAL("communicator and matrix live on different devices");
  if (A->kind != 1 || A->m != A->n) TS_INVAL("row sharding takes a square local CSR block");
  if (row_offset < 0 || row_offset + A->m > n_global)
    TS_INVAL("shard rows [%lld, %lld) outside 0..%lld", (long long)row_offset,
             (long long)(row_offset + A->m), (long long)n_global);
  if (A->halo > A->m) TS_INVAL("halo (%lld) wider than the local block (%lld)", (long long)A->halo,
                               (long long)A->m);
  if (2 * A->halo > (int64_t)c->vec_cap) TS_INVAL("communicator vector capacity below 2 * halo");
  destroy_instances(A);
  A->comm = c;
  A->row_shard = 1;
  A->tall_shard = 0;
  A->n_global = n_global;
  A->m_global = n_global;
  A->row_off = row_offset;
  A->col_off = row_offset;
  A->fro = fro_global;
  return 0;
}

int ts_time_pass(const ts_matrix* A, int32_t trans, int32_t reps, double* avg_ms, void* stream) {
  TS_CHECK_HANDLE(A);
  if (reps < 1) TS_INVAL("reps must be positive");
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  float ms = 0.f;
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk, A->npart));
    double *dx, *dy;
    const int64_t nin = trans ? A->m : A->n, nout = trans ? A->n : A->m;
    TS_CHECK(ar.get(&dx, nin));
    TS_CHECK(ar.get(&dy, nout));
    TS_CUDA(cudaMemsetAsync(dx, 0, nin * sizeof(double), st));
    EpiStore e;
    e.y = dy;
    TS_CHECK(pass(*A, trans, dx, XS{}, e, wk, st));  // warm-up
    cudaEvent_t e0, e1;
    TS_CUDA(cudaEventCreate(&e0));
    TS_CUDA(cudaEventCreate(&e1));
    TS_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; ++i) TS_CHECK(pass(*A, trans, dx, XS{}, e, wk, st));
    TS_CUDA(cudaEventRecord(e1, st));
    TS_CUDA(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  *avg_ms = ms / reps;
  return 0;
}

int ts_cta_solve(const ts_matrix* A, const double* b, const ts_cta_options* o, double* x_out,
                 ts_trace_row* trace, int64_t trace_cap, ts_result* res, void* stream) {
  TS_CHECK_HANDLE(A);
  if (!o || !res || !b) TS_INVAL("null argument");
  if (!(o->epsilon > 0.0 && o->epsilon < 1.0)) TS_INVAL("epsilon must lie in (0, 1)");
  if (o->t_max < 1) TS_INVAL("t_max must be at least 1");
  if (o->h_mode != 0 && o->h_mode != 1) TS_INVAL("unknown h_mode");
  int t_max = (int)std::min<int64_t>(o->t_max, A->m);
  if (t_max > kTMax) TS_INVAL("t_max=%d exceeds the device limit %d", t_max, kTMax);
  if (o->h_mode == 1 && A->m != A->n && !o->normal_operand)
    TS_INVAL("symmetric mode requires a square matrix");
  if (o->h_mode == 1 && A->comm) TS_INVAL("symmetric mode is not supported on a column-sharded matrix");
  if (o->normal_operand && A->comm) TS_INVAL("the normal operand A^T A is not supported on a sharded matrix");
  if (o->normal_operand) t_max = (int)std::min<int64_t>(o->t_max, A->n);
  if (t_max > kTMax) TS_INVAL("t_max=%d exceeds the device limit %d", t_max, kTMax);
  memset(res, 0, sizeof(*res));
  DeviceGuard g(A->dev);
  CtaArgs a;
  a.epsilon = o->epsilon;
  a.t_max = t_max;
  a.gram = o->h_mode == 0;
  a.max_iters = o->max_iters;
  a.known_solvable = o->known_solvable;
  a.recheck_every = o->recheck_every;
  a.rcond = o->rcond;
  a.accelerate = o->accelerate;
  a.accel_patience = o->accel_patience;
  a.accel_ratio = o->accel_ratio;
  a.x_start = o->x_start;
  a.enhanced = (o->enhanced && !o->known_solvable) ? 1 : 0;  // centering.py:306
  a.normal = o->normal_operand ? 1 : 0;
  return cta_solve(*A, b, a, x_out, trace, trace_cap, res, (cudaStream_t)stream);
}

int ts_ta_adaptive(const ts_matrix* A, const double* b, const ts_ta_options* o, double* x_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                   void* stream) {
  TS_CHECK_HANDLE(A);
  if (!o || !res || !b) TS_INVAL("null argument");
  memset(res, 0, sizeof(*res));
  DeviceGuard g(A->dev);
  if (A->comm && o->gram) TS_INVAL("the Gram pair is not supported on a column-sharded matrix");
  TaArgs a;
  a.mode = MODE_ADAPTIVE;
  a.gram = o->gram ? 1 : 0;
  a.eps = o->eps;
  a.eps_prime = o->eps_prime;
  a.rho_cap = o->rho_cap;
  a.max_iters = o->max_iters;
  a.halvings = o->restart_halvings;
  a.x0 = o->x0;
  return ta_solve(*A, b, a, x_out, nullptr, trace, trace_cap, res, (cudaStream_t)stream);
}

int ts_ta_in_ball(const ts_matrix* A, const double* b, const ts_ball_options* o, double* x_out,
                  double* b_prime_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                  void* stream) {
  TS_CHECK_HANDLE(A);
  if (!o || !res || !b) TS_INVAL("null argument");
  if (!(o->rho > 0.0)) TS_INVAL("rho must be positive");
  memset(res, 0, sizeof(*res));
  DeviceGuard g(A->dev);
  if (A->comm && o->gram) TS_INVAL("the Gram pair is not supported on a column-sharded matrix");
  TaArgs a;
  a.mode = MODE_BALL;
  a.gram = o->gram ? 1 : 0;
  a.eps = o->eps;
  a.eps_prime = o->eps_prime;
  a.rho = o->rho;
  a.max_iters = o->max_iters;
  a.x0 = o->x0;
  const int rc = ta_solve(*A, b, a, x_out, b_prime_out, trace, trace_cap, res, (cudaStream_t)stream);
  if (!rc && res->trivial) TS_INVAL("b must be nonzero");
  return rc;
}

int ts_lp_feasibility(const ts_matrix* A, const double* b, const ts_lp_options* o, double* x_out,
                      ts_trace_row* trace, int64_t trace_cap, ts_result* res, void* stream) {
  TS_CHECK_HANDLE(A);
  if (!o || !res || !b) TS_INVAL("null argument");
  if (o->rho_max >= 0.0 && !(o->rho_max > 0.0)) TS_INVAL("rho_max must be positive");
  memset(res, 0, sizeof(*res));
  DeviceGuard g(A->dev);
  if (A->comm && o->gram) TS_INVAL("the Gram pair is not supported on a column-sharded matrix");
  TaArgs a;
  a.mode = MODE_LP;
  a.gram = o->gram ? 1 : 0;
  a.eps = o->eps;
  a.rho_max = o->rho_max;
  a.max_iters = o->max_iters;
  const int rc = ta_solve(*A, b, a, x_out, nullptr, trace, trace_cap, res, (cudaStream_t)stream);
  if (!rc && res->trivial) TS_INVAL("b must be nonzero");
  return rc;
}

}  // extern "C"
