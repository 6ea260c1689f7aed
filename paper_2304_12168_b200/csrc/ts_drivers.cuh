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
  TS_CUDA(cudaStreamBeginCaptureToGraph(cap, g, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeThreadLocal));
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

static SolveState* pinned_state() {
  static thread_local SolveState* hs = nullptr;
  if (!hs) {
    if (cudaHostAlloc(&hs, sizeof(SolveState) + 64, cudaHostAllocDefault) != cudaSuccess) {
      hs = nullptr;
    }
  }
  return hs;
}

struct SolveCtx {
  const Mat& M;
  cudaStream_t st;
  Arena ar;
  Work wk;
  SolveState* ds = nullptr;
  SolveState* hs = nullptr;
  long long* hflushed = nullptr;
  ts_trace_row* dtrace = nullptr;
  int seg_cap = 1;
  ts_trace_row* utrace = nullptr;
  int64_t ucap = 0;
  long long flushed = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  long long direct = 0, body_kernels = 0, l_start = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  SolveCtx(const Mat& m, cudaStream_t s) : M(m), st(s), ar(s) {}
  ~SolveCtx() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (cap) cudaStreamDestroy(cap);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }

  int init(SolveState& init_state, int64_t max_iters, ts_trace_row* trace, int64_t trace_cap) {
    l_start = g_launches;
    hs = pinned_state();
    if (!hs) {
      set_error("cudaHostAlloc for the solve state failed");
      return TS_ENOMEM;
    }
    hflushed = reinterpret_cast<long long*>(reinterpret_cast<char*>(hs) + sizeof(SolveState));
    TS_CHECK(make_work(ar, work_blocks(M.sms), &wk));
    TS_CHECK(ar.get(&ds, 1));
    long long want = max_iters + 2;
    if (want < 16) want = 16;
    seg_cap = (int)std::min<long long>(want, 8192);
    TS_CHECK(ar.get(&dtrace, (size_t)seg_cap));
    utrace = trace;
    ucap = trace ? trace_cap : 0;
    init_state.trace = dtrace;
    init_state.seg_cap = seg_cap;
    for (int i = 0; i < 4; ++i) init_state.kt[i] = KTimer{~0ull, 0ull, 0, 0};
    *hs = init_state;
    TS_CUDA(cudaMemcpyAsync(ds, hs, sizeof(SolveState), cudaMemcpyHostToDevice, st));
    TS_CUDA(cudaEventCreate(&ev0));
    TS_CUDA(cudaEventCreate(&ev1));
    TS_CUDA(cudaEventRecord(ev0, st));
    return 0;
  }

  int read_state() {
    TS_CUDA(cudaMemcpyAsync(hs, ds, sizeof(SolveState), cudaMemcpyDeviceToHost, st));
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("device failure during solve: %s", cudaGetErrorString(e));
      return TS_ECUDA;
    }
    return 0;
  }

  int flush() {
    const long long upto = hs->trace_count;
    while (flushed < upto) {
      const long long ring = flushed % seg_cap;
      long long chunk = std::min<long long>(upto - flushed, seg_cap - ring);
      if (flushed < ucap) {
        const long long n = std::min<long long>(chunk, ucap - flushed);
        TS_CUDA(cudaMemcpyAsync(utrace + flushed, dtrace + ring, n * sizeof(ts_trace_row),
                                cudaMemcpyDefault, st));
      }
      flushed += chunk;
    }
    *hflushed = flushed;
    TS_CUDA(cudaMemcpyAsync(&ds->trace_flushed, hflushed, sizeof(long long),
                            cudaMemcpyHostToDevice, st));
    TS_CUDA(cudaStreamSynchronize(st));  // hflushed / ring reuse
    return 0;
  }

  int build(const GraphFn& gbody) {
    TS_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    TS_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    TS_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
    cudaGraph_t bodyg = np.conditional.phGraph_out[0];
    TS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    const long long l0 = g_launches;
    TS_CHECK(gbody(bodyg, h, cap));
    body_kernels = g_launches - l0;  // captured once (per-trip count is derived on device)
    TS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    return 0;
  }

  int run(const BodyFn& body, const GraphFn& gbody,
          const std::function<int(cudaStream_t)>& maint) {
    TS_CHECK(read_state());
    TS_CHECK(flush());
    static const bool no_graph = getenv("TS_NO_GRAPH") != nullptr;
    while (hs->status == TS_RUNNING) {
      if (hs->maint != MAINT_NONE) {
        TS_CHECK(maint(st));
      } else if (!no_graph) {
        if (!exec) TS_CHECK(build(gbody));
        TS_CUDA(cudaGraphLaunch(exec, st));
      } else {
        TS_CHECK(body(st));
      }
      TS_CHECK(read_state());
      TS_CHECK(flush());
    }
    return 0;
  }

  int finish_timing(ts_result* res) {
    TS_CUDA(cudaEventRecord(ev1, st));
    TS_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    res->elapsed_ms = ms;
    // direct launches counted on the host; graph-executed kernels counted on
    // the device (every pass / scalar kernel bumps its class counter)
    res->kernel_launches = hs->launches;  // every solver kernel bumps it on the device
    return 0;
  }
};

// count every launch we enqueue (graph bodies are counted once at capture)
template <class Epi>
static int pass(const Mat& M, int trans, const double* x, XS xs, const Epi& e, const Work& w,
                cudaStream_t s) {
  ++g_launches;
  if constexpr (std::is_base_of<EpiBase, Epi>::value) {
    Epi e2 = e;
    e2.tclass = trans ? 1 : 0;
    return launch_pass(M, trans, x, xs, e2, w, s);
  } else {
    return launch_pass(M, trans, x, xs, e, w, s);
  }
}
template <class Epi>
static int vecpass(const Mat& M, int64_t len, const Epi& e, const Work& w, cudaStream_t s) {
  ++g_launches;
  if constexpr (std::is_base_of<EpiBase, Epi>::value) {
    Epi e2 = e;
    e2.tclass = 2;
    return launch_vec(len, M.sms, e2, w, s);
  } else {
    return launch_vec(len, M.sms, e, w, s);
  }
}

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

static int ta_solve(const Mat& M, const double* b_in, const TaArgs& a, double* x_out,
                    double* bp_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                    cudaStream_t st) {
  const int64_t mo = a.gram ? M.n : M.m;  // operator rows (TA's b-space)
  const int64_t no = M.n;                 // operator cols (x-space)
  const int64_t mx = std::max(mo, no);
  SolveCtx c(M, st);
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
  s0.m_rows = mo;
  s0.n_cols = no;
  s0.x_min = 0.0;
  s0.lower_bound = 0.0;
  TS_CHECK(c.init(s0, a.max_iters, trace, trace_cap));
  Arena& ar = c.ar;
  double *b, *bp, *gap, *d, *x, *cv, *fr, *t1 = nullptr, *x0 = nullptr;
  TS_CHECK(stage_in(ar, b_in, mo, &b));
  TS_CHECK(ar.get(&bp, mo));
  TS_CHECK(ar.get(&gap, mo));
  TS_CHECK(ar.get(&d, mo));
  TS_CHECK(ar.get(&fr, mo));
  TS_CHECK(ar.get(&x, no));
  TS_CHECK(ar.get(&cv, no));
  if (a.gram) TS_CHECK(ar.get(&t1, M.m));
  if (a.x0) TS_CHECK(stage_in(ar, a.x0, no, &x0));
  SolveState* ds = c.ds;
  const Work& wk = c.wk;
  const int relu = a.mode == MODE_LP;

  // operator products with fused epilogue: y = Op v  (Op = A, or A^T A)
  auto op_apply = [&](cudaStream_t s, const double* v, XS xs, auto epi, int pred) -> int {
    if (!a.gram) return pass(M, 0, v, xs, epi, wk, s);
    EpiStore es;
    es.st = ds; es.y = t1; es.pred = pred;
    TS_CHECK(pass(M, 0, v, xs, es, wk, s));
    return pass(M, 1, t1, XS{}, epi, wk, s);
  };
  auto op_apply_t = [&](cudaStream_t s, const double* v, auto epi, int pred) -> int {
    if (!a.gram) return pass(M, 1, v, XS{}, epi, wk, s);
    EpiStore es;
    es.st = ds; es.y = t1; es.pred = pred;
    TS_CHECK(pass(M, 0, v, XS{}, es, wk, s));
    return pass(M, 1, t1, XS{}, epi, wk, s);
  };

  // ---- init
  if (x0) {
    EpiNormTo en;
    en.st = ds; en.use_cond = 0; en.v = x0; en.len = no; en.what = 0;
    TS_CHECK(vecpass(M, no, en, wk, st));
    EpiCopyWarm ec;
    ec.st = ds; ec.use_cond = 0; ec.src = x0; ec.dst = x;
    TS_CHECK(vecpass(M, no, ec, wk, st));
    EpiTaBp eb;
    eb.st = ds; eb.use_cond = 0; eb.b = b; eb.bp = bp; eb.gap = gap; eb.kind = 0;
    TS_CHECK(op_apply(st, x, XS{}, eb, 0));
  } else {
    EpiTaInitZero ez;
    ez.st = ds; ez.use_cond = 0; ez.b = b; ez.bp = bp; ez.gap = gap; ez.x = x; ez.m = mo; ez.n = no;
    TS_CHECK(vecpass(M, mx, ez, wk, st));
  }

  // one TA iteration: c = Op^T gap (finisher decides pivot / expand / stop)
  auto c_pass = [&](cudaStream_t s, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hsw,
                    int use) -> int {
    EpiTaC ec;
    ec.st = ds; ec.c = cv; ec.cond = hw; ec.use_cond = use; ec.sw = hsw; ec.use_sw = use;
    return op_apply_t(s, gap, ec, 1);
  };
  // pivot: v = Op pre (fused d.d, gap.d), then the convex-combination update
  auto pivot = [&](cudaStream_t s, cudaGraphConditionalHandle hw, int use) -> int {
    EpiTaV ev;
    ev.st = ds; ev.bp = bp; ev.gap = gap; ev.d = d;
    XS xs;
    xs.sp = &ds->scale;
    xs.relu = relu;
    TS_CHECK(op_apply(s, cv, xs, ev, 2));
    EpiTaUpd eu;
    eu.st = ds; eu.cond = hw; eu.use_cond = use;
    eu.b = b; eu.d = d; eu.c = cv; eu.bp = bp; eu.gap = gap; eu.x = x; eu.m = mo; eu.n = no;
    eu.relu = relu;
    return vecpass(M, mx, eu, wk, s);
  };
  BodyFn body = [&](cudaStream_t s) -> int {
    TS_CHECK(c_pass(s, 0, 0, 0));
    return pivot(s, 0, 0);
  };
  // graph body: [c pass] -> SWITCH{0: pivot}  (expand / stop select no case)
  GraphFn gbody = [&](cudaGraph_t bodyg, cudaGraphConditionalHandle hw, cudaStream_t cap) -> int {
    cudaGraphConditionalHandle hsw;
    TS_CUDA(cudaGraphConditionalHandleCreate(&hsw, bodyg, 0, 0));
    cudaGraph_t* cases = nullptr;
    TS_CHECK(capture_into(cap, bodyg, [&](cudaStream_t s) -> int {
      TS_CHECK(c_pass(s, hw, hsw, 1));
      return capture_switch(s, hsw, 1, &cases);
    }));
    return capture_into(cap, cases[0], [&](cudaStream_t s) -> int { return pivot(s, hw, 1); });
  };
  auto maint = [&](cudaStream_t s) -> int {
    EpiTaBp eb;
    eb.st = ds; eb.b = b; eb.bp = bp; eb.gap = gap; eb.kind = 1;
    return op_apply(s, x, XS{}, eb, 0);
  };
  TS_CHECK(c.run(body, gbody, maint));
  if (c.hs->error == TS_EDEGENERATE) {
    set_error("degenerate pivot: v coincides with the iterate");
    return TS_EDEGENERATE;
  }
  if (c.hs->trivial) {
    TS_CUDA(cudaMemsetAsync(x, 0, no * sizeof(double), st));
  } else {
    EpiFinalR efr;
    efr.st = ds; efr.use_cond = 0; efr.b = b; efr.fr = fr;
    TS_CHECK(op_apply(st, x, XS{}, efr, 0));
    EpiFinalNR enr;
    enr.st = ds; enr.use_cond = 0; enr.out = nullptr;
    TS_CHECK(op_apply_t(st, fr, enr, 0));
  }
  TS_CHECK(c.read_state());
  if (x_out) TS_CUDA(cudaMemcpyAsync(x_out, x, no * sizeof(double), cudaMemcpyDefault, st));
  if (bp_out) TS_CUDA(cudaMemcpyAsync(bp_out, bp, mo * sizeof(double), cudaMemcpyDefault, st));
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
};

struct CtaBuffers {
  double *b = nullptr, *x = nullptr, *fr = nullptr, *xs = nullptr;
  KrylovPtrs kp;
};

static int cta_alloc(Arena& ar, const Mat& M, int t_max, int gram, CtaBuffers* B) {
  memset(&B->kp, 0, sizeof(B->kp));
  for (int i = 0; i <= t_max; ++i) TS_CHECK(ar.get(&B->kp.p[i], M.m));
  if (gram)
    for (int i = 0; i < t_max; ++i) TS_CHECK(ar.get(&B->kp.q[i], M.n));
  TS_CHECK(ar.get(&B->x, M.n));
  TS_CHECK(ar.get(&B->fr, M.m));
  return 0;
}

// moments pairs for orders 1..npairs (predicated on state t); `solve_last`
// makes the pair that equals the state's t run the Hankel solves
static int cta_pairs(const Mat& M, SolveState* ds, const Work& wk, const CtaBuffers& B, int npairs,
                     int gram, int solve_last, cudaStream_t s) {
  for (int i = 1; i <= npairs; ++i) {
    if (gram) {
      EpiCtaQ eq;
      eq.st = ds; eq.q = B.kp.q[i - 1]; eq.i = i;
      TS_CHECK(pass(M, 1, B.kp.p[i - 1], XS{}, eq, wk, s));
      EpiCtaP ep;
      ep.st = ds; ep.pprev = B.kp.p[i - 1]; ep.p = B.kp.p[i]; ep.i = i; ep.with_solve = solve_last;
      TS_CHECK(pass(M, 0, B.kp.q[i - 1], XS{}, ep, wk, s));
    } else {
      EpiCtaP ep;
      ep.st = ds; ep.pprev = B.kp.p[i - 1]; ep.p = B.kp.p[i]; ep.i = i; ep.with_solve = solve_last;
      TS_CHECK(pass(M, 0, B.kp.p[i - 1], XS{}, ep, wk, s));
    }
  }
  return 0;
}

// one CTA step of at most `npairs` pairs: moments (+ Hankel in the last pair's
// finisher), candidate norms / retry rule, fused r / x update (tail)
static int cta_step_kernels(const Mat& M, SolveState* ds, const Work& wk, const CtaBuffers& B,
                            int npairs, int gram, cudaStream_t s, cudaGraphConditionalHandle h,
                            int use) {
  TS_CHECK(cta_pairs(M, ds, wk, B, npairs, gram, 1, s));
  EpiCtaCand ecd;
  ecd.st = ds; ecd.kp = B.kp; ecd.m = M.m;
  TS_CHECK(vecpass(M, M.m, ecd, wk, s));
  EpiCtaUpd eu;
  eu.st = ds; eu.cond = h; eu.use_cond = use; eu.kp = B.kp; eu.x = B.x; eu.m = M.m; eu.n = M.n;
  eu.gram = gram;
  return vecpass(M, std::max(M.m, M.n), eu, wk, s);
}

static int cta_solve(const Mat& M, const double* b_in, const CtaArgs& a, double* x_out,
                     ts_trace_row* trace, int64_t trace_cap, ts_result* res, cudaStream_t st) {
  SolveCtx c(M, st);
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
  s0.a_fro = M.fro;
  s0.m_rows = M.m;
  s0.n_cols = M.n;
  s0.warm = 1;
  TS_CHECK(c.init(s0, a.max_iters, trace, trace_cap));
  Arena& ar = c.ar;
  CtaBuffers B;
  TS_CHECK(stage_in(ar, b_in, M.m, &B.b));
  TS_CHECK(cta_alloc(ar, M, a.t_max, a.gram, &B));
  SolveState* ds = c.ds;
  const Work& wk = c.wk;
  if (a.x_start) {
    TS_CHECK(stage_in(ar, a.x_start, M.n, &B.xs));
    EpiCopyWarm ec;
    ec.st = ds; ec.use_cond = 0; ec.src = B.xs; ec.dst = B.x;
    TS_CHECK(vecpass(M, M.n, ec, wk, st));
    EpiCtaInitR ei;
    ei.st = ds; ei.use_cond = 0; ei.b = B.b; ei.r = B.kp.p[0];
    TS_CHECK(pass(M, 0, B.x, XS{}, ei, wk, st));
  } else {
    EpiCtaInit ei;
    ei.st = ds; ei.use_cond = 0; ei.b = B.b; ei.r = B.kp.p[0]; ei.x = B.x; ei.m = M.m; ei.n = M.n;
    TS_CHECK(vecpass(M, std::max(M.m, M.n), ei, wk, st));
  }
  BodyFn body = [&](cudaStream_t s) -> int {
    return cta_step_kernels(M, ds, wk, B, a.t_max, a.gram, s, 0, 0);
  };
  // graph body: [head: switch = t - 1] -> SWITCH{order 1 .. t_max}: each case
  // launches exactly its t pairs + candidate + update
  GraphFn gbody = [&](cudaGraph_t bodyg, cudaGraphConditionalHandle hw, cudaStream_t cap) -> int {
    cudaGraphConditionalHandle hsw;
    TS_CUDA(cudaGraphConditionalHandleCreate(&hsw, bodyg, 0, 0));
    cudaGraph_t* cases = nullptr;
    TS_CHECK(capture_into(cap, bodyg, [&](cudaStream_t s) -> int {
      ++g_launches;
      k_cta_head<<<1, 32, 0, s>>>(ds, hsw, a.t_max);
      TS_CUDA(cudaGetLastError());
      return capture_switch(s, hsw, a.t_max, &cases);
    }));
    for (int k = 0; k < a.t_max; ++k)
      TS_CHECK(capture_into(cap, cases[k], [&](cudaStream_t s) -> int {
        return cta_step_kernels(M, ds, wk, B, k + 1, a.gram, s, hw, 1);
      }));
    return 0;
  };
  auto maint = [&](cudaStream_t s) -> int {
    EpiNormTo en;
    en.st = ds; en.v = B.x; en.len = M.n; en.what = 1;
    TS_CHECK(vecpass(M, M.n, en, wk, s));
    EpiCtaRecheck er;
    er.st = ds; er.b = B.b; er.r = B.kp.p[0];
    return pass(M, 0, B.x, XS{}, er, wk, s);
  };
  TS_CHECK(c.run(body, gbody, maint));
  if (!c.hs->trivial) {
    EpiFinalR efr;
    efr.st = ds; efr.use_cond = 0; efr.b = B.b; efr.fr = B.fr;
    TS_CHECK(pass(M, 0, B.x, XS{}, efr, wk, st));
    EpiFinalNR enr;
    enr.st = ds; enr.use_cond = 0; enr.out = nullptr;
    TS_CHECK(pass(M, 1, B.fr, XS{}, enr, wk, st));
  }
  TS_CHECK(c.read_state());
  if (x_out) TS_CUDA(cudaMemcpyAsync(x_out, B.x, M.n * sizeof(double), cudaMemcpyDefault, st));
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

int ts_matvec(const ts_matrix* A, const double* x, double* y, void* stream) {
  TS_CHECK_HANDLE(A);
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk));
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
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk));
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
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  {
    Arena ar(st);
    Work wk;
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk));
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
  if (t < 1 || t > kTMax || t > A->m) TS_INVAL("order t=%d outside 1..%lld", t, (long long)std::min<int64_t>(A->m, kTMax));
  if (h_mode == 1 && A->m != A->n) TS_INVAL("symmetric mode requires a square matrix");
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int gram = h_mode == 0;
  {
    SolveCtx c(*A, st);
    SolveState s0;
    memset(&s0, 0, sizeof(s0));
    s0.mode = MODE_CTA;
    s0.t = t;
    s0.gram = gram;
    TS_CHECK(c.init(s0, 16, nullptr, 0));
    CtaBuffers B;
    TS_CHECK(cta_alloc(c.ar, *A, t, gram, &B));
    TS_CUDA(cudaMemcpyAsync(B.kp.p[0], r, A->m * sizeof(double), cudaMemcpyDefault, st));
    TS_CHECK(cta_pairs(*A, c.ds, c.wk, B, t, gram, 0, st));
    TS_CHECK(c.read_state());
    memcpy(phi, c.hs->phi, 2 * t * sizeof(double));
    if (krylov)
      for (int i = 0; i <= t; ++i)
        TS_CUDA(cudaMemcpyAsync(krylov + (size_t)i * A->m, B.kp.p[i], A->m * sizeof(double),
                                cudaMemcpyDefault, st));
    if (transposed && gram)
      for (int i = 0; i < t; ++i)
        TS_CUDA(cudaMemcpyAsync(transposed + (size_t)i * A->n, B.kp.q[i], A->n * sizeof(double),
                                cudaMemcpyDefault, st));
    TS_CUDA(cudaStreamSynchronize(st));
  }
  return 0;
}

int ts_cta_step(const ts_matrix* A, int32_t h_mode, const double* x, const double* r, int32_t t,
                double rcond, double* x_out, double* r_out, int32_t* order_out,
                double* atr_norm_out, int32_t* status_out, void* stream) {
  TS_CHECK_HANDLE(A);
  if (t < 1 || t > kTMax || t > A->m) TS_INVAL("order t=%d outside 1..%lld", t, (long long)std::min<int64_t>(A->m, kTMax));
  if (h_mode == 1 && A->m != A->n) TS_INVAL("symmetric mode requires a square matrix");
  DeviceGuard g(A->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int gram = h_mode == 0;
  {
    SolveCtx c(*A, st);
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
    TS_CHECK(c.init(s0, 16, nullptr, 0));
    CtaBuffers B;
    TS_CHECK(cta_alloc(c.ar, *A, t, gram, &B));
    TS_CUDA(cudaMemcpyAsync(B.kp.p[0], r, A->m * sizeof(double), cudaMemcpyDefault, st));
    TS_CUDA(cudaMemcpyAsync(B.x, x, A->n * sizeof(double), cudaMemcpyDefault, st));
    // r_norm for the monotone test
    double* rn;
    TS_CHECK(c.ar.get(&rn, 1));
    EpiDot e{B.kp.p[0], B.kp.p[0], &c.ds->r_norm, 1};
    TS_CHECK(vecpass(*A, A->m, e, c.wk, st));
    TS_CHECK(cta_step_kernels(*A, c.ds, c.wk, B, t, gram, st, 0, 0));
    TS_CHECK(c.read_state());
    const int nestatus = (c.hs->status == TS_NORMAL_EQ_SOLUTION) ? TS_NORMAL_EQ_SOLUTION : 0;
    if (c.hs->status == TS_NUMERICAL_FAILURE) {
      set_error("moment solve failed: SVD did not converge in Linear Least Squares");
      return TS_EINVAL;
    }
    if (status_out) *status_out = nestatus;
    if (!nestatus) {
      if (order_out) *order_out = c.hs->sel_order;
      if (atr_norm_out) *atr_norm_out = c.hs->atr_norm;
      if (x_out) TS_CUDA(cudaMemcpyAsync(x_out, B.x, A->n * sizeof(double), cudaMemcpyDefault, st));
      if (r_out)
        TS_CUDA(cudaMemcpyAsync(r_out, B.kp.p[0], A->m * sizeof(double), cudaMemcpyDefault, st));
    }
    TS_CUDA(cudaStreamSynchronize(st));
  }
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
    TS_CHECK(make_work(ar, work_blocks(A->sms), &wk));
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
  if (o->enhanced && !o->known_solvable)
    TS_INVAL("enhanced probe (first_order_probe) is not implemented on the device path");
  int t_max = (int)std::min<int64_t>(o->t_max, A->m);
  if (t_max > kTMax) TS_INVAL("t_max=%d exceeds the device limit %d", t_max, kTMax);
  if (o->h_mode == 1 && A->m != A->n) TS_INVAL("symmetric mode requires a square matrix");
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
  return cta_solve(*A, b, a, x_out, trace, trace_cap, res, (cudaStream_t)stream);
}

int ts_ta_adaptive(const ts_matrix* A, const double* b, const ts_ta_options* o, double* x_out, ts_trace_row* trace, int64_t trace_cap, ts_result* res,
                   void* stream) {
  TS_CHECK_HANDLE(A);
  if (!o || !res || !b) TS_INVAL("null argument");
  memset(res, 0, sizeof(*res));
  DeviceGuard g(A->dev);
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
