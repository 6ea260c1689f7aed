// Latency-bound pass chains (C3-like: tridiagonal n = 100001, everything
// L2-resident): what does one dependent "pass" cost — a pass = read the solver
// state, y = scale * A x, a deterministic grid-wide reduction of y.y, a
// finisher that writes the next state — under
//   (a) one kernel per pass inside a graph WHILE body (the library's model),
//       last-block finisher;
//   (b) the same with programmatic dependent launch: the matrix rows are
//       loaded before griddepcontrol.wait;
//   (c) one persistent kernel: block-resident rows, every block publishes its
//       partial + boundary entries under a per-block sequence flag and reads
//       ALL blocks' partials (one-stage all-gather, no last-block hop), every
//       block runs the finisher redundantly on its own copy of the state.
// Design study for the library's resident CTA loop; not part of the library.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/microbench/lat_chain tools/microbench/lat_chain.cu
#include <algorithm>
#include <cmath>
#include <cstdio>
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

constexpr int NT = 256;

struct Args {
  const double *lo, *di, *up;  // tridiagonal rows
  const double* x;
  double* y;
  double* bacc;
  unsigned* ticket;
  double* state;  // [0] scale for the next pass, [1] last y.y
  unsigned long long* trips;
  unsigned long long stop;
  cudaGraphConditionalHandle h;
  int n, pdl, use_cond;
};

__device__ __forceinline__ double block_sum(double v, double* sm) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) s += sm[i];
  return s;
}

template <int HEAVY>
__global__ void __launch_bounds__(NT) k_pass(Args A) {
  __shared__ double sm[NT / 32];
  __shared__ int last;
  if (A.pdl) asm volatile("griddepcontrol.launch_dependents;");
  const int P = gridDim.x * NT;
  const int i0 = blockIdx.x * NT + threadIdx.x;
  // independent of the previous pass: the matrix is immutable
  double lo[3], di[3], up[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int i = i0 + u * P;
    lo[u] = i < A.n ? __ldg(A.lo + i) : 0.0;
    di[u] = i < A.n ? __ldg(A.di + i) : 0.0;
    up[u] = i < A.n ? __ldg(A.up + i) : 0.0;
  }
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const double scale = __ldcg(A.state);
  double acc = 0;
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int i = i0 + u * P;
    if (i < A.n) {
      const double xm = i > 0 ? __ldcg(A.x + i - 1) : 0.0;
      const double xc = __ldcg(A.x + i);
      const double xp = i + 1 < A.n ? __ldcg(A.x + i + 1) : 0.0;
      const double v = (lo[u] * xm + di[u] * xc + up[u] * xp) * scale;
      A.y[i] = v;
      acc = fma(v, v, acc);
    }
  }
  const double bs = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    A.bacc[blockIdx.x] = bs;
    __threadfence();
    last = atomicAdd(A.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double t = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += NT) t += __ldcg(A.bacc + b);
    const double s = block_sum(t, sm);
    if (threadIdx.x == 0) {
      double f = s;
      if (HEAVY) {  // a serial finisher of a few hundred dependent flops (the Hankel solve)
        for (int k = 0; k < 200; ++k) f = sqrt(f * f + 1e-300);
      }
      A.state[1] = f;
      A.state[0] = 1.0 / sqrt(f / A.n);  // keeps |y| ~ 1
      *A.ticket = 0;
      if (A.use_cond) {
        const unsigned long long v = ++*A.trips;
        cudaGraphSetConditional(A.h, v < A.stop ? 1u : 0u);
      }
    }
  }
}

static void launch(cudaStream_t s, const Args& a, int P, int heavy) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(NT);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a.pdl ? at : nullptr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  if (heavy) CK(cudaLaunchKernelEx(&cfg, k_pass<1>, a));
  else CK(cudaLaunchKernelEx(&cfg, k_pass<0>, a));
}

// ------------------------------------------------------------ persistent ----
struct PArgs {
  const double *lo, *di, *up;
  double* x0;       // initial x (n)
  double* edge;     // [2][P][2] boundary entries of every block's piece, by pass parity
  double* part;     // [2][P] partials by pass parity
  unsigned* seq;    // [P] pass number published by each block
  double* state;    // out
  double* yout;     // final y (n)
  int n, passes, rows;  // rows per block
};

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// RPT rows per thread, rows of a block contiguous: row = b * rows + t * RPT + u
template <int RPT, int HEAVY>
__global__ void __launch_bounds__(NT, 1) k_persist(PArgs A) {
  __shared__ double sm[NT / 32];
  __shared__ double gat[1024];
  __shared__ double s_scale;
  __shared__ double xs[NT * RPT + 2];
  const int P = gridDim.x, b = blockIdx.x, t = threadIdx.x;
  const int r0 = b * A.rows;
  const int nr = min(A.rows, A.n - r0);
  double lo[RPT], di[RPT], up[RPT], xv[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int l = t * RPT + u;
    const bool ok = l < nr;
    lo[u] = ok ? A.lo[r0 + l] : 0.0;
    di[u] = ok ? A.di[r0 + l] : 0.0;
    up[u] = ok ? A.up[r0 + l] : 0.0;
    xv[u] = ok ? A.x0[r0 + l] : 0.0;
  }
  double xl = r0 > 0 ? A.x0[r0 - 1] : 0.0;                // left neighbour's last entry
  double xr = r0 + nr < A.n ? A.x0[r0 + nr] : 0.0;        // right neighbour's first entry
  double scale = 1.0;
  for (int pass = 1; pass <= A.passes; ++pass) {
    const int par = pass & 1;
    // stage x piece with halo
#pragma unroll
    for (int u = 0; u < RPT; ++u) xs[1 + t * RPT + u] = xv[u];
    if (t == 0) { xs[0] = xl; xs[1 + nr] = xr; }
    __syncthreads();
    double acc = 0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int l = t * RPT + u;
      if (l < nr) {
        const double v = (lo[u] * xs[l] + di[u] * xs[l + 1] + up[u] * xs[l + 2]) * scale;
        xv[u] = v;
        acc = fma(v, v, acc);
      }
    }
    const double bs = block_sum(acc, sm);
    // publish: boundary entries, partial, then the sequence flag
    if (t == 0) {
      A.part[par * P + b] = bs;
    }
    if (t * RPT == 0) A.edge[(par * P + b) * 2 + 0] = xv[0];
    {
      const int l = nr - 1;
      if (l / RPT == t) {
        double last = xv[0];
#pragma unroll
        for (int u = 0; u < RPT; ++u) if (u == l % RPT) last = xv[u];
        A.edge[(par * P + b) * 2 + 1] = last;
      }
    }
    __syncthreads();
    if (t == 0) {
      __threadfence();
      st_release(A.seq + b, (unsigned)pass);
    }
    // gather: thread q waits for block q
    for (int q = t; q < P; q += NT) {
      while (ld_acquire(A.seq + q) < (unsigned)pass) {}
      gat[q] = __ldcg(A.part + par * P + q);
    }
    if (t == 32 && b > 0) {
      while (ld_acquire(A.seq + b - 1) < (unsigned)pass) {}
      xl = __ldcg(A.edge + (par * P + b - 1) * 2 + 1);
      gat[1000] = xl;
    }
    if (t == 64 && b + 1 < P) {
      while (ld_acquire(A.seq + b + 1) < (unsigned)pass) {}
      xr = __ldcg(A.edge + (par * P + b + 1) * 2 + 0);
      gat[1001] = xr;
    }
    __syncthreads();
    // fixed-order sum of the P partials: warp 0, lane l adds q = l, l + 32, ...; then a tree
    if (t < 32) {
      double s = 0;
      for (int q = t; q < P; q += 32) s += gat[q];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (t == 0) {
        double f = s;
        if (HEAVY) {
          for (int k = 0; k < 200; ++k) f = sqrt(f * f + 1e-300);
        }
        s_scale = 1.0 / sqrt(f / A.n);
        if (b == 0) A.state[1] = f;
      }
    }
    __syncthreads();
    scale = s_scale;
    if (t == 0) {
      if (b > 0) xl = gat[1000];
      if (b + 1 < P) xr = gat[1001];
    }
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int l = t * RPT + u;
    if (l < nr) A.yout[r0 + l] = xv[u];
  }
}

int main() {
  const int n = 100001;
  std::vector<double> lo(n), di(n, 0.0), up(n), x(n, 1.0);
  for (int i = 0; i < n; ++i) {
    lo[i] = i > 0 ? sqrt((double)i * (n - i)) / (n / 2.0) : 0.0;
    up[i] = i + 1 < n ? sqrt((double)(i + 1) * (n - 1 - i)) / (n / 2.0) : 0.0;
    di[i] = 0.1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto up_ = [](const std::vector<double>& v) {
    double* p;
    CK(cudaMalloc(&p, v.size() * 8));
    CK(cudaMemcpy(p, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    return p;
  };
  double *dlo = up_(lo), *ddi = up_(di), *dup = up_(up), *x0 = up_(x), *x1 = up_(x);
  double *bacc, *state;
  unsigned* ticket;
  unsigned long long* trips;
  CK(cudaMalloc(&bacc, 4096 * 8));
  CK(cudaMalloc(&state, 16));
  CK(cudaMalloc(&ticket, 16));
  CK(cudaMalloc(&trips, 8));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int K = 8, REP = 500;
  for (int heavy = 0; heavy < 2; ++heavy)
    for (int P : {sms, (n + 3 * NT - 1) / (3 * NT)})
      for (int pdl = 0; pdl < 2; ++pdl) {
        Args a = {};
        a.lo = dlo; a.di = ddi; a.up = dup; a.bacc = bacc; a.ticket = ticket; a.state = state;
        a.trips = trips; a.n = n; a.pdl = pdl;
        const double st0[2] = {1.0, 0.0};
        CK(cudaMemcpy(state, st0, 16, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(x0, x.data(), n * 8, cudaMemcpyHostToDevice));
        CK(cudaMemset(ticket, 0, 16));
        cudaGraph_t wg;
        CK(cudaGraphCreate(&wg, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, wg, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, wg, nullptr, 0, &np));
        cudaGraph_t body = np.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal));
        for (int k = 0; k < K; ++k) {
          Args c = a;
          c.x = (k & 1) ? x1 : x0;
          c.y = (k & 1) ? x0 : x1;
          c.use_cond = k == K - 1;
          c.h = h;
          c.stop = REP;
          launch(s, c, P, heavy);
        }
        CK(cudaStreamEndCapture(s, &body));
        cudaGraphExec_t we;
        CK(cudaGraphInstantiate(&we, wg, 0));
        float ms = 0;
        for (int w = 0; w < 3; ++w) {
          CK(cudaMemset(trips, 0, 8));
          CK(cudaEventRecord(e0, s));
          CK(cudaGraphLaunch(we, s));
          CK(cudaEventRecord(e1, s));
          CK(cudaEventSynchronize(e1));
          cudaEventElapsedTime(&ms, e0, e1);
        }
        unsigned long long tr;
        CK(cudaMemcpy(&tr, trips, 8, cudaMemcpyDeviceToHost));
        double st[2];
        CK(cudaMemcpy(st, state, 16, cudaMemcpyDeviceToHost));
        printf("graph WHILE  heavy=%d P=%4d pdl=%d : %6.2f us/pass  (%llu trips, y.y %.17g)\n", heavy, P, pdl,
               ms * 1e3 / (tr * K), tr, st[1]);
        CK(cudaGraphExecDestroy(we));
        CK(cudaGraphDestroy(wg));
      }
  // per-trip cost of the conditional nodes: WHILE{K passes} for several K, and
  // WHILE{SWITCH{K passes}} (the case is re-selected by the last pass of a trip)
  for (int sw = 0; sw < 2; ++sw)
    for (int K2 : {1, 2, 4, 8, 16}) {
      const int P = sms, REP2 = 400;
      Args a = {};
      a.lo = dlo; a.di = ddi; a.up = dup; a.bacc = bacc; a.ticket = ticket; a.state = state;
      a.trips = trips; a.n = n; a.pdl = 0;
      const double st0[2] = {1.0, 0.0};
      CK(cudaMemcpy(state, st0, 16, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(x0, x.data(), n * 8, cudaMemcpyHostToDevice));
      CK(cudaMemset(ticket, 0, 16));
      cudaGraph_t wg;
      CK(cudaGraphCreate(&wg, 0));
      cudaGraphConditionalHandle h;
      CK(cudaGraphConditionalHandleCreate(&h, wg, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams np = {};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, wg, nullptr, 0, &np));
      cudaGraph_t body = np.conditional.phGraph_out[0];
      cudaGraph_t target = body;
      if (sw) {
        cudaGraphConditionalHandle hs;
        CK(cudaGraphConditionalHandleCreate(&hs, body, 0, cudaGraphCondAssignDefault));  // always case 0
        cudaGraphNodeParams sp = {};
        sp.type = cudaGraphNodeTypeConditional;
        sp.conditional.handle = hs;
        sp.conditional.type = cudaGraphCondTypeSwitch;
        sp.conditional.size = 2;
        cudaGraphNode_t sn;
        CK(cudaGraphAddNode(&sn, body, nullptr, 0, &sp));
        target = sp.conditional.phGraph_out[0];
      }
      CK(cudaStreamBeginCaptureToGraph(s, target, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal));
      for (int k = 0; k < K2; ++k) {
        Args c = a;
        c.x = (k & 1) ? x1 : x0;
        c.y = (k & 1) ? x0 : x1;
        c.use_cond = k == K2 - 1;
        c.h = h;
        c.stop = REP2;
        launch(s, c, P, 0);
      }
      CK(cudaStreamEndCapture(s, &target));
      cudaGraphExec_t we;
      CK(cudaGraphInstantiate(&we, wg, 0));
      float ms = 0;
      for (int w = 0; w < 3; ++w) {
        CK(cudaMemset(trips, 0, 8));
        CK(cudaEventRecord(e0, s));
        CK(cudaGraphLaunch(we, s));
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
      }
      unsigned long long tr;
      CK(cudaMemcpy(&tr, trips, 8, cudaMemcpyDeviceToHost));
      printf("WHILE%s K=%2d : %7.2f us/trip = %6.2f us/pass  (%llu trips)\n", sw ? "{SWITCH}" : "        ", K2,
             ms * 1e3 / tr, ms * 1e3 / (tr * K2), tr);
      CK(cudaGraphExecDestroy(we));
      CK(cudaGraphDestroy(wg));
    }
  // persistent
  for (int heavy = 0; heavy < 2; ++heavy) {
    const int P = sms;
    const int rows = (n + P - 1) / P;  // 676
    PArgs a = {};
    a.lo = dlo; a.di = ddi; a.up = dup; a.x0 = x0; a.n = n; a.rows = rows; a.state = state;
    CK(cudaMemcpy(x0, x.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&a.edge, 2 * P * 2 * 8));
    CK(cudaMalloc(&a.part, 2 * P * 8));
    CK(cudaMalloc(&a.seq, P * 4));
    a.yout = x1;
    a.passes = K * REP;
    float ms = 0;
    for (int w = 0; w < 3; ++w) {
      CK(cudaMemsetAsync(a.seq, 0, P * 4, s));
      void* args[] = {&a};
      CK(cudaEventRecord(e0, s));
      if (heavy) CK(cudaLaunchCooperativeKernel((void*)k_persist<3, 1>, dim3(P), dim3(NT), args, 0, s));
      else CK(cudaLaunchCooperativeKernel((void*)k_persist<3, 0>, dim3(P), dim3(NT), args, 0, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
    }
    double st[2];
    CK(cudaMemcpy(st, state, 16, cudaMemcpyDeviceToHost));
    printf("persistent   heavy=%d P=%4d       : %6.2f us/pass  (y.y %.17g)\n", heavy, P, ms * 1e3 / (K * REP), st[1]);
  }
  return 0;
}
