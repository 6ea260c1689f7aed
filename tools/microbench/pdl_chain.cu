// Does programmatic dependent launch (PDL) hide a pass kernel's tail (the
// last-block finisher) and the kernel boundary when the dependent kernel
// prefetches its first matrix stages BEFORE griddepcontrol.wait?
// A chain of C4-like (5-point, n = 1e6) streamed CSR passes, each ending in a
// deterministic last-block reduction that writes a "state" scalar the next
// pass reads at entry, as the library's solver state machine does.
// Modes: plain stream / linear graph / WHILE-node body, PDL off/on.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/microbench/pdl_chain tools/microbench/pdl_chain.cu
#include <algorithm>
#include <cstdio>
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

constexpr int CAP = 1024, ROWS = 256, S = 4, NB = 4;
struct __align__(16) Stage {
  double val[CAP + 2];
  int idx[CAP + 4];
  int rp[ROWS + 8];
};
constexpr int SMEM = S * (int)sizeof(Stage);

struct Args {
  const int *rp, *ci;
  const double* val;
  const int2* chunks;
  const int* blk;
  const double* x;  // input vector (previous pass output)
  double* y;        // output vector
  double* bacc;     // [P] partials
  unsigned* done;
  double* state;    // [0] scale read at entry, [1] last reduction
  unsigned long long* trips;
  cudaGraphConditionalHandle h;
  int use_cond;
  unsigned long long stop;
  int pdl;
};

__global__ void __launch_bounds__(256, NB) k_pass(Args A) {
  extern __shared__ __align__(128) unsigned char raw[];
  Stage* stg = reinterpret_cast<Stage*>(raw);
  __shared__ __align__(8) unsigned long long full[S];
  __shared__ double sm[8];
  __shared__ int sflag;
  const int tid = threadIdx.x;
  const int c0 = __ldg(A.blk + blockIdx.x), c1 = __ldg(A.blk + blockIdx.x + 1);
  auto issue = [&](int c, int s) {
    const int2 a = __ldg(A.chunks + c), z = __ldg(A.chunks + c + 1);
    const int e0v = a.y & ~1, e0i = a.y & ~3, r0 = a.x & ~3;
    const unsigned bv = (unsigned)(((z.y - e0v) * 8 + 15) & ~15);
    const unsigned bi = (unsigned)(((z.y - e0i) * 4 + 15) & ~15);
    const unsigned br = (unsigned)(((z.x + 1 - r0) * 4 + 15) & ~15);
    mbar_expect_tx(&full[s], bv + bi + br);
    bulk_g2s(stg[s].val, A.val + e0v, bv, &full[s]);
    bulk_g2s(stg[s].idx, A.ci + e0i, bi, &full[s]);
    bulk_g2s(stg[s].rp, A.rp + r0, br, &full[s]);
  };
  // independent prologue: the matrix is immutable, so its first stages can
  // stream in while the previous pass is still finishing
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    for (int s = 0; s < S && c0 + s < c1; ++s) issue(c0 + s, s);
  }
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const double scale = A.state[0];  // dependent: written by the previous finisher
  __syncthreads();
  double acc = 0;
  int2 a = c0 < c1 ? __ldg(A.chunks + c0) : make_int2(0, 0);
  for (int c = c0, g = 0; c < c1; ++c, ++g) {
    const int s = g % S;
    const int2 z = __ldg(A.chunks + c + 1);
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
        xv[u] = k < ne ? __ldcg(A.x + si[k]) : 0.0;
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
      sum *= scale;
      A.y[a.x + r] = sum;
      acc = fma(sum, sum, acc);
    }
    __syncthreads();
    if (tid == 0 && c + S < c1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + S, s);
    }
    a = z;
  }
  // the dependent grid may start launching now (its blocks fill SMs as ours exit)
  if (A.pdl) asm volatile("griddepcontrol.launch_dependents;");
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) sm[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0;
    for (int i = 0; i < 8; ++i) s += sm[i];
    A.bacc[blockIdx.x] = s;
  }
  if (arrive_last(A.done, gridDim.x, &sflag)) {
    double t = 0;
    for (int b = tid; b < (int)gridDim.x; b += 256) t += __ldcg(A.bacc + b);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    __syncthreads();
    if ((tid & 31) == 0) sm[tid >> 5] = t;
    __syncthreads();
    if (tid == 0) {
      double s = 0;
      for (int i = 0; i < 8; ++i) s += sm[i];
      A.state[1] = s;
      A.state[0] = 1.0 / (1.0 + 1e-300 * s);  // "step size" for the next pass (== 1)
      if (A.use_cond) {
        const unsigned long long v = ++*A.trips;
        cudaGraphSetConditional(A.h, v < A.stop ? 1u : 0u);
      }
    }
  }
}

static void launch(cudaStream_t s, const Args& a, int P) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a.pdl ? at : nullptr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, k_pass, a));
}

int main() {
  const int G = 1000, m = G * G;
  std::vector<int> rp(m + 1), ci;
  std::vector<double> v;
  for (int iy = 0; iy < G; ++iy)
    for (int ix = 0; ix < G; ++ix) {
      const int k = ix + G * iy;
      rp[k] = (int)ci.size();
      if (iy > 0) { ci.push_back(k - G); v.push_back(-0.25); }
      if (ix > 0) { ci.push_back(k - 1); v.push_back(-0.25); }
      ci.push_back(k); v.push_back(1.0);
      if (ix < G - 1) { ci.push_back(k + 1); v.push_back(-0.25); }
      if (iy < G - 1) { ci.push_back(k + G); v.push_back(-0.25); }
    }
  rp[m] = (int)ci.size();
  const long long nnz = rp[m];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int P = sms * NB;
  std::vector<int2> ch;
  for (int r = 0; r < m;) {
    ch.push_back(make_int2(r, rp[r]));
    int e = r + 1;
    while (e < m && e - r < ROWS && rp[e + 1] - rp[r] <= CAP) ++e;
    r = e;
  }
  ch.push_back(make_int2(m, (int)nnz));
  const int nc = (int)ch.size() - 1;
  std::vector<int> blk(P + 1);
  for (int b = 0; b <= P; ++b) {
    if (b == P) { blk[b] = nc; continue; }
    const long long t = nnz * b / P;
    blk[b] = (int)(std::lower_bound(ch.begin(), ch.end() - 1, t, [](const int2& q, long long tt) { return q.y < tt; }) - ch.begin());
  }
  Args a = {};
  int *drp, *dci, *dblk;
  double *dval, *x0, *x1, *bacc, *state;
  int2* dch;
  unsigned* done;
  unsigned long long* trips;
  CK(cudaMalloc(&drp, (m + 8) * 4));
  CK(cudaMalloc(&dci, (nnz + 8) * 4));
  CK(cudaMalloc(&dval, (nnz + 4) * 8));
  CK(cudaMalloc(&dch, ch.size() * 8));
  CK(cudaMalloc(&dblk, blk.size() * 4));
  CK(cudaMalloc(&x0, m * 8));
  CK(cudaMalloc(&x1, m * 8));
  CK(cudaMalloc(&bacc, P * 8));
  CK(cudaMalloc(&state, 16));
  CK(cudaMalloc(&done, 16));
  CK(cudaMalloc(&trips, 8));
  CK(cudaMemcpy(drp, rp.data(), (m + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dval, v.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dch, ch.data(), ch.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dblk, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice));
  std::vector<double> ones(m, 1.0);
  CK(cudaMemcpy(x0, ones.data(), m * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(x1, ones.data(), m * 8, cudaMemcpyHostToDevice));
  const double st0[2] = {1.0, 0.0};
  CK(cudaMemcpy(state, st0, 16, cudaMemcpyHostToDevice));
  CK(cudaMemset(done, 0, 16));
  CK(cudaFuncSetAttribute(k_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  a.rp = drp; a.ci = dci; a.val = dval; a.chunks = dch; a.blk = dblk;
  a.bacc = bacc; a.done = done; a.state = state; a.trips = trips;
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int K = 10, REP = 40;
  double ref = 0;
  for (int pdl = 0; pdl < 2; ++pdl) {
    a.pdl = pdl;
    auto chain = [&](int k, int use_cond, cudaGraphConditionalHandle h, unsigned long long stop) {
      Args b = a;
      b.x = (k & 1) ? x1 : x0;
      b.y = (k & 1) ? x0 : x1;
      b.use_cond = use_cond;
      b.h = h;
      b.stop = stop;
      launch(s, b, P);
    };
    float ms;
    // stream
    for (int w = 0; w < 2; ++w) {
      CK(cudaEventRecord(e0, s));
      for (int r = 0; r < REP; ++r)
        for (int k = 0; k < K; ++k) chain(k, 0, 0, 0);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double st[2];
    CK(cudaMemcpy(st, state, 16, cudaMemcpyDeviceToHost));
    if (!pdl) ref = st[1];
    printf("pdl=%d stream      : %7.2f us/pass  (check %s)\n", pdl, ms * 1e3 / (REP * K),
           st[1] == ref ? "same" : "DIFF");
    // linear graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int k = 0; k < K; ++k) chain(k, 0, 0, 0);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int w = 0; w < 2; ++w) {
      CK(cudaEventRecord(e0, s));
      for (int r = 0; r < REP; ++r) CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d linear graph: %7.2f us/pass\n", pdl, ms * 1e3 / (REP * K));
    // WHILE node: body = K passes, REP trips
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
    for (int k = 0; k < K; ++k) chain(k, k == K - 1, h, REP);
    CK(cudaStreamEndCapture(s, &body));
    cudaGraphExec_t we;
    CK(cudaGraphInstantiate(&we, wg, 0));
    for (int w = 0; w < 2; ++w) {
      CK(cudaMemset(trips, 0, 8));
      CK(cudaEventRecord(e0, s));
      CK(cudaGraphLaunch(we, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long tr;
    CK(cudaMemcpy(&tr, trips, 8, cudaMemcpyDeviceToHost));
    printf("pdl=%d WHILE body  : %7.2f us/pass  (%llu trips)\n", pdl, ms * 1e3 / (tr * K), tr);
  }
  return 0;
}
