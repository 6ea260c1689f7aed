// Kernel-boundary cost inside CUDA graphs on this GPU: a chain of K trivial
// 592-block kernels, (a) plain stream, (b) captured linear graph, (c) inside a
// conditional WHILE body, each with and without programmatic dependent launch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(unsigned long long* c, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(c, 1ull);
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}
__global__ void k_cond(unsigned long long* c, cudaGraphConditionalHandle h, unsigned long long stop, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long v = atomicAdd(c, 1ull) + 1;
    cudaGraphSetConditional(h, v < stop ? 1u : 0u);
  }
}

static void launch(cudaStream_t s, unsigned long long* c, int pdl, int blocks) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_tiny, c, pdl);
}

int main() {
  unsigned long long* c;
  cudaMalloc(&c, 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int K = 12, blocks = 592, REP = 200;
  for (int pdl = 0; pdl < 2; ++pdl) {
    // (a) stream
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      for (int r = 0; r < REP; ++r) for (int k = 0; k < K; ++k) launch(s, c, pdl, blocks);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d stream launches      : %6.2f us/kernel\n", pdl, ms * 1e3 / (REP * K));
    // (b) linear graph of K kernels, launched REP times
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < K; ++k) launch(s, c, pdl, blocks);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      for (int r = 0; r < REP; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d linear graph         : %6.2f us/kernel (%s)\n", pdl, ms * 1e3 / (REP * K),
           cudaGetErrorString(cudaGetLastError()));
    // (c) WHILE node: body = K-1 tiny kernels + 1 cond kernel; REP trips
    cudaGraph_t wg;
    cudaGraphCreate(&wg, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, wg, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    cudaGraphAddNode(&node, wg, nullptr, 0, &np);
    cudaGraph_t body = np.conditional.phGraph_out[0];
    cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < K - 1; ++k) launch(s, c, pdl, blocks);
    {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = pdl ? at : nullptr;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, k_cond, c, h, 0ull, pdl);  // placeholder stop patched below
    }
    cudaGraph_t outb;
    cudaStreamEndCapture(s, &outb);
    // the stop value is baked in the kernel args; rebuild with the right value:
    cudaGraphExec_t we;
    cudaError_t ie = cudaGraphInstantiate(&we, wg, 0);
    cudaMemset(c, 0, 8);
    // stop = 0 -> one trip; measure REP trips by re-launching REP times
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      for (int r = 0; r < REP; ++r) cudaGraphLaunch(we, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d WHILE body (1 trip)  : %6.2f us/kernel (inst %s, %s)\n", pdl, ms * 1e3 / (REP * K),
           cudaGetErrorString(ie), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
