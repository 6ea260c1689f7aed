// Which kernels may set a SWITCH node's conditional handle?  The CTA loop is
// WHILE{ SWITCH{case t} }; the case kernels' finisher knows the next case, so
// the per-iteration "head" kernel that only translates state -> switch value
// can go IF (a) a kernel of one trip may set the value the NEXT trip's SWITCH
// reads, and (b) the first trip's value can come from a kernel node placed in
// the OUTER graph before the WHILE node.
// Variants: handle owned by the body graph / by the top-level graph.
// Prints the case sequence each variant executed (expected: 0 1 2 0 1 2 ...).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench/cond_handle \
//        tools/microbench/cond_handle.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

struct Log {
  int n;
  int seq[64];
  int next;
  int trips;
};

// after the SWITCH on every trip: stops the loop when no case ever clears it
__global__ void k_guard(Log* l, cudaGraphConditionalHandle wh) {
  if (threadIdx.x == 0) {
    l->trips += 1;
    if (l->trips > 40) cudaGraphSetConditional(wh, 0u);
  }
}

__global__ void k_first(Log* l, cudaGraphConditionalHandle sw) {
  if (threadIdx.x == 0) cudaGraphSetConditional(sw, (unsigned)l->next);
}
__global__ void k_case(Log* l, int me, int ncases, int stop, cudaGraphConditionalHandle sw,
                       cudaGraphConditionalHandle wh) {
  if (threadIdx.x == 0) {
    if (l->n < 64) l->seq[l->n] = me;
    l->n += 1;
    l->next = (me + 1) % ncases;
    cudaGraphSetConditional(sw, (unsigned)l->next);
    cudaGraphSetConditional(wh, l->n < stop ? 1u : 0u);
  }
}

static int run(int own_top, int outer_first) {
  Log* l;
  CK(cudaMalloc(&l, sizeof(Log)));
  CK(cudaMemset(l, 0, sizeof(Log)));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle wh;
  CK(cudaGraphConditionalHandleCreate(&wh, g, 1, cudaGraphCondAssignDefault));
  const int nc = 3;
  // outer: [k_first] -> WHILE
  cudaGraphNode_t first = nullptr;
  cudaGraphConditionalHandle sw = 0;
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = wh;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  // the SWITCH handle must exist before k_first's parameters are baked: when it is
  // owned by the body graph the WHILE node has to be added first
  cudaGraphNode_t wnode;
  if (own_top) CK(cudaGraphConditionalHandleCreate(&sw, g, 0, 0));
  if (own_top && outer_first) {
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    void* args[2] = {&l, &sw};
    kp.kernel.func = (void*)k_first;
    kp.kernel.gridDim = dim3(1);
    kp.kernel.blockDim = dim3(32);
    kp.kernel.kernelParams = args;
    CK(cudaGraphAddNode(&first, g, nullptr, 0, &kp));
    CK(cudaGraphAddNode(&wnode, g, &first, 1, &wp));
  } else {
    CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
  }
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  if (!own_top) CK(cudaGraphConditionalHandleCreate(&sw, body, 0, 0));
  if (!own_top && outer_first) {
    // add k_first afterwards and make the WHILE node depend on it
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    void* args[2] = {&l, &sw};
    kp.kernel.func = (void*)k_first;
    kp.kernel.gridDim = dim3(1);
    kp.kernel.blockDim = dim3(32);
    kp.kernel.kernelParams = args;
    CK(cudaGraphAddNode(&first, g, nullptr, 0, &kp));
    CK(cudaGraphAddDependencies(g, &first, &wnode, 1));
  }
  cudaGraphNodeParams sp = {};
  sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = sw;
  sp.conditional.type = cudaGraphCondTypeSwitch;
  sp.conditional.size = nc;
  cudaGraphNode_t snode;
  cudaGraphNode_t dep = nullptr;
  if (!outer_first) {  // classic: a head kernel inside the body
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    void* args[2] = {&l, &sw};
    kp.kernel.func = (void*)k_first;
    kp.kernel.gridDim = dim3(1);
    kp.kernel.blockDim = dim3(32);
    kp.kernel.kernelParams = args;
    CK(cudaGraphAddNode(&dep, body, nullptr, 0, &kp));
  }
  CK(cudaGraphAddNode(&snode, body, dep ? &dep : nullptr, dep ? 1 : 0, &sp));
  {
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    void* args[2] = {&l, &wh};
    kp.kernel.func = (void*)k_guard;
    kp.kernel.gridDim = dim3(1);
    kp.kernel.blockDim = dim3(32);
    kp.kernel.kernelParams = args;
    cudaGraphNode_t gn;
    CK(cudaGraphAddNode(&gn, body, &snode, 1, &kp));
  }
  for (int c = 0; c < nc; ++c) {
    cudaGraph_t cg = sp.conditional.phGraph_out[c];
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    int me = c, ncases = nc, stop = 10;
    void* args[6] = {&l, &me, &ncases, &stop, &sw, &wh};
    kp.kernel.func = (void*)k_case;
    kp.kernel.gridDim = dim3(1);
    kp.kernel.blockDim = dim3(32);
    kp.kernel.kernelParams = args;
    cudaGraphNode_t kn;
    CK(cudaGraphAddNode(&kn, cg, nullptr, 0, &kp));
  }
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, g, 0));
  Log h;
  for (int rep = 0; rep < 2; ++rep) {  // second launch: continues from l->next = 1
    CK(cudaGraphLaunch(ex, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(&h, l, sizeof(h), cudaMemcpyDeviceToHost));
    printf("own_top=%d outer_first=%d launch %d: trips=%d n=%d seq:", own_top, outer_first, rep, h.trips, h.n);
    for (int i = 0; i < h.n && i < 64; ++i) printf(" %d", h.seq[i]);
    printf("\n");
    h.n = 0;
    h.trips = 0;
    h.next = 1;
    CK(cudaMemcpy(l, &h, sizeof(h), cudaMemcpyHostToDevice));
  }
  cudaGraphExecDestroy(ex);
  cudaGraphDestroy(g);
  cudaFree(l);
  return 0;
}

int main() {
  for (int own_top = 0; own_top < 2; ++own_top)
    for (int outer_first = 0; outer_first < 2; ++outer_first) {
      const int rc = run(own_top, outer_first);
      if (rc) {
        printf("own_top=%d outer_first=%d: FAILED to build / run\n", own_top, outer_first);
        cudaGetLastError();
      }
      fflush(stdout);
    }
  return 0;
}
