// Minimal repro: WHILE node whose body is stream-captured, with an IF node
// added mid-capture (cudaStreamGetCaptureInfo + cudaGraphAddNode +
// cudaStreamUpdateCaptureDependencies) and its body captured on a second
// stream; then walk the body's nodes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cif profiles/r02/cond_if_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    printf("%-90s -> %s\n", #x, cudaGetErrorString(e_));                             \
    if (e_ != cudaSuccess) return 1;                                                 \
  } while (0)

__global__ void k_step(int* c, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi) {
  c[0] += 1;
  cudaGraphSetConditional(hw, c[0] < 10 ? 1u : 0u);
  cudaGraphSetConditional(hi, (c[0] & 1) ? 1u : 0u);
}
__global__ void k_odd(int* c) { c[1] += 1; }

int main() {
  int* c;
  CK(cudaMalloc(&c, 8));
  CK(cudaMemset(c, 0, 8));
  cudaStream_t st, st2;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw;
  CK(cudaGraphConditionalHandleCreate(&hw, g, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = hw;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t wn;
  CK(cudaGraphAddNode(&wn, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaGraphConditionalHandle hi;
  CK(cudaGraphConditionalHandleCreate(&hi, body, 0u, cudaGraphCondAssignDefault));
  CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  k_step<<<1, 1, 0, st>>>(c, hw, hi);
  cudaStreamCaptureStatus cs;
  cudaGraph_t cg = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
  printf("capture graph == body: %d, deps %zu\n", cg == body, nd);
  cudaGraphNodeParams ip{};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = hi;
  ip.conditional.type = cudaGraphCondTypeIf;
  ip.conditional.size = 1;
  cudaGraphNode_t ifn;
  CK(cudaGraphAddNode(&ifn, cg, deps, nd, &ip));
  CK(cudaStreamUpdateCaptureDependencies(st, &ifn, 1, cudaStreamSetCaptureDependencies));
  CK(cudaStreamBeginCaptureToGraph(st2, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  k_odd<<<1, 1, 0, st2>>>(c);
  cudaGraph_t ib;
  CK(cudaStreamEndCapture(st2, &ib));
  cudaGraph_t cap;
  CK(cudaStreamEndCapture(st, &cap));
  size_t cnt = 0;
  CK(cudaGraphGetNodes(body, nullptr, &cnt));
  std::vector<cudaGraphNode_t> nodes(cnt);
  CK(cudaGraphGetNodes(body, nodes.data(), &cnt));
  for (auto n : nodes) {
    cudaGraphNodeType t;
    cudaError_t e = cudaGraphNodeGetType(n, &t);
    printf("  node %s: type %d (%s)\n", n == ifn ? "if" : "-", (int)t, cudaGetErrorString(e));
    cudaGetLastError();
  }
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, g, 0));
  CK(cudaGraphLaunch(ex, st));
  CK(cudaStreamSynchronize(st));
  int h[2];
  CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
  printf("iterations %d odd %d (expect 10, 5)\n", h[0], h[1]);
  return 0;
}
