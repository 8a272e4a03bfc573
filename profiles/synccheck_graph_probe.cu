// Does compute-sanitizer synccheck report barrier divergence for a kernel
// that is correct when launched normally but runs inside a CUDA graph WHILE
// conditional node?  (The device-driven loop in engine.cu uses one.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/scp profiles/synccheck_graph_probe.cu
//   compute-sanitizer --tool synccheck /tmp/scp plain   # normal launches
//   compute-sanitizer --tool synccheck /tmp/scp graph   # WHILE-node body
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>

__global__ void k_reduce(const double* x, int n, double* out) {
  __shared__ double s[32];
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m += x[i];
  for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
  __syncwarp();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m += s[i];
    atomicAdd(out, m);
  }
}

__global__ void k_step(unsigned* iter, int limit, cudaGraphConditionalHandle h) {
  const unsigned k = ++*iter;
  cudaGraphSetConditional(h, k < (unsigned)limit ? 1u : 0u);
}

int main(int argc, char** argv) {
  const bool graph = argc > 1 && !std::strcmp(argv[1], "graph");
  const int n = 1 << 20;
  double* x;
  double* out;
  unsigned* iter;
  cudaMalloc(&x, n * sizeof(double));
  cudaMalloc(&out, sizeof(double));
  cudaMalloc(&iter, sizeof(unsigned));
  cudaMemset(x, 0, n * sizeof(double));
  cudaMemset(out, 0, sizeof(double));
  cudaMemset(iter, 0, sizeof(unsigned));
  cudaStream_t st;
  cudaStreamCreate(&st);
  if (!graph) {
    for (int i = 0; i < 4; ++i) k_reduce<<<148, 256, 0, st>>>(x, n, out);
  } else {
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    cudaGraphAddNode(&node, g, nullptr, 0, &p);
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaStream_t cap;
    cudaStreamCreate(&cap);
    cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    k_reduce<<<148, 256, 0, cap>>>(x, n, out);
    k_step<<<1, 1, 0, cap>>>(iter, 4, h);
    cudaStreamEndCapture(cap, &body);
    cudaGraphExec_t ex;
    cudaGraphInstantiate(&ex, g, 0);
    cudaGraphLaunch(ex, st);
  }
  const cudaError_t e = cudaStreamSynchronize(st);
  unsigned it = 0;
  cudaMemcpy(&it, iter, sizeof it, cudaMemcpyDeviceToHost);
  std::printf("%s: %s iterations=%u\n", graph ? "graph" : "plain", cudaGetErrorString(e), it);
  return e == cudaSuccess ? 0 : 1;
}
