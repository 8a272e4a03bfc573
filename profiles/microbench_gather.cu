// Microbenchmark: throughput of random 8-byte gathers on B200 from
//   (a) global memory, L2-resident working set   (ld.global.nc)
//   (b) the CTA's own shared memory              (ld.shared)
//   (c) an 8-CTA cluster's distributed shared memory (ld.shared::cluster)
// Decides whether a cluster-shared "hot contribution" cache can beat the L2
// request ceiling of the rank-update sweep.  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb profiles/microbench_gather.cu
//   ./mb
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr int kSlots = 24576;  // doubles per CTA (192 KB)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__global__ void k_global(const double* __restrict__ a, uint32_t mask, int iters, double* out) {
  double acc = 0.0;
  uint32_t s = blockIdx.x * kThreads + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += __ldg(a + (hash(s + q * 7919u + i * 104729u) & mask));
  }
  if (acc == 123.0) out[0] = acc;
}

__global__ void k_smem(int iters, double* out) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < kSlots; i += kThreads) sm[i] = i;
  __syncthreads();
  double acc = 0.0;
  uint32_t s = blockIdx.x * kThreads + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += sm[hash(s + q * 7919u + i * 104729u) % kSlots];
  }
  if (acc == 123.0) out[0] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) k_dsmem(int iters, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < kSlots; i += kThreads) sm[i] = i;
  cl.sync();
  double acc = 0.0;
  uint32_t s = blockIdx.x * kThreads + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t h = hash(s + q * 7919u + i * 104729u);
      const double* p = cl.map_shared_rank(sm + (h >> 3) % kSlots, h & 7);
      acc += *p;
    }
  }
  cl.sync();
  if (acc == 123.0) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* a;
  const size_t n = 1u << 21;  // 16 MB: L2-resident
  cudaMalloc(&a, n * 8);
  cudaMemset(a, 0, n * 8);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int blocks = sms;  // one 1024-thread CTA per SM
  const double elems = (double)blocks * kThreads * iters * 8;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_global<<<blocks, kThreads>>>(a, (uint32_t)(n - 1), iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("global L2-resident random 8B gathers: %.1f G/s\n", elems / ms / 1e6);
  }
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * 8);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_smem<<<blocks, kThreads, kSlots * 8>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("shared memory random 8B reads:        %.1f G/s (%s)\n", elems / ms / 1e6,
                    cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * 8);
  const int cblocks = (sms / 8) * 8;
  const double celems = (double)cblocks * kThreads * iters * 8;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_dsmem<<<cblocks, kThreads, kSlots * 8>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("DSMEM (8-CTA cluster) random 8B reads: %.1f G/s (%s)\n", celems / ms / 1e6,
                    cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
