// Microbenchmark (not part of the product): where does the ~1 random
// request / SM / clock ceiling of L2-resident gathers come from, and what
// do distributed shared memory and mixed smem+global gathers deliver?
//   (1) L2-resident 8 B gathers with only k SMs busy (SM-side vs L2-side limit)
//   (2) DSMEM random 8 B reads, clusters of 2/4/8/16 CTAs (1 CTA per SM)
//   (3) mixed: a fraction f of the gathers from local smem, the rest global
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb3 profiles/microbench_gather3.cu && ./mb3
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// (1) blocks on SMs >= active_sms exit immediately
__global__ void __launch_bounds__(256) k_g8_sms(const double* __restrict__ a, uint32_t mask, int iters,
                                                uint32_t active_sms, double* out) {
  if (smid() >= active_sms) return;
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __ldg(a + (hash(s * 8 + q + i * 0x9e3779b9u) & mask));
#pragma unroll
    for (int q = 0; q < 8; q += 2) { acc0 += x[q]; acc1 += x[q + 1]; }
  }
  if (acc0 + acc1 == 123.0) out[0] = acc0;
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)out + 1, 1ull);
}

constexpr int kSlots = 24576;  // 192 KB per CTA

// (2) DSMEM random reads within a cluster (cluster size from launch attribute)
__global__ void __launch_bounds__(1024, 1) k_dsmem(int iters, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned csize = cl.num_blocks();
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x) sm[i] = i;
  cl.sync();
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t h = hash(s * 8 + q + i * 0x9e3779b9u);
      const double* p = cl.map_shared_rank(sm + (h >> 4) % kSlots, (h & 15) % csize);
      x[q] = *p;
    }
#pragma unroll
    for (int q = 0; q < 8; q += 2) { acc0 += x[q]; acc1 += x[q + 1]; }
  }
  cl.sync();
  if (acc0 + acc1 == 123.0) out[0] = acc0;
}

// (3) a fraction (frac/16) of gathers from local smem, the rest from global (L2-resident)
__global__ void __launch_bounds__(1024, 1) k_mixed(const double* __restrict__ a, uint32_t mask, int frac, int iters,
                                                   double* out) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t h = hash(s * 8 + q + i * 0x9e3779b9u);
      x[q] = ((h >> 28) < (uint32_t)frac) ? sm[(h >> 3) % kSlots] : __ldg(a + (h & mask));
    }
#pragma unroll
    for (int q = 0; q < 8; q += 2) { acc0 += x[q]; acc1 += x[q + 1]; }
  }
  if (acc0 + acc1 == 123.0) out[0] = acc0;
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double clk = clk_khz * 1e3;
  const size_t n = 1ull << 22;  // 32 MB: L2-resident
  double* a;
  cudaMalloc(&a, n * 8);
  cudaMemset(a, 0, n * 8);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 64;
  for (int act : {16, 37, 74, 111, 148}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(out, 0, 64);
      cudaEventRecord(e0);
      k_g8_sms<<<sms * 8, 256>>>(a, (uint32_t)(n - 1), iters, act, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    unsigned long long blocks = 0;
    cudaMemcpy(&blocks, (unsigned long long*)out + 1, 8, cudaMemcpyDeviceToHost);
    const double el = (double)blocks * 256 * iters * 8;
    const double gs = el / (ms * 1e-3);
    printf("L2 gathers, %3d SMs active: %7.1f G/s total, %5.2f /active SM/clk\n", act, gs / 1e9, gs / act / clk);
  }
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * 8);
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    const int blocks = (sms / cs) * cs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = kSlots * 8;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t err = cudaSuccess;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      err = cudaLaunchKernelEx(&cfg, k_dsmem, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const double el = (double)blocks * 1024 * iters * 8;
    const double gs = el / (ms * 1e-3);
    printf("DSMEM random 8B, cluster %2d: %7.1f G/s, %5.2f /SM/clk (%s / %s)\n", cs, gs / 1e9, gs / blocks / clk,
           cudaGetErrorString(err), cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * 8);
  for (int frac : {0, 4, 8, 12, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_mixed<<<sms, 1024, kSlots * 8>>>(a, (uint32_t)(n - 1), frac, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const double el = (double)sms * 1024 * iters * 8;
    const double gs = el / (ms * 1e-3);
    printf("mixed: %3d%% smem / rest L2: %7.1f G/s, %5.2f /SM/clk (%s)\n", frac * 100 / 16, gs / 1e9, gs / sms / clk,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
