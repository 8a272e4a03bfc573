// Microbenchmark (not part of the product): do bulk-copy (TMA engine) and
// LDGSTS gathers add request capacity beside the LSU/L1TEX path, whose random
// L2 requests cap at ~1 per SM per clock (microbench_gather3)?
//   (a) ld.global.nc 8 B gathers                              (baseline)
//   (b) cp.async.bulk 16 B per lane -> smem, mbarrier completion
//   (c) cp.async.ca 8 B (LDGSTS) per lane -> smem
//   (d) half of the gathers via (a), half via (b)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb4 profiles/microbench_gather4.cu && ./mb4
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

constexpr int kThreads = 128;
constexpr int kDepth = 8;  // gathers in flight per thread per round

__global__ void __launch_bounds__(kThreads) k_ldg(const double* __restrict__ a, uint32_t mask, int iters,
                                                  double* out) {
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double x[kDepth];
#pragma unroll
    for (int q = 0; q < kDepth; ++q) x[q] = __ldg(a + (hash(s * 8 + q + i * 0x9e3779b9u) & mask));
#pragma unroll
    for (int q = 0; q < kDepth; q += 2) { acc0 += x[q]; acc1 += x[q + 1]; }
  }
  if (acc0 + acc1 == 123.0) out[0] = acc0;
}

// (b) + (d): every lane issues bulk copies of the 16 B line piece holding its
// element; `ldg_share` of 8 gathers per round go through ld.global instead.
__global__ void __launch_bounds__(kThreads) k_bulk(const double* __restrict__ a, uint32_t mask, int iters,
                                                   int ldg_share, double* out) {
  __shared__ __align__(16) double buf[2][kThreads * kDepth * 2];
  __shared__ __align__(8) unsigned long long bar[2];
  const int t = threadIdx.x;
  if (t == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(kThreads));
  }
  __syncthreads();
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = kDepth - ldg_share;
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1;
    const uint32_t mb = smem_u32(&bar[b]);
    // arrive + expect the bytes of this thread's copies
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(nb * 16) : "memory");
    for (int q = 0; q < nb; ++q) {
      const uint32_t e = hash(s * 8 + q + i * 0x9e3779b9u) & mask & ~1u;  // 16 B aligned pair
      double* dst = &buf[b][(t * kDepth + q) * 2];
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(smem_u32(dst)),
          "l"(a + e), "r"(mb)
          : "memory");
    }
    double x[kDepth];
    for (int q = nb; q < kDepth; ++q) x[q] = __ldg(a + (hash(s * 8 + q + i * 0x9e3779b9u) & mask));
    // wait for phase (i >> 1) & 1 of bar[b]
    const uint32_t parity = (i >> 1) & 1;
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(mb),
        "r"(parity)
        : "memory");
    for (int q = 0; q < nb; ++q) x[q] = buf[b][(t * kDepth + q) * 2];
    for (int q = 0; q < kDepth; q += 2) { acc0 += x[q]; acc1 += x[q + 1]; }
    __syncthreads();  // buffer reuse two rounds later
  }
  if (acc0 + acc1 == 123.0) out[0] = acc0;
}

__global__ void __launch_bounds__(kThreads) k_ldgsts(const double* __restrict__ a, uint32_t mask, int iters,
                                                     double* out) {
  __shared__ __align__(16) double buf[kThreads * kDepth];
  const int t = threadIdx.x;
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < kDepth; ++q) {
      const uint32_t e = hash(s * 8 + q + i * 0x9e3779b9u) & mask;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&buf[t * kDepth + q])), "l"(a + e)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
    for (int q = 0; q < kDepth; q += 2) { acc0 += buf[t * kDepth + q]; acc1 += buf[t * kDepth + q + 1]; }
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
  const int blocks = sms * 16;
  const double el = (double)blocks * kThreads * iters * kDepth;
  auto rep = [&](const char* name) {
    const double gs = el / (ms * 1e-3);
    printf("%-40s %7.1f G/s  %5.2f /SM/clk (%s)\n", name, gs / 1e9, gs / sms / clk,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0);
    k_ldg<<<blocks, kThreads>>>(a, (uint32_t)(n - 1), iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  rep("(a) ld.global.nc 8B");
  for (int share : {0, 2, 4, 6}) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0);
      k_bulk<<<blocks, kThreads>>>(a, (uint32_t)(n - 1), iters, share, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    char nm[64];
    snprintf(nm, sizeof nm, "(b/d) bulk 16B x%d + ldg x%d", kDepth - share, share);
    rep(nm);
  }
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0);
    k_ldgsts<<<blocks, kThreads>>>(a, (uint32_t)(n - 1), iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  rep("(c) cp.async.ca 8B (LDGSTS)");
  return 0;
}
