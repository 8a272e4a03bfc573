// Microbenchmark (not part of the product): random-gather throughput on
// B200 by footprint and load flavour, to size the rank-update sweep design.
//   global 8 B gathers (ld.global.nc / .cg / L1::no_allocate) over 32 KB..512 MB
//   global 4 B and 16 B gathers (is the limit requests or bytes?)
//   shared-memory 8 B random reads
// Reports G gathers/s and gathers per SM per clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb2 profiles/microbench_gather2.cu && ./mb2
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int MODE>
__device__ __forceinline__ double ld8(const double* p) {
  double v;
  if (MODE == 0) v = __ldg(p);
  else if (MODE == 1) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_g8(const double* __restrict__ a, uint32_t mask, int iters, double* out) {
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = ld8<MODE>(a + (hash(s * 8 + q + i * 0x9e3779b9u) & mask));
#pragma unroll
    for (int q = 0; q < 8; q += 2) { acc0 += x[q]; acc1 += x[q + 1]; }
  }
  if (acc0 + acc1 == 123.0) out[0] = acc0;
}

__global__ void __launch_bounds__(256) k_g4(const uint32_t* __restrict__ a, uint32_t mask, int iters, uint32_t* out) {
  uint32_t acc = 0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= __ldg(a + (hash(s * 8 + q + i * 0x9e3779b9u) & mask));
  }
  if (acc == 123u) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_g16(const double2* __restrict__ a, uint32_t mask, int iters, double* out) {
  double acc = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double2 x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __ldg(a + (hash(s * 8 + q + i * 0x9e3779b9u) & mask));
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += x[q].x + x[q].y;
  }
  if (acc == 123.0) out[0] = acc;
}

// shared memory: slots doubles per CTA
__global__ void k_smem(int slots_log2, int iters, double* out) {
  extern __shared__ double sm[];
  const uint32_t slots = 1u << slots_log2;
  for (uint32_t i = threadIdx.x; i < slots; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double acc0 = 0.0, acc1 = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = sm[hash(s * 8 + q + i * 0x9e3779b9u) & (slots - 1)];
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
  const size_t maxn = 1ull << 26;  // 512 MB of doubles
  double* a;
  cudaMalloc(&a, maxn * 8);
  cudaMemset(a, 0, maxn * 8);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 64;
  const int blocks = sms * 8;  // 8 x 256 threads per SM
  const double elems = (double)blocks * 256 * iters * 8;
  auto report = [&](const char* name, size_t bytes, float ms) {
    const double gs = elems / (ms * 1e-3);
    printf("%-34s footprint %9.3f MB : %7.1f G/s  %5.2f /SM/clk\n", name, bytes / 1e6, gs / 1e9, gs / sms / clk);
  };
  float ms;
  for (int lg = 12; lg <= 26; lg += 2) {
    const uint32_t mask = (1u << lg) - 1;
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k_g8<0><<<blocks, 256>>>(a, mask, iters, out);
        if (mode == 1) k_g8<1><<<blocks, 256>>>(a, mask, iters, out);
        if (mode == 2) k_g8<2><<<blocks, 256>>>(a, mask, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const char* nm[3] = {"8B ld.global.nc", "8B ld.global.cg", "8B ld.global.nc.L1::no_allocate"};
      report(nm[mode], (size_t)8 << lg, ms);
    }
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_g4<<<blocks, 256>>>((const uint32_t*)a, (1u << (lg + 1)) - 1, iters, (uint32_t*)out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    report("4B ld.global.nc", (size_t)8 << lg, ms);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_g16<<<blocks, 256>>>((const double2*)a, (1u << (lg - 1)) - 1, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    report("16B ld.global.nc", (size_t)8 << lg, ms);
  }
  for (int lg = 10; lg <= 14; ++lg) {
    const int per_sm = lg <= 12 ? 8 : (lg == 13 ? 3 : 1);
    const size_t smem = (size_t)8 << lg;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_smem<<<sms * per_sm, 256, smem>>>(lg, iters * 4, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const double el = (double)sms * per_sm * 256 * iters * 4 * 8;
    const double gs = el / (ms * 1e-3);
    printf("smem 8B random, %d CTA/SM x %6zu B     : %7.1f G/s  %5.2f /SM/clk (%s)\n", per_sm, smem, gs / 1e9,
           gs / sms / clk, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
