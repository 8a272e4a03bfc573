// Random 8-byte gathers three ways, to see whether the TMA unit adds request
// throughput on top of the LSU/L1 path that bounds the sweep
// (profiles/r02/README.md "Request-pipe evidence"):
//   ldg   -- the sweep's path: 16-byte coalesced index loads, __ldg gathers,
//            8 in flight per thread;
//   tma   -- per lane one cp.async.bulk.tensor.2d.tile::gather4 per 4
//            indices (rows of 16 bytes = the pair holding the value), into a
//            per-warp smem stage completed on an mbarrier, kStages deep;
//   mixed -- half of each warp's index groups through each path.
// Output: gathers per second and per SM per clock, for an L2-resident and
// a DRAM-sized value array.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_tma profiles/microbench_tma_gather.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);        \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kStages = 4;
constexpr int kSmem = kWarps * kStages * 32 * 128;  // TMA destinations are 128-byte aligned

__device__ __forceinline__ uint4 ld_idx4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// groups: ngroups uint4 index groups; warp w of the grid takes groups
// [w*32 .. w*32+31] + k * (total warps * 32)
__global__ void __launch_bounds__(kThreads) k_ldg(const uint4* __restrict__ idx, uint64_t ngroups,
                                                  const double* __restrict__ val, double* out) {
  const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  double s = 0.0;
  uint64_t g = tid;
  for (; g + stride < ngroups; g += 2 * stride) {
    const uint4 a = ld_idx4((const uint32_t*)(idx + g));
    const uint4 b = ld_idx4((const uint32_t*)(idx + g + stride));
    const double x0 = __ldg(val + a.x), x1 = __ldg(val + a.y), x2 = __ldg(val + a.z), x3 = __ldg(val + a.w);
    const double y0 = __ldg(val + b.x), y1 = __ldg(val + b.y), y2 = __ldg(val + b.z), y3 = __ldg(val + b.w);
    s += ((x0 + x1) + (x2 + x3)) + ((y0 + y1) + (y2 + y3));
  }
  for (; g < ngroups; g += stride) {
    const uint4 a = ld_idx4((const uint32_t*)(idx + g));
    s += (__ldg(val + a.x) + __ldg(val + a.y)) + (__ldg(val + a.z) + __ldg(val + a.w));
  }
  out[tid] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_arrive(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, uint64_t* bar, void* dst, uint4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
      : "memory");
}

// tma_every: 1 = every group through TMA; 2 = every other group (the rest LDG)
__global__ void __launch_bounds__(kThreads) k_tma(const __grid_constant__ CUtensorMap map, const uint4* __restrict__ idx,
                                                  uint64_t ngroups, const double* __restrict__ val, double* out,
                                                  int tma_every) {
  extern __shared__ __align__(128) double2 dyn[];  // [kWarps][kStages][32][8]: 64 of 128 B per lane per stage
  __shared__ alignas(8) uint64_t bar[kWarps][kStages];
  auto slot = [&](unsigned w_, int st_, unsigned l_) { return dyn + (((w_ * kStages + st_) * 32 + l_) * 8); };
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[w][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t gw = (uint64_t)blockIdx.x * kWarps + w, nw = (uint64_t)gridDim.x * kWarps;
  // step k of this warp: groups (gw + k * nw) * 32 + lane
  const uint64_t nsteps_all = (ngroups / 32 + nw - 1 - gw) / nw;
  double s = 0.0;
  uint32_t lows = 0;  // 4 low index bits per stage
  unsigned phase = 0;  // bit per stage
  uint64_t issued = 0, done = 0;
  auto group_of = [&](uint64_t k) { return (gw + k * nw) * 32 + lane; };
  while (done < nsteps_all) {
    // issue while stages are free
    while (issued < nsteps_all && issued - done < kStages) {
      const uint64_t kk = issued;
      const int st = (int)(kk % kStages);
      const uint4 u = ld_idx4((const uint32_t*)(idx + group_of(kk)));
      if (tma_every == 1 || (kk & 1) == 0) {
        const uint32_t lo = (u.x & 1) | (u.y & 1) << 1 | (u.z & 1) << 2 | (u.w & 1) << 3;
        lows = (lows & ~(0xFu << (4 * st))) | lo << (4 * st);
        __syncwarp();
        if (lane == 0) mbar_expect_arrive(&bar[w][st], 32 * 64);
        tma_gather4(&map, &bar[w][st], slot(w, st, lane), make_uint4(u.x >> 1, u.y >> 1, u.z >> 1, u.w >> 1));
      } else {
        s += (__ldg(val + u.x) + __ldg(val + u.y)) + (__ldg(val + u.z) + __ldg(val + u.w));
      }
      ++issued;
    }
    {
      const uint64_t kk = done;
      const int st = (int)(kk % kStages);
      if (tma_every == 1 || (kk & 1) == 0) {
        mbar_wait(&bar[w][st], (phase >> st) & 1);
        phase ^= 1u << st;
        const double2* r = slot(w, st, lane);
        const uint32_t lo = (lows >> (4 * st)) & 0xF;
        const double x0 = (lo & 1) ? r[0].y : r[0].x, x1 = (lo & 2) ? r[1].y : r[1].x;
        const double x2 = (lo & 4) ? r[2].y : r[2].x, x3 = (lo & 8) ? r[3].y : r[3].x;
        s += (x0 + x1) + (x2 + x3);
        __syncwarp();
      }
      ++done;
    }
  }
  out[(uint64_t)blockIdx.x * kThreads + threadIdx.x] = s;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  const uint64_t ngather = 1ull << 28, ngroups = ngather / 4;
  std::vector<uint32_t> hidx(ngather);
  double* out;
  uint4* idx;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  CK(cudaMalloc(&out, (size_t)sms * 32 * kThreads * sizeof(double)));
  CK(cudaMalloc(&idx, ngather * 4));
  for (int log_n : {22, 24}) {
    const uint64_t n = 1ull << log_n;
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (uint64_t i = 0; i < ngather; ++i) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      hidx[i] = (uint32_t)(x & (n - 1));
    }
    CK(cudaMemcpy(idx, hidx.data(), ngather * 4, cudaMemcpyHostToDevice));
    double* val;
    CK(cudaMalloc(&val, n * 8));
    CK(cudaMemset(val, 0, n * 8));
    CUtensorMap map;
    const cuuint64_t dims[2] = {2, n / 2};
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {2, 1};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, val, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      return 1;
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int mode = 0; mode < 3; ++mode) {
      for (int bps : {1, 2, 3, 4, 6, 8}) {
        if (mode && bps > 1) continue;  // 128 KB of stages per CTA
        const unsigned grid = sms * bps;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(e0));
          if (mode == 0)
            k_ldg<<<grid, kThreads>>>(idx, ngroups, val, out);
          else
            k_tma<<<grid, kThreads, kSmem>>>(map, idx, ngroups, val, out, mode);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          CK(cudaGetLastError());
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (rep && ms < best) best = ms;
        }
        const double gps = ngather / (best * 1e-3);
        printf("n=2^%d %-5s %d CTA/SM: %.3f ms  %.1f Ggather/s  %.3f gathers/SM/clk(base %d MHz)\n", log_n,
               mode == 0 ? "ldg" : mode == 1 ? "tma" : "mixed", bps, best, gps / 1e9,
               gps / sms / (clk_khz * 1e3), clk_khz / 1000);
      }
    }
    CK(cudaFree(val));
  }
  return 0;
}
