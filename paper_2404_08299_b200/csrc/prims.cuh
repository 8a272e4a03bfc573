// Device-wide primitives of the graph build / ingest / layout paths (north_star
// subsystem 5), hand-written for sm_100a: exclusive prefix sums, stable
// compaction (select / unique) and an LSD radix sort of 32- or 64-bit keys
// with optional 32-bit values.
//
// Every primitive is stream-ordered and allocation-free after the first call
// of a size (grow-only context workspace), and takes its element count
// either from the host or from a device counter (`count_dev`, with the host
// value an upper bound for the grid), so a chain of ingest kernels needs no
// host round trip to learn intermediate sizes.
//
// Scan and select are three-phase (tile reduce -> one-block scan of the tile
// totals -> tile apply): each pass is a coalesced stream, and the one-block
// middle phase touches only count / 2048 words.  The radix sort is the
// classic LSD pass per 8-bit digit -- tile histograms (digit-major, so one
// exclusive scan of the histogram yields every tile's scatter base) and a
// stable scatter whose in-tile ranks come from warp match-any groups (each
// warp owns a digit-counter row, so no shared-memory atomics).
#pragma once

#include <utility>

#include "common.cuh"

namespace dynpr_b200 {
namespace prims {
namespace {

constexpr int kPT = 256;            // threads per block (scan / select / sort)
constexpr int kPW = kPT / 32;
constexpr int kPI = 8;              // scan / select items per thread
constexpr int kPTile = kPT * kPI;   // 2048 items per tile
constexpr int kRI = 16;             // sort keys per thread (large inputs: 4096-key tiles)
constexpr int kRISmall = 4;         // (inputs up to kSmallSort keys: 1024-key tiles)
constexpr uint64_t kSmallSort = 1ull << 18;
constexpr uint64_t kLocalScanTiles = 64;  // scatter derives its bases itself up to this many tiles
constexpr unsigned kAll = 0xffffffffu;

__device__ __forceinline__ uint64_t dev_count(uint64_t count, const unsigned long long* cd) {
  return cd ? (uint64_t)*cd : count;
}

template <class T>
__device__ __forceinline__ T warp_incl_scan(T x) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(kAll, x, o);
    if ((int)lane >= o) x += y;
  }
  return x;
}

template <class T>
__device__ __forceinline__ T warp_total(T x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kAll, x, o);
  return x;
}

// Array loads (the common case of the functor-driven primitives).
template <class T>
struct Arr {
  const T* p;
  __device__ __forceinline__ T operator()(uint64_t i) const { return p[i]; }
};
template <class TO, class TI>
struct Widen {
  const TI* p;
  __device__ __forceinline__ TO operator()(uint64_t i) const { return (TO)p[i]; }
};
struct Iota32 {
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return (uint32_t)i; }
};
template <class T>
struct Nonzero {
  const T* p;
  __device__ __forceinline__ bool operator()(uint64_t i) const { return p[i] != 0; }
};
// unique(): keeps the first of every run of equal keys
template <class K>
struct RunHead {
  const K* p;
  __device__ __forceinline__ bool operator()(uint64_t i) const { return i == 0 || p[i] != p[i - 1]; }
};

// ---- scan ---------------------------------------------------------------------------
template <class T, class Load>
__global__ void __launch_bounds__(kPT) k_tile_sum(Load load, uint64_t count, const unsigned long long* cd,
                                                  T* partial) {
  __shared__ T s_w[kPW];
  const uint64_t n = dev_count(count, cd);
  const uint64_t base = (uint64_t)blockIdx.x * kPTile;
  T s = T(0);
#pragma unroll
  for (int j = 0; j < kPI; ++j) {
    const uint64_t i = base + (uint64_t)j * kPT + threadIdx.x;
    if (i < n) s += load(i);
  }
  s = warp_total(s);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = T(0);
#pragma unroll
    for (int w = 0; w < kPW; ++w) t += s_w[w];
    partial[blockIdx.x] = t;
  }
}

// One block: exclusive scan of the tile totals in place; *total = their sum.
// Each thread takes kScanR consecutive totals per round (8192 per round), so
// a 134 M-item scan (65536 tiles) runs 8 block rounds instead of 64.
constexpr int kScanR = 8;
template <class T>
__global__ void __launch_bounds__(1024) k_scan_tiles(T* partial, uint64_t ntiles, T* total) {
  __shared__ T s_w[32];
  __shared__ T s_carry;
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = T(0);
  __syncthreads();
  for (uint64_t b = 0; b < ntiles; b += 1024 * kScanR) {
    const uint64_t i0 = b + (uint64_t)threadIdx.x * kScanR;
    T x[kScanR];
    T sum = T(0);
#pragma unroll
    for (int r = 0; r < kScanR; ++r) {
      x[r] = i0 + r < ntiles ? partial[i0 + r] : T(0);
      sum += x[r];
    }
    const T inc = warp_incl_scan(sum);
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    if (w == 0) {
      const T y = s_w[lane];
      s_w[lane] = warp_incl_scan(y) - y;
    }
    __syncthreads();
    T ex = s_carry + s_w[w] + inc - sum;
#pragma unroll
    for (int r = 0; r < kScanR; ++r) {
      if (i0 + r < ntiles) partial[i0 + r] = ex;
      ex += x[r];
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = ex;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = s_carry;
}

// Tile apply: warp w owns items [base + 256 w, base + 256 w + 256) as 8
// coalesced rounds of 32; every item of the block is loaded before the
// block barrier, so `out` may alias the array `load` reads at i.
template <class T, class Load>
__global__ void __launch_bounds__(kPT) k_scan_apply(Load load, uint64_t count, const unsigned long long* cd,
                                                    const T* partial, T* out) {
  __shared__ T s_w[kPW];
  const uint64_t n = dev_count(count, cd);
  const uint64_t base = (uint64_t)blockIdx.x * kPTile;
  if (base >= n) return;  // whole block
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t wb = base + (uint64_t)w * (32 * kPI);
  T x[kPI];
  T ws = T(0);
#pragma unroll
  for (int r = 0; r < kPI; ++r) {
    const uint64_t i = wb + 32 * r + lane;
    x[r] = i < n ? load(i) : T(0);
    ws += x[r];
  }
  ws = warp_total(ws);
  if (lane == 0) s_w[w] = ws;
  __syncthreads();
  T off = partial[blockIdx.x];
  for (unsigned j = 0; j < w; ++j) off += s_w[j];
#pragma unroll
  for (int r = 0; r < kPI; ++r) {
    const T inc = warp_incl_scan(x[r]);
    const uint64_t i = wb + 32 * r + lane;
    if (i < n) out[i] = off + inc - x[r];
    off += __shfl_sync(kAll, inc, 31);
  }
}

// ---- select (stable compaction) ----------------------------------------------------------
template <class Flag>
__global__ void __launch_bounds__(kPT) k_tile_count(Flag flag, uint64_t count, const unsigned long long* cd,
                                                    unsigned long long* partial) {
  __shared__ unsigned s_w[kPW];
  const uint64_t n = dev_count(count, cd);
  const uint64_t base = (uint64_t)blockIdx.x * kPTile;
  unsigned c = 0;
#pragma unroll
  for (int j = 0; j < kPI; ++j) {
    const uint64_t i = base + (uint64_t)j * kPT + threadIdx.x;
    if (i < n && flag(i)) ++c;
  }
  c = warp_total(c);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
#pragma unroll
    for (int w = 0; w < kPW; ++w) t += s_w[w];
    partial[blockIdx.x] = t;
  }
}

template <class T, class Flag, class Val>
__global__ void __launch_bounds__(kPT) k_select_apply(Flag flag, Val val, uint64_t count,
                                                      const unsigned long long* cd,
                                                      const unsigned long long* partial, T* out) {
  __shared__ unsigned s_w[kPW];
  const uint64_t n = dev_count(count, cd);
  const uint64_t base = (uint64_t)blockIdx.x * kPTile;
  if (base >= n) return;
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t wb = base + (uint64_t)w * (32 * kPI);
  bool f[kPI];
  unsigned wc = 0;
#pragma unroll
  for (int r = 0; r < kPI; ++r) {
    const uint64_t i = wb + 32 * r + lane;
    f[r] = i < n && flag(i);
    wc += __popc(__ballot_sync(kAll, f[r]));
  }
  if (lane == 0) s_w[w] = wc;
  __syncthreads();
  unsigned long long off = partial[blockIdx.x];
  for (unsigned j = 0; j < w; ++j) off += s_w[j];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kPI; ++r) {
    const unsigned m = __ballot_sync(kAll, f[r]);
    if (f[r]) out[off + __popc(m & lt)] = val(wb + 32 * r + lane);
    off += __popc(m);
  }
}

// ---- radix sort -----------------------------------------------------------------------------
template <class K>
__device__ __forceinline__ unsigned digit_of(K k, int shift) {
  return (unsigned)(k >> shift) & 0xffu;
}

// Tile histograms (RI keys per thread), written digit-major:
// hist[d * ntiles + tile].
template <class K, int RI>
__global__ void __launch_bounds__(kPT) k_radix_hist(const K* __restrict__ keys, uint64_t n, int shift,
                                                    uint32_t* hist, uint64_t ntiles) {
  __shared__ uint32_t h[kPW][256];
  for (int i = threadIdx.x; i < kPW * 256; i += kPT) (&h[0][0])[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t wb = (uint64_t)blockIdx.x * (kPT * RI) + (uint64_t)w * (32 * RI);
#pragma unroll 4
  for (int r = 0; r < RI; ++r) {
    const uint64_t i = wb + 32 * r + lane;
    const bool valid = i < n;
    const unsigned d = valid ? digit_of(keys[i], shift) : 0x100u;
    const unsigned peers = __match_any_sync(kAll, d);
    if (valid && (int)lane == __ffs(peers) - 1) h[w][d] += __popc(peers);  // one writer per digit
    __syncwarp();
  }
  __syncthreads();
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kPW; ++j) c += h[j][threadIdx.x];  // thread t = digit t (kPT == 256)
  hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = c;
}

// Stable scatter: tile `base` from the scanned histogram, then warps in
// order, rounds in order, lanes in order (match-any peers below the lane).
// LOCAL: `hist` is the raw tile histogram (few tiles) and every block
// derives its own bases from it -- digit totals scanned over the digits plus
// the counts of the tiles before it -- instead of a separate scan pass.
template <class K, class V, bool HASV, int RI, bool LOCAL>
__global__ void __launch_bounds__(kPT) k_radix_scatter(const K* __restrict__ keys, const V* __restrict__ vals,
                                                       uint64_t n, int shift, const uint32_t* hist,
                                                       uint64_t ntiles, K* __restrict__ okeys,
                                                       V* __restrict__ ovals) {
  __shared__ uint32_t h[kPW][256];
  __shared__ uint32_t s_w[kPW];
  for (int i = threadIdx.x; i < kPW * 256; i += kPT) (&h[0][0])[i] = 0;
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t run;  // thread t = digit t: the tile's first output position for t
  if (LOCAL) {
    const uint32_t* ht = hist + (uint64_t)threadIdx.x * ntiles;
    uint32_t tot = 0, pre = 0;
    for (uint64_t j = 0; j < ntiles; ++j) {
      const uint32_t c = ht[j];
      tot += c;
      if (j < blockIdx.x) pre += c;
    }
    const uint32_t inc = warp_incl_scan(tot);
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t off = 0;
    for (unsigned j = 0; j < w; ++j) off += s_w[j];
    run = off + inc - tot + pre;
  } else {
    run = hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x];
  }
  __syncthreads();
  const uint64_t wb = (uint64_t)blockIdx.x * (kPT * RI) + (uint64_t)w * (32 * RI);
  K k[RI];
  V v[RI];
#pragma unroll
  for (int r = 0; r < RI; ++r) {
    const uint64_t i = wb + 32 * r + lane;
    k[r] = i < n ? keys[i] : K(0);
    if (HASV) v[r] = i < n ? vals[i] : V(0);
  }
#pragma unroll
  for (int r = 0; r < RI; ++r) {
    const bool valid = wb + 32 * r + lane < n;
    const unsigned d = valid ? digit_of(k[r], shift) : 0x100u;
    const unsigned peers = __match_any_sync(kAll, d);
    if (valid && (int)lane == __ffs(peers) - 1) h[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPW; ++j) {  // exclusive over the warps, from the tile's base
    const uint32_t c = h[j][threadIdx.x];
    h[j][threadIdx.x] = run;
    run += c;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < RI; ++r) {
    const bool valid = wb + 32 * r + lane < n;
    const unsigned d = valid ? digit_of(k[r], shift) : 0x100u;
    const unsigned peers = __match_any_sync(kAll, d);
    uint32_t pos = 0;
    if (valid) pos = h[w][d] + __popc(peers & lt);
    __syncwarp();
    if (valid && (int)lane == __ffs(peers) - 1) h[w][d] += __popc(peers);
    __syncwarp();
    if (valid) {
      okeys[pos] = k[r];
      if (HASV) ovals[pos] = v[r];
    }
  }
}

// Staged scatter (large inputs): the tile is first ordered by digit in
// shared memory, then written out as runs -- consecutive threads write
// consecutive positions of one digit bucket, so the stores coalesce (the
// direct scatter wrote 8-byte keys at up to 32 buckets per warp
// instruction).  Same stable order as k_radix_scatter.
template <class K, class V, bool HASV, int RI>
__global__ void __launch_bounds__(kPT) k_radix_scatter_staged(const K* __restrict__ keys, const V* __restrict__ vals,
                                                              uint64_t n, int shift, const uint32_t* hist,
                                                              uint64_t ntiles, K* __restrict__ okeys,
                                                              V* __restrict__ ovals) {
  extern __shared__ unsigned char s_dyn[];
  K* s_k = reinterpret_cast<K*>(s_dyn);
  V* s_v = reinterpret_cast<V*>(s_dyn + sizeof(K) * kPT * RI);
  __shared__ uint32_t h[kPW][256];
  __shared__ uint32_t s_start[256];  // tile-local start of each digit
  __shared__ uint32_t s_gbase[256];  // global start of each digit for this tile
  __shared__ uint32_t s_w[kPW];
  for (int i = threadIdx.x; i < kPW * 256; i += kPT) (&h[0][0])[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t tb = (uint64_t)blockIdx.x * (kPT * RI);
  const uint64_t wb = tb + (uint64_t)w * (32 * RI);
  K k[RI];
  V v[RI];
#pragma unroll
  for (int r = 0; r < RI; ++r) {
    const uint64_t i = wb + 32 * r + lane;
    k[r] = i < n ? keys[i] : K(0);
    if (HASV) v[r] = i < n ? vals[i] : V(0);
  }
#pragma unroll
  for (int r = 0; r < RI; ++r) {
    const bool valid = wb + 32 * r + lane < n;
    const unsigned d = valid ? digit_of(k[r], shift) : 0x100u;
    const unsigned peers = __match_any_sync(kAll, d);
    if (valid && (int)lane == __ffs(peers) - 1) h[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {  // thread t = digit t: tile total, exclusive scan over digits, warps' starts
    uint32_t tot = 0;
#pragma unroll
    for (int j = 0; j < kPW; ++j) tot += h[j][threadIdx.x];
    const uint32_t inc = warp_incl_scan(tot);
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t off = 0;
    for (unsigned j = 0; j < w; ++j) off += s_w[j];
    uint32_t run = off + inc - tot;
    s_start[threadIdx.x] = run;
    s_gbase[threadIdx.x] = hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x];
#pragma unroll
    for (int j = 0; j < kPW; ++j) {
      const uint32_t c = h[j][threadIdx.x];
      h[j][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < RI; ++r) {
    const bool valid = wb + 32 * r + lane < n;
    const unsigned d = valid ? digit_of(k[r], shift) : 0x100u;
    const unsigned peers = __match_any_sync(kAll, d);
    uint32_t pos = 0;
    if (valid) pos = h[w][d] + __popc(peers & lt);
    __syncwarp();
    if (valid && (int)lane == __ffs(peers) - 1) h[w][d] += __popc(peers);
    __syncwarp();
    if (valid) {
      s_k[pos] = k[r];
      if (HASV) s_v[pos] = v[r];
    }
  }
  __syncthreads();
  const uint32_t cnt = n - tb < (uint64_t)(kPT * RI) ? (uint32_t)(n - tb) : (uint32_t)(kPT * RI);
  for (uint32_t i = threadIdx.x; i < cnt; i += kPT) {
    const K key = s_k[i];
    const unsigned d = digit_of(key, shift);
    const uint32_t g = s_gbase[d] + (i - s_start[d]);
    okeys[g] = key;
    if (HASV) ovals[g] = s_v[i];
  }
}

}  // namespace

// ---- host entry points ------------------------------------------------------------------
// out[i] = sum of load(j) for j < i, i < count (or *count_dev); *total (device)
// = the sum of all.  `out` may be the array `load` reads element-wise.
template <class T, class Load>
void scan_exclusive(dynpr_context* ctx, Load load, T* out, uint64_t count, cudaStream_t st, T* total = nullptr,
                    const unsigned long long* count_dev = nullptr) {
  const uint64_t ntiles = (count + kPTile - 1) / kPTile;
  if (!ntiles) {
    if (total) DYNPR_CK(cudaMemsetAsync(total, 0, sizeof(T), st));
    return;
  }
  T* partial = ctx->prims_tmp.as<T>(ntiles + 1);
  k_tile_sum<T><<<(unsigned)ntiles, kPT, 0, st>>>(load, count, count_dev, partial);
  k_scan_tiles<T><<<1, 1024, 0, st>>>(partial, ntiles, total);
  k_scan_apply<T><<<(unsigned)ntiles, kPT, 0, st>>>(load, count, count_dev, partial, out);
  check_launch();
  count_launch(ctx, 3);
}
template <class T>
void scan_array(dynpr_context* ctx, const T* in, T* out, uint64_t count, cudaStream_t st, T* total = nullptr,
                const unsigned long long* count_dev = nullptr) {
  scan_exclusive<T>(ctx, Arr<T>{in}, out, count, st, total, count_dev);
}

// Stable compaction: out[0..*num) = val(i) for the i < count (or *count_dev)
// with flag(i), in order; *num is a device counter.
template <class T, class Flag, class Val>
void select_if(dynpr_context* ctx, Flag flag, Val val, uint64_t count, T* out, unsigned long long* num,
               cudaStream_t st, const unsigned long long* count_dev = nullptr) {
  const uint64_t ntiles = (count + kPTile - 1) / kPTile;
  if (!ntiles) {
    DYNPR_CK(cudaMemsetAsync(num, 0, sizeof(unsigned long long), st));
    return;
  }
  auto* partial = ctx->prims_tmp.as<unsigned long long>(ntiles + 1);
  k_tile_count<<<(unsigned)ntiles, kPT, 0, st>>>(flag, count, count_dev, partial);
  k_scan_tiles<unsigned long long><<<1, 1024, 0, st>>>(partial, ntiles, num);
  k_select_apply<T><<<(unsigned)ntiles, kPT, 0, st>>>(flag, val, count, count_dev, partial, out);
  check_launch();
  count_launch(ctx, 3);
}

// Sorted keys -> the first of every run of equal keys (std::unique).
template <class K>
void unique_sorted(dynpr_context* ctx, const K* keys, uint64_t count, K* out, unsigned long long* num,
                   cudaStream_t st, const unsigned long long* count_dev = nullptr) {
  select_if<K>(ctx, RunHead<K>{keys}, Arr<K>{keys}, count, out, num, st, count_dev);
}

// Stable LSD radix sort of n keys on bits [begin_bit, end_bit) (higher
// bits zero), 8 bits per pass, ping-ponging between (keys, vals) and
// (keys_alt, vals_alt); returns the buffer holding the sorted keys and sets
// *vals_out to the matching values buffer.  vals may be null (keys only).
template <class K, class V, int RI>
void radix_pass(dynpr_context* ctx, const K* ks, const V* vs, uint64_t n, int shift, K* kd, V* vd, cudaStream_t st) {
  constexpr uint64_t tile = (uint64_t)kPT * RI;
  const uint64_t ntiles = (n + tile - 1) / tile;
  uint32_t* hist = ctx->sort_hist.as<uint32_t>(256 * ntiles);
  k_radix_hist<K, RI><<<(unsigned)ntiles, kPT, 0, st>>>(ks, n, shift, hist, ntiles);
  check_launch();
  count_launch(ctx);
  if (ntiles <= kLocalScanTiles) {
    if (vs)
      k_radix_scatter<K, V, true, RI, true><<<(unsigned)ntiles, kPT, 0, st>>>(ks, vs, n, shift, hist, ntiles, kd, vd);
    else
      k_radix_scatter<K, V, false, RI, true><<<(unsigned)ntiles, kPT, 0, st>>>(ks, vs, n, shift, hist, ntiles, kd, vd);
  } else {
    scan_array<uint32_t>(ctx, hist, hist, 256 * ntiles, st);
    const size_t smem = (size_t)kPT * RI * (sizeof(K) + (vs ? sizeof(V) : 0));
    if (vs) {
      auto kern = k_radix_scatter_staged<K, V, true, RI>;
      DYNPR_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<(unsigned)ntiles, kPT, smem, st>>>(ks, vs, n, shift, hist, ntiles, kd, vd);
    } else {
      auto kern = k_radix_scatter_staged<K, V, false, RI>;
      DYNPR_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<(unsigned)ntiles, kPT, smem, st>>>(ks, vs, n, shift, hist, ntiles, kd, vd);
    }
  }
  check_launch();
  count_launch(ctx);
}

// Stable LSD radix sort of n keys on bits [begin_bit, end_bit) (higher
// bits zero), 8 bits per pass, ping-ponging between (keys, vals) and
// (keys_alt, vals_alt); returns the buffer holding the sorted keys and sets
// *vals_out to the matching values buffer.  vals may be null (keys only).
// Small inputs (batch lists) use 1024-key tiles so the passes spread over
// the SMs, and derive the tile bases inside the scatter (2 launches a pass).
template <class K, class V>
K* radix_sort(dynpr_context* ctx, K* keys, K* keys_alt, V* vals, V* vals_alt, uint64_t n, int begin_bit,
              int end_bit, cudaStream_t st, V** vals_out = nullptr) {
  if (n >= (1ull << 32)) invalid("radix sort: more than 2^32 keys");
  K* ks = keys;
  K* kd = keys_alt;
  V* vs = vals;
  V* vd = vals_alt;
  if (n > 1 && end_bit > begin_bit) {
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
      if (n <= kSmallSort)
        radix_pass<K, V, kRISmall>(ctx, ks, vs, n, shift, kd, vd, st);
      else
        radix_pass<K, V, kRI>(ctx, ks, vs, n, shift, kd, vd, st);
      std::swap(ks, kd);
      std::swap(vs, vd);
    }
  }
  if (vals_out) *vals_out = vs;
  return ks;
}

namespace {
__global__ void __launch_bounds__(kPT) k_reduce_max_u32(const uint32_t* a, uint64_t n, unsigned* out) {
  unsigned m = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * kPT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kPT) m = max(m, a[i]);
  m = __reduce_max_sync(kAll, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
}  // namespace

// max of n u32 values into *out (device; zeroed here first).
inline void reduce_max_u32(dynpr_context* ctx, const uint32_t* a, uint64_t n, unsigned* out, cudaStream_t st) {
  DYNPR_CK(cudaMemsetAsync(out, 0, sizeof(unsigned), st));
  if (n) {
    k_reduce_max_u32<<<grid_for(n, kPT, ctx->num_sms * 8), kPT, 0, st>>>(a, n, out);
    check_launch();
    count_launch(ctx);
  }
}

}  // namespace prims
}  // namespace dynpr_b200
