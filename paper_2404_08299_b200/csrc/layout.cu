// Builder of the engine layout (see layout.cuh): degree sort, relabelling,
// SELL-32 segment slices, relabelled forward CSR.
#include "comm.cuh"
#include "layout.cuh"
#include "prims.cuh"
#include "sweep.cuh"

namespace dynpr_b200 {

namespace {

// Layout arrays come from the building context's pool (explicit, so
// contexts building layouts concurrently on several host threads never
// share allocation state).
template <class T>
T* dalloc(dynpr_context* ctx, uint64_t count) {
  return pool_alloc_n<T>(ctx, count ? count : 1);
}

#define GRID_STRIDE(i, count)                                                      \
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (count); \
       i += (uint64_t)gridDim.x * blockDim.x)

__global__ void k_degrees_keys(const uint64_t* offT, const uint64_t* offF, uint32_t n, uint32_t* indeg_old,
                               uint32_t* outdeg_old, uint32_t* iota) {
  GRID_STRIDE(v, n) {
    indeg_old[v] = (uint32_t)(offT[v + 1] - offT[v]);
    outdeg_old[v] = (uint32_t)(offF[v + 1] - offF[v]);
    iota[v] = (uint32_t)v;
  }
}
__global__ void k_desc_keys(const uint32_t* deg, uint32_t n, uint32_t maxdeg, uint32_t* keys) {
  GRID_STRIDE(v, n) keys[v] = maxdeg - deg[v];
}
__global__ void k_relabel(const uint32_t* perm, uint32_t n, const uint32_t* indeg_old, const uint32_t* outdeg_old,
                          uint32_t* inv, uint32_t* indeg, uint32_t* outdeg) {
  GRID_STRIDE(i, n) {
    const uint32_t o = perm[i];
    inv[o] = (uint32_t)i;
    indeg[i] = indeg_old[o];
    outdeg[i] = outdeg_old[o];
  }
}
// M = number of vertices with in-degree > thr (a prefix: degrees descend)
__global__ void k_count_above(const uint32_t* indeg, uint32_t n, uint32_t thr, unsigned* out) {
  unsigned c = 0;
  GRID_STRIDE(i, n) c += indeg[i] > thr;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
// single region: slice lengths (x32) for the exclusive scan
__global__ void k_single_slice_len(const uint32_t* indeg, uint32_t M, uint32_t n, uint64_t S, uint64_t* len32) {
  GRID_STRIDE(s, S + 1) len32[s] = s < S ? 32ull * ((indeg[M + 32 * s] + 3u) & ~3u) : 0ull;
}
// multi region: chunk counts per multi vertex
__global__ void k_multi_nch(const uint32_t* indeg, uint32_t M, uint32_t* nch) {
  GRID_STRIDE(v, (uint64_t)M + 1) nch[v] = v < M ? (indeg[v] + 255u) / 256u : 0u;
}
__global__ void k_multi_segments(const uint32_t* indeg, uint32_t M, const uint32_t* pbase, uint32_t* mseg_v,
                                 uint32_t* mseg_len) {
  GRID_STRIDE(v, M) {
    const uint32_t d = indeg[v], b = pbase[v];
    const uint32_t nch = (d + 255u) / 256u;
    for (uint32_t j = 0; j < nch; ++j) {
      mseg_v[b + j] = (uint32_t)v;
      mseg_len[b + j] = (j + 1 < nch) ? 256u : d - 256u * j;
    }
  }
}
__global__ void k_multi_slice_len(const uint32_t* mseg_len, uint64_t nseg, uint64_t S, uint64_t* len32) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t s = warp; s <= S; s += nw) {
    const uint64_t seg = s * 32 + lane;
    const unsigned l = (s < S && seg < nseg) ? mseg_len[seg] : 0u;
    const unsigned mx = __reduce_max_sync(0xffffffffu, l);
    if (lane == 0) len32[s] = 32ull * ((mx + 3u) & ~3u);
  }
}
// One lane's segment into SELL-32x4: 4 consecutive elements per 16-byte
// store, so each warp store covers 512 contiguous bytes.
// 16 elements per round: the 16 source loads, then the 16 relabel gathers,
// are independent (one round trip each instead of one per element pair)
__device__ __forceinline__ void fill_lane(uint32_t* sell, uint64_t base, unsigned lane, uint32_t L, uint32_t len,
                                          const uint32_t* src, const uint32_t* inv) {
  for (uint32_t k = 0; k < L; k += 16) {
    uint32_t x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = k + q < len ? src[k + q] : 0u;
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = k + q < len ? inv[x[q]] : 0u;
#pragma unroll
    for (int q = 0; q < 16; q += 4)
      if (k + q < L) *reinterpret_cast<uint4*>(sell + sell_pos(base, lane, k + q)) =
          make_uint4(x[q], x[q + 1], x[q + 2], x[q + 3]);
  }
}

// SELL fill, single region: warp per slice, lane per vertex
__global__ void k_fill_single(const uint64_t* offT, const uint32_t* tgtT, const uint32_t* perm, const uint32_t* inv,
                              const uint32_t* indeg, uint32_t M, uint32_t n, uint64_t s_lo, uint64_t s_hi,
                              const uint64_t* sbase, uint32_t* sell) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t s = s_lo + warp; s < s_hi; s += nw) {
    const uint64_t vn = M + s * 32 + lane;
    const bool valid = vn < n;
    const uint32_t deg = valid ? indeg[vn] : 0u;
    const uint64_t src = valid ? offT[perm[vn]] : 0;
    const uint64_t base = sbase[s];
    const uint32_t L = (uint32_t)((sbase[s + 1] - base) / 32);
    fill_lane(sell, base, lane, L, deg, tgtT + src, inv);
  }
}
// SELL fill, multi region: warp per slice, lane per 256-edge segment
__global__ void k_fill_multi(const uint64_t* offT, const uint32_t* tgtT, const uint32_t* perm, const uint32_t* inv,
                             const uint32_t* pbase, const uint32_t* mseg_v, const uint32_t* mseg_len, uint64_t nseg,
                             uint64_t s_lo, uint64_t s_hi, const uint64_t* mbase, uint32_t* sell) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t s = s_lo + warp; s < s_hi; s += nw) {
    const uint64_t seg = s * 32 + lane;
    const bool valid = seg < nseg;
    uint32_t len = 0;
    uint64_t src = 0;
    if (valid) {
      const uint32_t v = mseg_v[seg];
      len = mseg_len[seg];
      src = offT[perm[v]] + 256ull * (seg - pbase[v]);
    }
    const uint64_t base = mbase[s];
    const uint32_t L = (uint32_t)((mbase[s + 1] - base) / 32);
    fill_lane(sell, base, lane, L, len, tgtT + src, inv);
  }
}
// relabelled forward CSR: warp per new vertex
__global__ void k_outdeg64(const uint32_t* outdeg, uint32_t n, uint64_t* off) {
  GRID_STRIDE(v, (uint64_t)n + 1) off[v] = v < n ? outdeg[v] : 0ull;
}
// Relabelled forward CSR (rows and columns in new ids): the output is cut
// into fixed 1024-element chunks, warp per chunk, so a hub row (RMAT-24:
// ~4e5 out-edges) is spread over hundreds of warps and a run of short rows
// keeps all 32 lanes busy.  The row of output element `pos` is found by a
// binary search of the new offsets restricted to the chunk's row range (a
// few L1-resident probes); 4 elements in flight per lane.
constexpr uint64_t kFillChunk = 1024;
__device__ __forceinline__ uint64_t last_le(const uint64_t* off, uint64_t lo, uint64_t hi, uint64_t pos) {
  // last w in [lo, hi] with off[w] <= pos (off[lo] <= pos guaranteed)
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= pos) lo = mid; else hi = mid - 1;
  }
  return lo;
}
__global__ void k_fill_forward(const uint64_t* offF, const uint32_t* tgtF, const uint32_t* perm, const uint32_t* inv,
                               uint32_t n, const uint64_t* noff, uint32_t* ntgt) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  const uint64_t m = noff[n];
  const uint64_t nchunks = (m + kFillChunk - 1) / kFillChunk;
  for (uint64_t c = warp; c < nchunks; c += nw) {
    const uint64_t p0 = c * kFillChunk, p1 = p0 + kFillChunk < m ? p0 + kFillChunk : m;
    uint64_t w0 = 0, w1 = 0;
    if (lane == 0) w0 = last_le(noff, 0, n - 1, p0);
    if (lane == 1) w1 = last_le(noff, 0, n - 1, p1 - 1);
    w0 = __shfl_sync(0xffffffffu, w0, 0);
    w1 = __shfl_sync(0xffffffffu, w1, 1);
    for (uint64_t base = p0; base < p1; base += 128) {
      uint32_t x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t pos = base + 32 * q + lane;
        x[q] = 0;
        if (pos < p1) {
          const uint64_t w = last_le(noff, w0, w1, pos);
          x[q] = tgtF[offF[perm[w]] + (pos - noff[w])];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t pos = base + 32 * q + lane;
        if (pos < p1) ntgt[pos] = inv[x[q]];
      }
    }
  }
}

__global__ void k_gather_perm_f64(const uint32_t* perm, uint32_t n, const double* src, double* dst) {
  GRID_STRIDE(i, n) dst[i] = src[perm[i]];
}
__global__ void k_gather_perm_u8(const uint32_t* perm, uint32_t n, const uint8_t* src, uint8_t* dst) {
  GRID_STRIDE(i, n) dst[i] = src[perm[i]];
}
__global__ void k_scatter_inv_f64(const uint32_t* inv, uint32_t n, const double* src, double* dst) {
  GRID_STRIDE(o, n) dst[o] = src[inv[o]];
}
__global__ void k_scatter_inv_u8(const uint32_t* inv, uint32_t n, const uint8_t* src, uint8_t* dst) {
  GRID_STRIDE(o, n) dst[o] = src[inv[o]];
}


// A SELL block owned (shared) by layout L: freed when the last layout
// reading it goes.
uint32_t* new_block(dynpr_context* ctx, Layout* L, uint64_t words) {
  uint32_t* p = dalloc<uint32_t>(ctx, words);
  L->blocks.emplace_back(p, [ctx](uint32_t* q) { pool_free(ctx, q); });
  return p;
}
// 64-bit element offset of `p` from base `b` (two's complement when p < b):
// `b + offset` addresses p
uint64_t rel_words(const uint32_t* b, const uint32_t* p) {
  const int64_t bytes = (int64_t)((uintptr_t)p - (uintptr_t)b);
  return (uint64_t)(bytes / 4);
}

// ---- incremental derivation (build_incremental) --------------------------------
// touched rows (old ids): flag in the relabelled space + the new degree
__global__ void k_mark_rows(const uint32_t* rows, uint64_t cnt, const uint32_t* inv, const uint64_t* off,
                            uint8_t* flag, uint32_t* deg) {
  GRID_STRIDE(i, cnt) {
    const uint32_t u = rows[i], w = inv[u];
    flag[w] = 1;
    deg[w] = (uint32_t)(off[u + 1] - off[u]);
  }
}
// single region, stale order: slice length = the longest of its 32 segments
__global__ void k_single_slice_len_max(const uint32_t* indeg, uint32_t M, uint32_t n, uint64_t S, uint64_t* len32) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t s = warp; s <= S; s += nw) {
    const uint64_t v = (uint64_t)M + 32 * s + lane;
    const unsigned d = (s < S && v < n) ? indeg[v] : 0u;
    const unsigned mx = __reduce_max_sync(0xffffffffu, d);
    if (lane == 0) len32[s] = 32ull * ((mx + 3u) & ~3u);
  }
}
// One lane's segment copied from its position in the parent layout (column
// ids are in the same relabelled space): 16-byte groups, zero padding.
__device__ __forceinline__ void copy_lane(uint32_t* sell, uint64_t base, unsigned lane, uint32_t L, uint32_t len,
                                          const uint32_t* old, uint64_t obase, unsigned olane) {
  for (uint32_t k = 0; k < L; k += 4) {
    const uint4 w = k < len ? *reinterpret_cast<const uint4*>(old + sell_pos(obase, olane, k)) : make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(sell + sell_pos(base, lane, k)) = w;
  }
}
// single region, copy-on-write: a slice is re-built iff one of its vertices'
// in-lists changed; its length is then the longest of its 32 new segments
// (the relabelling is no longer sorted), else it is shared.
// Driven by the touched rows (old ids), O(batch) instead of a pass over
// every slice: a warp per touched single-region vertex computes its slice's
// length (len32 zeroed before; two touched vertices of one slice write the
// same value).
__global__ void k_slice_touched_len_rows(const uint32_t* rows, uint64_t cnt, const uint32_t* inv,
                                         const uint32_t* indeg, uint32_t M, uint32_t n, uint64_t* len32) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t i = warp; i < cnt; i += nw) {
    const uint32_t vn = inv[rows[i]];
    if (vn < M) continue;  // (warp-uniform) multi region
    const uint64_t s = (vn - (uint64_t)M) / 32;
    const uint64_t v = (uint64_t)M + 32 * s + lane;
    const unsigned d = v < n ? indeg[v] : 0u;
    const unsigned mx = __reduce_max_sync(0xffffffffu, d);
    if (lane == 0) len32[s] = 32ull * ((mx + 3u) & ~3u);
  }
}
__global__ void k_sbase_cow(const uint64_t* sbase0, const uint64_t* len32, const uint64_t* dpos, uint64_t S,
                            uint64_t rel, uint64_t* sbase) {
  GRID_STRIDE(s, S + 1) sbase[s] = (s < S && len32[s]) ? rel + dpos[s] : sbase0[s];
}
// A warp per touched single-region vertex rebuilds its slice: touched lanes
// re-gathered, the others copied from the parent (a slice holding several
// touched vertices is rebuilt once per vertex, with identical words).
__global__ void k_fill_single_cow_rows(const uint32_t* rows, uint64_t cnt, const uint64_t* offT, const uint32_t* tgtT,
                                       const uint32_t* perm, const uint32_t* inv, const uint32_t* indeg, uint32_t M,
                                       uint32_t n, const uint64_t* len32, const uint64_t* sbase, uint32_t* sell,
                                       const uint8_t* touched, const uint64_t* sbase0) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t i = warp; i < cnt; i += nw) {
    const uint32_t w = inv[rows[i]];
    if (w < M) continue;  // (warp-uniform) multi region
    const uint64_t s = (w - (uint64_t)M) / 32;
    const uint32_t L = (uint32_t)(len32[s] / 32);
    const uint64_t vn = (uint64_t)M + s * 32 + lane;
    const bool valid = vn < n;
    const uint32_t deg = valid ? indeg[vn] : 0u;
    if (valid && touched[vn])
      fill_lane(sell, sbase[s], lane, L, deg, tgtT + offT[perm[vn]], inv);
    else
      copy_lane(sell, sbase[s], lane, L, deg, sell, sbase0[s], lane);
  }
}
// multi region, copy-on-write: the chunks of a vertex whose in-list changed
// are retired in place (length 0: every sweep skips them) and re-built as
// new segments appended after the parent's (from a slice boundary on); the
// vertex's pbase points to them.  Untouched vertices keep their slices.
__global__ void k_multi_touched_nch(const uint32_t* indeg, const uint8_t* touched, uint32_t M, uint32_t* nch) {
  GRID_STRIDE(v, (uint64_t)M + 1) nch[v] = (v < M && touched[v]) ? (indeg[v] + 255u) / 256u : 0u;
}
// A warp per touched multi vertex, its lanes striding over the chunks (a
// hub's thousands of chunks are not one thread's serial loop).
__global__ void k_multi_cow_segments_rows(const uint32_t* rows, uint64_t cnt, const uint32_t* inv,
                                          const uint32_t* indeg, const uint32_t* indeg0, uint32_t M,
                                          const uint32_t* apos, uint64_t first, const uint32_t* pbase0,
                                          uint32_t* pbase, uint32_t* mseg_v, uint32_t* mseg_len) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t i = warp; i < cnt; i += nw) {
    const uint32_t v = inv[rows[i]];
    if (v >= M) continue;  // (warp-uniform) single region
    const uint32_t d0 = indeg0[v], p0 = pbase0[v];
    for (uint32_t j = lane; j < (d0 + 255u) / 256u; j += 32) mseg_len[p0 + j] = 0u;  // retired
    const uint32_t d = indeg[v], b = (uint32_t)(first + apos[v]);
    const uint32_t nch = (d + 255u) / 256u;
    if (lane == 0) pbase[v] = b;
    for (uint32_t j = lane; j < nch; j += 32) {
      mseg_v[b + j] = v;
      mseg_len[b + j] = (j + 1 < nch) ? 256u : d - 256u * j;
    }
  }
}
__global__ void k_mbase_append(uint64_t* mbase, uint64_t s0, uint64_t cnt, uint64_t rel) {
  GRID_STRIDE(i, cnt + 1) mbase[s0 + i] += rel;
}

// relabelled forward CSR, touched rows (the untouched ones are copied as
// runs, graph.cu copy_untouched_rows): rows cut into 4K-element items so a
// touched hub spreads over many warps; item t -> row by binary search of the
// items' exclusive scan.  rows: old ids of the touched forward rows.
constexpr uint64_t kRowItem = 4096;
struct RowWords {  // new out-degree of touched row j (0 past the list)
  const uint32_t* rows;
  const uint32_t* inv;
  const uint32_t* outdeg;
  uint64_t c;
  __device__ __forceinline__ unsigned long long operator()(uint64_t j) const {
    return j < c ? (unsigned long long)outdeg[inv[rows[j]]] : 0ull;
  }
};
struct RowChunks {
  const uint32_t* rows;
  const uint32_t* inv;
  const uint32_t* outdeg;
  uint64_t c;
  __device__ __forceinline__ uint32_t operator()(uint64_t j) const {
    return j < c ? (uint32_t)((outdeg[inv[rows[j]]] + kRowItem - 1) / kRowItem) : 0u;
  }
};
// Touched row j (old id u, new id w) rewritten into the new block at
// wpos[j]: relabelled targets of the new forward graph's row u; the first
// item of the row re-points begF[w] (blk_rel: the block's offset from the
// shared base).
__global__ void k_refill_rows(const uint32_t* rows, uint64_t c, const uint32_t* istart, const unsigned long long* wpos,
                              const uint64_t* offF, const uint32_t* tgtF, const uint32_t* inv, uint64_t blk_rel,
                              const uint32_t* base, uint64_t* begF, uint32_t* blk) {
  const uint32_t total = istart[c];
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  (void)base;
  for (uint64_t t = warp; t < total; t += nw) {
    const uint64_t j = upper_bound_u32(istart, c + 1, (uint32_t)t) - 1;
    const uint32_t u = rows[j], w = inv[u];
    const uint64_t len = offF[u + 1] - offF[u];
    const uint64_t k0 = (t - istart[j]) * kRowItem, k1 = k0 + kRowItem < len ? k0 + kRowItem : len;
    const uint32_t* src = tgtF + offF[u];
    uint32_t* dst = blk + wpos[j];
    if (k0 == 0 && lane == 0) begF[w] = blk_rel + wpos[j];
    for (uint64_t kb = k0; kb < k1; kb += 32 * 8) {  // 8 loads, then 8 gathers, in flight per lane
      uint32_t x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint64_t k = kb + 32 * q + lane;
        x[q] = k < k1 ? src[k] : 0u;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint64_t k = kb + 32 * q + lane;
        if (k < k1) x[q] = inv[x[q]];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint64_t k = kb + 32 * q + lane;
        if (k < k1) dst[k] = x[q];
      }
    }
  }
}

unsigned grid(dynpr_context* ctx, uint64_t items) { return grid_for(items, 256, ctx->num_sms * 32); }

uint64_t read_u64(dynpr_context* ctx, const void* d) {
  uint64_t h = 0;
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  std::memcpy(&h, ctx->pinned, 8);
  return h;
}

// The relabelled forward graph of a full build: CSR order, so begF is the
// exclusive scan of the out-degrees (n + 1 entries); its target array is a
// shared block that derived layouts keep reading (copy-on-write rows).
void build_forward(dynpr_context* ctx, Layout* L, const dynpr_graph* gF) {
  cudaStream_t st = ctx->stream;
  L->begF = dalloc<uint64_t>(ctx, (uint64_t)L->n + 1);
  L->tgtF = new_block(ctx, L, L->m);
  L->fwd_words = L->m;
  k_outdeg64<<<grid(ctx, (uint64_t)L->n + 1), 256, 0, st>>>(L->outdeg, L->n, L->begF);
  check_launch();
  prims::scan_array(ctx, L->begF, L->begF, (uint64_t)L->n + 1, st);
  k_fill_forward<<<grid(ctx, (L->m + kFillChunk - 1) / kFillChunk * 32), 256, 0, st>>>(
      gF->off, gF->tgt, L->perm, L->inv, L->n, L->begF, L->tgtF);
  check_launch();
  count_launch(ctx, 2);
  L->has_forward = true;
}

Layout* build_layout(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF, uint32_t T) {
  cudaStream_t st = ctx->stream;
  const uint32_t n = gT->n;
  auto* L = new Layout();
  L->ctx = ctx;
  uint32_t* tmp = nullptr;
  try {
    L->n = n;
    L->m = gT->m;
    L->T = T;
    L->gF_id = gF->id;
    L->loops = gT->all_loops;
    // the relabelling: shared blocks (derived layouts keep the order)
    L->perm = new_block(ctx, L, n);
    L->inv = new_block(ctx, L, n);
    L->indeg = dalloc<uint32_t>(ctx, n);
    L->outdeg = dalloc<uint32_t>(ctx, n);
    // temporaries from the pool (the context's stage buffers may hold the
    // caller's staged inputs when the build happens inside an engine call)
    // temporaries in a context-owned grow-only buffer: a pool allocation of
    // this size per snapshot occasionally had to map fresh memory (measured
    // up to 74 ms inside the ingest)
    tmp = ctx->layout_tmp.as<uint32_t>(5ull * ((uint64_t)n + 1));
    uint32_t* indeg_old = tmp;
    uint32_t* outdeg_old = tmp + (n + 1ull);
    uint32_t* keys = tmp + 2ull * (n + 1ull);
    uint32_t* keys2 = tmp + 3ull * (n + 1ull);
    uint32_t* iota = tmp + 4ull * (n + 1ull);
    k_degrees_keys<<<grid(ctx, n), 256, 0, st>>>(gT->off, gF->off, n, indeg_old, outdeg_old, iota);
    check_launch();
    // max in-degree -> descending sort keys
    auto* mx = reinterpret_cast<uint32_t*>(ctx->scratch64a.as<unsigned long long>(2));
    prims::reduce_max_u32(ctx, indeg_old, n, mx, st);
    const uint32_t maxdeg = (uint32_t)(read_u64(ctx, mx) & 0xffffffffu);
    k_desc_keys<<<grid(ctx, n), 256, 0, st>>>(indeg_old, n, maxdeg, keys);
    check_launch();
    count_launch(ctx, 2);
    const int eb = bits_for(maxdeg);
    if (eb > 0) {
      uint32_t* vsorted = nullptr;
      prims::radix_sort<uint32_t, uint32_t>(ctx, keys, keys2, iota, L->perm, n, 0, eb, st, &vsorted);
      if (vsorted != L->perm)
        DYNPR_CK(cudaMemcpyAsync(L->perm, vsorted, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      DYNPR_CK(cudaMemcpyAsync(L->perm, iota, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    }
    k_relabel<<<grid(ctx, n), 256, 0, st>>>(L->perm, n, indeg_old, outdeg_old, L->inv, L->indeg, L->outdeg);
    check_launch();
    // multi vertices: in-degree > max(T, 256)
    const uint32_t thr = T > 256u ? T : 256u;
    auto* cnt = reinterpret_cast<unsigned*>(ctx->scratch64a.as<unsigned long long>(2));
    DYNPR_CK(cudaMemsetAsync(cnt, 0, 8, st));
    k_count_above<<<grid(ctx, n), 256, 0, st>>>(L->indeg, n, thr, cnt);
    check_launch();
    count_launch(ctx, 2);
    L->M = (uint32_t)(read_u64(ctx, cnt) & 0xffffffffu);
    const uint32_t M = L->M;
    DYNPR_CK(cudaMemsetAsync(cnt, 0, 8, st));
    k_count_above<<<grid(ctx, n), 256, 0, st>>>(L->indeg, n, kHeavyDeg < thr ? kHeavyDeg : thr, cnt);
    check_launch();
    count_launch(ctx);
    {
      const uint32_t nh = (uint32_t)(read_u64(ctx, cnt) & 0xffffffffu);
      L->n_hslices = nh > M ? ((uint64_t)(nh - M) + 31) / 32 : 0;
    }
    L->mcount = dalloc<uint32_t>(ctx, (uint64_t)M + 1);
    DYNPR_CK(cudaMemsetAsync(L->mcount, 0, ((size_t)M + 1) * 4, st));
    // single region slices
    L->n_sslices = ((uint64_t)(n - M) + 31) / 32;
    L->sbase = dalloc<uint64_t>(ctx, L->n_sslices + 1);
    k_single_slice_len<<<grid(ctx, L->n_sslices + 1), 256, 0, st>>>(L->indeg, M, n, L->n_sslices, L->sbase);
    check_launch();
    prims::scan_array(ctx, L->sbase, L->sbase, (uint64_t)L->n_sslices + 1, st);
    // multi region segments
    L->pbase = dalloc<uint32_t>(ctx, (uint64_t)M + 1);
    k_multi_nch<<<grid(ctx, (uint64_t)M + 1), 256, 0, st>>>(L->indeg, M, L->pbase);
    check_launch();
    prims::scan_array(ctx, L->pbase, L->pbase, (uint64_t)M + 1, st);
    {
      uint32_t h = 0;  // pbase is uint32: read exactly 4 bytes
      DYNPR_CK(cudaMemcpyAsync(ctx->pinned, L->pbase + M, 4, cudaMemcpyDeviceToHost, st));
      sync(ctx);
      std::memcpy(&h, ctx->pinned, 4);
      L->n_mseg = h;
    }
    L->mseg_v = dalloc<uint32_t>(ctx, L->n_mseg);
    L->mseg_len = dalloc<uint32_t>(ctx, L->n_mseg);
    L->n_mslices = (L->n_mseg + 31) / 32;
    L->mbase = dalloc<uint64_t>(ctx, L->n_mslices + 1);
    if (M) {
      k_multi_segments<<<grid(ctx, M), 256, 0, st>>>(L->indeg, M, L->pbase, L->mseg_v, L->mseg_len);
      check_launch();
    }
    k_multi_slice_len<<<grid(ctx, (L->n_mslices + 1) * 32), 256, 0, st>>>(L->mseg_len, L->n_mseg, L->n_mslices,
                                                                          L->mbase);
    check_launch();
    prims::scan_array(ctx, L->mbase, L->mbase, (uint64_t)L->n_mslices + 1, st);
    // the slices this context sweeps: all of them, or on a team context
    // the rank's edge-balanced range (its in-CSR rows only)
    uint64_t ss_lo = 0, ss_hi = L->n_sslices, ms_lo = 0, ms_hi = L->n_mslices;
    if (is_team(ctx)) {
      L->owned = true;
      L->own = plan_ranges(ctx, L, ctx->comm->world)[ctx->comm->rank];
      ss_lo = L->own.ss_lo;
      ss_hi = L->own.ss_hi;
      ms_lo = L->own.ms_lo;
      ms_hi = L->own.ms_hi;
    }
    const uint64_t s_w0 = read_u64(ctx, L->sbase + ss_lo), s_w1 = read_u64(ctx, L->sbase + ss_hi);
    const uint64_t m_w0 = read_u64(ctx, L->mbase + ms_lo), m_w1 = read_u64(ctx, L->mbase + ms_hi);
    uint32_t* sa = new_block(ctx, L, s_w1 - s_w0);
    uint32_t* ma = new_block(ctx, L, m_w1 - m_w0);
    L->sell_s = sa - s_w0;  // indexed by sbase[s], s in the owned range
    L->sell_m = ma - m_w0;
    L->sell_words = (s_w1 - s_w0) + (m_w1 - m_w0);
    if (ss_hi > ss_lo) {
      k_fill_single<<<grid(ctx, (ss_hi - ss_lo) * 32), 256, 0, st>>>(gT->off, gT->tgt, L->perm, L->inv, L->indeg, M,
                                                                     n, ss_lo, ss_hi, L->sbase, L->sell_s);
      check_launch();
    }
    if (ms_hi > ms_lo) {
      k_fill_multi<<<grid(ctx, (ms_hi - ms_lo) * 32), 256, 0, st>>>(gT->off, gT->tgt, L->perm, L->inv, L->pbase,
                                                                    L->mseg_v, L->mseg_len, L->n_mseg, ms_lo, ms_hi,
                                                                    L->mbase, L->sell_m);
      check_launch();
    }
    count_launch(ctx, 6);
  } catch (...) {
    destroy_layout(L);
    throw;
  }
  return L;
}


// The layout of a snapshot pair derived from its parent pair's (same vertex
// relabelling, so every column id already stored stays valid): in-lists the
// batch did not touch are copied segment by segment from the parent's SELL
// slices, touched ones re-gathered from the new transpose; the forward CSR
// likewise by rows.  Degrees, slice lengths and the multi-region chunk
// metadata are recomputed (O(n)).  The relabelling is no longer exactly
// sorted, which only affects scheduling: a slice's length is the maximum of
// its segments, and a vertex whose in-degree grew past the flat limit while
// in a single slice is summed by its lane in 256-element chunks (sweep.cu
// folds), bit-identical to the reference's chunked path.  nullptr = build
// from scratch instead (T above 256, team layouts, many derivations).
Layout* build_incremental(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF, uint32_t T,
                          const LayoutSeed& seed) {
  const Layout* P = seed.parent.get();
  constexpr int kMaxGenerations = 32;  // then rebuild (sorted order, tight slices)
  if (!P || P->ctx != ctx || P->owned || is_team(ctx) || P->T != T || T > 256u || P->n != gT->n ||
      P->generation >= kMaxGenerations || !gT->n)
    return nullptr;
  cudaStream_t st = ctx->stream;
  const uint32_t n = gT->n, M = P->M;
  auto* L = new Layout();
  L->ctx = ctx;
  try {
    L->n = n;
    L->m = gT->m;
    L->T = T;
    L->gF_id = gF->id;
    L->loops = gT->all_loops;
    L->M = M;
    L->generation = P->generation + 1;
    L->n_hslices = P->n_hslices;  // scheduling hint only
    L->blocks = P->blocks;  // shared relabelling, slices and forward rows (copy-on-write)
    L->perm = P->perm;
    L->inv = P->inv;
    L->indeg = dalloc<uint32_t>(ctx, n);
    L->outdeg = dalloc<uint32_t>(ctx, n);
    DYNPR_CK(cudaMemcpyAsync(L->indeg, P->indeg, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    DYNPR_CK(cudaMemcpyAsync(L->outdeg, P->outdeg, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    // touched rows in the relabelled space, in-lists (T) and out-lists (F),
    // and their new degrees
    auto* flagT = reinterpret_cast<uint8_t*>(ctx->layout_tmp.as<uint32_t>(((uint64_t)n + 4) / 2 + 2));
    uint8_t* flagF = flagT + n + 4;
    DYNPR_CK(cudaMemsetAsync(flagT, 0, 2 * ((size_t)n + 4), st));
    if (seed.n_T)
      k_mark_rows<<<grid(ctx, seed.n_T), 256, 0, st>>>(seed.rows_T, seed.n_T, L->inv, gT->off, flagT, L->indeg);
    if (seed.n_F)
      k_mark_rows<<<grid(ctx, seed.n_F), 256, 0, st>>>(seed.rows_F, seed.n_F, L->inv, gF->off, flagF, L->outdeg);
    check_launch();
    count_launch(ctx, 2);
    L->mcount = dalloc<uint32_t>(ctx, (uint64_t)M + 1);
    DYNPR_CK(cudaMemsetAsync(L->mcount, 0, ((size_t)M + 1) * 4, st));
    L->sell_s = P->sell_s;
    L->sell_m = P->sell_m;
    // single region: re-built slices into a new block
    const uint64_t S = P->n_sslices;
    L->n_sslices = S;
    L->sbase = dalloc<uint64_t>(ctx, S + 1);
    auto* len32 = reinterpret_cast<uint64_t*>(ctx->scratch64b.as<unsigned long long>(2 * (S + 1)));
    uint64_t* dpos = len32 + S + 1;
    // (the touched rows drive the slice passes: O(batch), not O(slices))
    DYNPR_CK(cudaMemsetAsync(len32, 0, (S + 1) * 8, st));
    if (seed.n_T)
      k_slice_touched_len_rows<<<grid(ctx, seed.n_T * 32), 256, 0, st>>>(seed.rows_T, seed.n_T, L->inv, L->indeg,
                                                                          M, n, len32);
    check_launch();
    prims::scan_array<uint64_t>(ctx, len32, dpos, S + 1, st);
    const uint64_t s_new = read_u64(ctx, dpos + S);
    uint32_t* ds = new_block(ctx, L, s_new);
    k_sbase_cow<<<grid(ctx, S + 1), 256, 0, st>>>(P->sbase, len32, dpos, S, rel_words(L->sell_s, ds), L->sbase);
    check_launch();
    if (s_new) {
      k_fill_single_cow_rows<<<grid(ctx, seed.n_T * 32), 256, 0, st>>>(seed.rows_T, seed.n_T, gT->off, gT->tgt,
                                                                        L->perm, L->inv, L->indeg, M, n, len32,
                                                                        L->sbase, L->sell_s, flagT, P->sbase);
      check_launch();
    }
    count_launch(ctx, 3);
    // multi region: touched vertices' chunks retired and appended
    uint32_t* apos = ctx->scratch32a.as<uint32_t>((uint64_t)M + 2);
    k_multi_touched_nch<<<grid(ctx, (uint64_t)M + 1), 256, 0, st>>>(L->indeg, flagT, M, apos);
    check_launch();
    prims::scan_array(ctx, apos, apos, (uint64_t)M + 1, st);
    uint64_t appended = 0, retired = 0;
    {
      uint32_t h = 0;
      DYNPR_CK(cudaMemcpyAsync(ctx->pinned, apos + M, 4, cudaMemcpyDeviceToHost, st));
      sync(ctx);
      std::memcpy(&h, ctx->pinned, 4);
      appended = h;
    }
    const uint64_t first = P->n_mslices * 32;  // appended segments start a slice
    L->n_mseg = first + appended;
    L->n_mslices = (L->n_mseg + 31) / 32;
    L->pbase = dalloc<uint32_t>(ctx, (uint64_t)M + 1);
    L->mseg_v = dalloc<uint32_t>(ctx, L->n_mseg);
    L->mseg_len = dalloc<uint32_t>(ctx, L->n_mseg);
    L->mbase = dalloc<uint64_t>(ctx, L->n_mslices + 1);
    DYNPR_CK(cudaMemcpyAsync(L->pbase, P->pbase, ((size_t)M + 1) * 4, cudaMemcpyDeviceToDevice, st));
    DYNPR_CK(cudaMemsetAsync(L->mseg_v, 0, L->n_mseg * 4, st));
    DYNPR_CK(cudaMemsetAsync(L->mseg_len, 0, L->n_mseg * 4, st));
    if (P->n_mseg) {
      DYNPR_CK(cudaMemcpyAsync(L->mseg_v, P->mseg_v, P->n_mseg * 4, cudaMemcpyDeviceToDevice, st));
      DYNPR_CK(cudaMemcpyAsync(L->mseg_len, P->mseg_len, P->n_mseg * 4, cudaMemcpyDeviceToDevice, st));
    }
    DYNPR_CK(cudaMemcpyAsync(L->mbase, P->mbase, (P->n_mslices + 1) * 8, cudaMemcpyDeviceToDevice, st));
    if (M && seed.n_T) {
      k_multi_cow_segments_rows<<<grid(ctx, seed.n_T * 32), 256, 0, st>>>(seed.rows_T, seed.n_T, L->inv, L->indeg,
                                                                           P->indeg, M, apos, first, P->pbase,
                                                                           L->pbase, L->mseg_v, L->mseg_len);
      check_launch();
    }
    DYNPR_CK(cudaMemcpyAsync(L->pbase + M, &L->n_mseg, 4, cudaMemcpyHostToDevice, st));  // (pageable: synchronous)
    const uint64_t s_lo = P->n_mslices, s_hi = L->n_mslices;
    if (s_hi > s_lo) {
      // the appended slices' lengths -> bases within a new block
      k_multi_slice_len<<<grid(ctx, (s_hi - s_lo + 1) * 32), 256, 0, st>>>(L->mseg_len + first, appended,
                                                                           s_hi - s_lo, L->mbase + s_lo);
      check_launch();
      prims::scan_array(ctx, L->mbase + s_lo, L->mbase + s_lo, (uint64_t)(s_hi - s_lo) + 1, st);
      const uint64_t m_new = read_u64(ctx, L->mbase + s_hi);
      uint32_t* dm = new_block(ctx, L, m_new);
      k_mbase_append<<<grid(ctx, s_hi - s_lo + 1), 256, 0, st>>>(L->mbase, s_lo, s_hi - s_lo, rel_words(L->sell_m, dm));
      check_launch();
      k_fill_multi<<<grid(ctx, (s_hi - s_lo) * 32), 256, 0, st>>>(gT->off, gT->tgt, L->perm, L->inv, L->pbase,
                                                                  L->mseg_v, L->mseg_len, L->n_mseg, s_lo, s_hi,
                                                                  L->mbase, L->sell_m);
      check_launch();
      count_launch(ctx, 4);
      L->sell_words = P->sell_words + s_new + m_new;
    } else {
      L->sell_words = P->sell_words + s_new;
    }
    {  // retired segments (old chunks of touched vertices + the slice padding)
      auto* cnt = reinterpret_cast<unsigned*>(ctx->scratch64a.as<unsigned long long>(2));
      DYNPR_CK(cudaMemsetAsync(cnt, 0, 8, st));
      k_count_above<<<grid(ctx, L->n_mseg), 256, 0, st>>>(L->mseg_len, (uint32_t)L->n_mseg, 0u, cnt);
      check_launch();
      count_launch(ctx, 2);
      retired = L->n_mseg - (read_u64(ctx, cnt) & 0xffffffffu);
      L->dead_segs = retired;
    }
    if (L->dead_segs > L->n_mseg / 4 + 64) {  // too fragmented: rebuild from scratch
      destroy_layout(L);
      return nullptr;
    }
    if (P->has_forward) {
      // copy-on-write forward rows: untouched rows keep their words in the
      // parent's blocks, the touched ones (batch sources) are rewritten into
      // one new block; begF is the parent's with those rows re-pointed
      L->tgtF = P->tgtF;
      L->begF = dalloc<uint64_t>(ctx, (uint64_t)n + 1);
      DYNPR_CK(cudaMemcpyAsync(L->begF, P->begF, ((size_t)n + 1) * 8, cudaMemcpyDeviceToDevice, st));
      const uint64_t c = seed.n_F;
      uint64_t words = 0;
      if (c) {
        auto* wpos = ctx->scratch64b.as<unsigned long long>(c + 1);
        uint32_t* items = ctx->scratch32a.as<uint32_t>(c + 2);
        prims::scan_exclusive<unsigned long long>(ctx, RowWords{seed.rows_F, L->inv, L->outdeg, c}, wpos, c + 1, st);
        words = read_u64(ctx, wpos + c);
        uint32_t* blk = new_block(ctx, L, words);
        prims::scan_exclusive<uint32_t>(ctx, RowChunks{seed.rows_F, L->inv, L->outdeg, c}, items, c + 1, st);
        k_refill_rows<<<(unsigned)ctx->num_sms * 16, 256, 0, st>>>(seed.rows_F, c, items, wpos, gF->off, gF->tgt,
                                                                   L->inv, rel_words(L->tgtF, blk), L->tgtF,
                                                                   L->begF, blk);
        check_launch();
        count_launch(ctx);
      }
      L->fwd_words = P->fwd_words + words;
      L->has_forward = true;
    }
  } catch (...) {
    destroy_layout(L);
    throw;
  }
  return L;
}
}  // namespace

Layout::~Layout() {
  // (perm, inv, the SELL storage and the forward rows are shared blocks)
  for (void* p : {(void*)indeg, (void*)outdeg, (void*)sbase, (void*)mbase, (void*)mseg_v, (void*)mseg_len,
                  (void*)pbase, (void*)mcount, (void*)begF})
    pool_free(ctx, p);
}

void destroy_layout(Layout* L) { delete L; }

std::shared_ptr<Layout> share_layout(Layout* L) { return std::shared_ptr<Layout>(L, destroy_layout); }

LayoutSeed::~LayoutSeed() {
  pool_free(ctx, rows_T);
  pool_free(ctx, rows_F);
}

Layout* get_layout(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF, uint32_t T, bool need_forward) {
  // The layout is cached on gT and freed with it through its context's pool:
  // build it only with the context that owns both graphs (a layout built by
  // another context could outlive that context, or sit on another device).
  if (gT->ctx != ctx || gF->ctx != ctx) invalid("engine: the graphs belong to another context");
  auto* g = const_cast<dynpr_graph*>(gT);
  Layout* L = g->layout.get();
  if (!L || L->gF_id != gF->id || L->T != T) {
    g->layout.reset();
    DYNPR_CK(cudaEventRecord(ctx->ev_s0, ctx->stream));
    L = nullptr;
    if (g->seed && g->seed->gF_id == gF->id) L = build_incremental(ctx, gT, gF, T, *g->seed);
    if (!L) L = build_layout(ctx, gT, gF, T);
    g->seed.reset();  // releases the parent layout
    g->layout = share_layout(L);
    DYNPR_CK(cudaEventRecord(ctx->ev_s1, ctx->stream));
    sync(ctx);
    float ms = 0.f;
    DYNPR_CK(cudaEventElapsedTime(&ms, ctx->ev_s0, ctx->ev_s1));
    L->build_ms = ms;
  }
  if (need_forward && !L->has_forward) {
    DYNPR_CK(cudaEventRecord(ctx->ev_s0, ctx->stream));
    build_forward(ctx, L, gF);
    DYNPR_CK(cudaEventRecord(ctx->ev_s1, ctx->stream));
    sync(ctx);
    float ms = 0.f;
    DYNPR_CK(cudaEventElapsedTime(&ms, ctx->ev_s0, ctx->ev_s1));
    L->build_ms += ms;
  }
  return L;
}

void launch_gather_perm_f64(dynpr_context* ctx, const Layout* L, const double* src, double* dst) {
  k_gather_perm_f64<<<grid(ctx, L->n), 256, 0, ctx->stream>>>(L->perm, L->n, src, dst);
  check_launch();
  count_launch(ctx);
}
void launch_gather_perm_u8(dynpr_context* ctx, const Layout* L, const uint8_t* src, uint8_t* dst) {
  k_gather_perm_u8<<<grid(ctx, L->n), 256, 0, ctx->stream>>>(L->perm, L->n, src, dst);
  check_launch();
  count_launch(ctx);
}
void launch_scatter_inv_f64(dynpr_context* ctx, const Layout* L, const double* src, double* dst) {
  k_scatter_inv_f64<<<grid(ctx, L->n), 256, 0, ctx->stream>>>(L->inv, L->n, src, dst);
  check_launch();
  count_launch(ctx);
}
void launch_scatter_inv_u8(dynpr_context* ctx, const Layout* L, const uint8_t* src, uint8_t* dst) {
  k_scatter_inv_u8<<<grid(ctx, L->n), 256, 0, ctx->stream>>>(L->inv, L->n, src, dst);
  check_launch();
  count_launch(ctx);
}

}  // namespace dynpr_b200
