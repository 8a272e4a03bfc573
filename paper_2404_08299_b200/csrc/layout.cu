// Builder of the engine layout (see layout.cuh): degree sort, relabelling,
// SELL-32 segment slices, relabelled forward CSR.
#include <cub/cub.cuh>

#include "comm.cuh"
#include "layout.cuh"
#include "sweep.cuh"

namespace dynpr_b200 {

namespace {

template <class F>
void cub_call(dynpr_context* ctx, F&& f) {
  size_t bytes = 0;
  DYNPR_CK(f(nullptr, bytes));
  void* tmp = ctx->cub_tmp.ensure(bytes);
  DYNPR_CK(f(tmp, bytes));
}

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
__device__ __forceinline__ void fill_lane(uint32_t* sell, uint64_t base, unsigned lane, uint32_t L, uint32_t len,
                                          const uint32_t* src, const uint32_t* inv) {
  for (uint32_t k = 0; k < L; k += 4) {
    uint4 w;
    w.x = k < len ? inv[src[k]] : 0u;
    w.y = k + 1 < len ? inv[src[k + 1]] : 0u;
    w.z = k + 2 < len ? inv[src[k + 2]] : 0u;
    w.w = k + 3 < len ? inv[src[k + 3]] : 0u;
    *reinterpret_cast<uint4*>(sell + sell_pos(base, lane, k)) = w;
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

unsigned grid(dynpr_context* ctx, uint64_t items) { return grid_for(items, 256, ctx->num_sms * 32); }

uint64_t read_u64(dynpr_context* ctx, const void* d) {
  uint64_t h = 0;
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  std::memcpy(&h, ctx->pinned, 8);
  return h;
}

void build_forward(dynpr_context* ctx, Layout* L, const dynpr_graph* gF) {
  cudaStream_t st = ctx->stream;
  L->offF = dalloc<uint64_t>(ctx, (uint64_t)L->n + 1);
  L->tgtF = dalloc<uint32_t>(ctx, L->m);
  k_outdeg64<<<grid(ctx, (uint64_t)L->n + 1), 256, 0, st>>>(L->outdeg, L->n, L->offF);
  check_launch();
  cub_call(ctx, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, L->offF, L->offF, (int64_t)L->n + 1, st);
  });
  k_fill_forward<<<grid(ctx, (L->m + kFillChunk - 1) / kFillChunk * 32), 256, 0, st>>>(
      gF->off, gF->tgt, L->perm, L->inv, L->n, L->offF, L->tgtF);
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
    L->perm = dalloc<uint32_t>(ctx, n);
    L->inv = dalloc<uint32_t>(ctx, n);
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
    cub_call(ctx, [&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, indeg_old, mx, (int64_t)n, st); });
    const uint32_t maxdeg = (uint32_t)(read_u64(ctx, mx) & 0xffffffffu);
    k_desc_keys<<<grid(ctx, n), 256, 0, st>>>(indeg_old, n, maxdeg, keys);
    check_launch();
    count_launch(ctx, 2);
    const int eb = bits_for(maxdeg);
    if (eb > 0) {
      cub::DoubleBuffer<uint32_t> kb(keys, keys2);
      cub::DoubleBuffer<uint32_t> vb(iota, L->perm);
      cub_call(ctx, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, kb, vb, (int64_t)n, 0, eb, st);
      });
      if (vb.Current() != L->perm)
        DYNPR_CK(cudaMemcpyAsync(L->perm, vb.Current(), (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
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
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, L->sbase, L->sbase, (int64_t)L->n_sslices + 1, st);
    });
    // multi region segments
    L->pbase = dalloc<uint32_t>(ctx, (uint64_t)M + 1);
    k_multi_nch<<<grid(ctx, (uint64_t)M + 1), 256, 0, st>>>(L->indeg, M, L->pbase);
    check_launch();
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, L->pbase, L->pbase, (int64_t)M + 1, st);
    });
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
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, L->mbase, L->mbase, (int64_t)L->n_mslices + 1, st);
    });
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
    L->sell_s_alloc = dalloc<uint32_t>(ctx, s_w1 - s_w0);
    L->sell_m_alloc = dalloc<uint32_t>(ctx, m_w1 - m_w0);
    L->sell_s = L->sell_s_alloc - s_w0;  // indexed by sbase[s], s in the owned range
    L->sell_m = L->sell_m_alloc - m_w0;
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

}  // namespace

Layout::~Layout() {
  for (void* p : {(void*)perm, (void*)inv, (void*)indeg, (void*)outdeg, (void*)sbase, (void*)sell_s_alloc,
                  (void*)mbase, (void*)mseg_v, (void*)mseg_len, (void*)pbase, (void*)sell_m_alloc, (void*)mcount,
                  (void*)offF, (void*)tgtF})
    pool_free(ctx, p);
}

void destroy_layout(Layout* L) { delete L; }

Layout* get_layout(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF, uint32_t T, bool need_forward) {
  // The layout is cached on gT and freed with it through its context's pool:
  // build it only with the context that owns both graphs (a layout built by
  // another context could outlive that context, or sit on another device).
  if (gT->ctx != ctx || gF->ctx != ctx) invalid("engine: the graphs belong to another context");
  Layout* L = gT->layout;
  if (!L || L->gF_id != gF->id || L->T != T) {
    if (L) {
      destroy_layout(L);
      const_cast<dynpr_graph*>(gT)->layout = nullptr;
    }
    DYNPR_CK(cudaEventRecord(ctx->ev_s0, ctx->stream));
    L = build_layout(ctx, gT, gF, T);
    const_cast<dynpr_graph*>(gT)->layout = L;
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
