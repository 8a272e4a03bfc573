// Rank-update sweep, degree schedule, frontier and norm kernels
// (north_star subsystems 2, 3 and 4).
//
// Arithmetic contract (SURVEY 8a, rank.cpp:42-115): every fp64 operation
// below is an explicitly rounded intrinsic (__dadd_rn / __dmul_rn / ...), this
// file is compiled with --fmad=false, and each vertex accumulates its
// in-neighbour contributions in exactly the reference's order:
//   in-degree <= lowDegreeThreshold : one flat running sum over the ascending
//                                     in-slice (rank.cpp:45-54)
//   otherwise                       : sequential partial sums over 256-edge
//                                     chunks, added in chunk order
//                                     (rank.cpp:59-75)
// so the ranks, the L-inf delta and hence every threshold decision are
// bit-identical to the reference CPU library.
//
// Parallel decomposition (B200-first, the paper's kernel pair refined):
//   k_sweep_low    thread per vertex, in-degree <= T (~93% of RMAT vertices)
//   k_sweep_chunks warp per 32 chunks of <= 256 edges; the warp stages 16
//                  contributions per chunk per round through shared memory
//                  with coalesced half-warp loads (two chunks per load
//                  instruction), then every lane sums its own chunk
//                  sequentially -> the reference order at full warp
//                  efficiency ("transposed" warp-cooperative gather)
//   k_sweep_multi  thread per vertex with more than one chunk: adds the
//                  chunk partials in order and finalises
// All three share one fused epilogue: closed-loop / plain rank formula,
// the next sweep's contribution r/outdeg (IEEE division, so gathering it is
// bit-identical to the reference's per-edge division), copy-through of
// unaffected vertices, prune / frontier flags with warp-aggregated
// append to the pending lists, and a block-level max / count reduction
// finished with one 64-bit atomic per block (L-inf fused into the update).
#include "sweep.cuh"

namespace dynpr_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRound = 16;  // contributions staged per chunk per round

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

// ---- block reductions ----------------------------------------------------
struct BlockRed {
  double dmax;
  unsigned long long proc, edges;
};

__device__ __forceinline__ void block_reduce_commit(double dmax,
                                                    unsigned long long proc,
                                                    unsigned long long edges,
                                                    SweepRed* red) {
  __shared__ double s_d[kWarps];
  __shared__ unsigned long long s_p[kWarps], s_e[kWarps];
  dmax = warp_max(dmax);
  proc = warp_sum(proc);
  edges = warp_sum(edges);
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) {
    s_d[w] = dmax;
    s_p[w] = proc;
    s_e[w] = edges;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    unsigned long long p = 0, e = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      d = fmax(d, s_d[i]);
      p += s_p[i];
      e += s_e[i];
    }
    if (d > 0.0) atomicMax(&red->delta_bits, (unsigned long long)__double_as_longlong(d));
    if (p) atomicAdd(&red->processed, p);
    if (e) atomicAdd(&red->edges, e);
  }
}

// Warp-aggregated append of pending vertices to the low/high out-degree
// lists (all 32 lanes must call it).
__device__ __forceinline__ void warp_append(bool pend, bool lowout, uint32_t v,
                                            uint32_t* pl, uint32_t* ph,
                                            SweepRed* red) {
  const unsigned ml = __ballot_sync(0xffffffffu, pend && lowout);
  const unsigned mh = __ballot_sync(0xffffffffu, pend && !lowout);
  if (!(ml | mh)) return;
  const unsigned lane = lane_id();
  unsigned bl = 0, bh = 0;
  if (lane == 0) {
    if (ml) bl = atomicAdd(&red->pend_low, (unsigned)__popc(ml));
    if (mh) bh = atomicAdd(&red->pend_high, (unsigned)__popc(mh));
  }
  bl = __shfl_sync(0xffffffffu, bl, 0);
  bh = __shfl_sync(0xffffffffu, bh, 0);
  const unsigned lt = (1u << lane) - 1u;
  if (pend && lowout) pl[bl + __popc(ml & lt)] = v;
  if (pend && !lowout) ph[bh + __popc(mh & lt)] = v;
}

// Unaffected vertex (rank.cpp:90-92): current = previous.  In engine mode
// only vertices written by the previous sweep differ between the buffers.
__device__ __forceinline__ void copy_through(const SweepArgs& a, uint32_t v) {
  if (a.copy_all) {
    a.rank_cur[v] = a.rank_prev[v];
    if (a.contrib_cur) a.contrib_cur[v] = a.contrib_prev[v];
  } else if (a.written[v]) {
    a.rank_cur[v] = a.rank_prev[v];
    a.contrib_cur[v] = a.contrib_prev[v];
    a.written[v] = 0;
  }
  if (a.np && !a.np_accumulate) a.np[v] = 0;
}

// Fused epilogue: rank formula (rank.cpp:97-106), next contribution, delta,
// flags (rank.cpp:108-115).
template <bool FLAGGED, bool CLOSED>
__device__ __forceinline__ void finalize(const SweepArgs& a, uint32_t v,
                                         double c, double& dmax, bool& pend,
                                         bool& lowout) {
  const double pv = a.rank_prev[v];
  const uint32_t od = (uint32_t)(a.offF[v + 1] - a.offF[v]);
  const double d = (double)od;
  double r;
  if (CLOSED) {
    r = __ddiv_rn(__dadd_rn(a.teleport, __dmul_rn(a.alpha, __dsub_rn(c, __ddiv_rn(pv, d)))),
                  __dsub_rn(1.0, __ddiv_rn(a.alpha, d)));
  } else {
    r = __dadd_rn(a.teleport, __dmul_rn(a.alpha, c));
  }
  a.rank_cur[v] = r;
  if (a.contrib_cur) a.contrib_cur[v] = __ddiv_rn(r, d);
  const double dr = fabs(__dsub_rn(r, pv));
  if (dr > dmax) dmax = dr;  // NaN never wins, like blockMax (parallel.hpp:66-73)
  if (FLAGGED) {
    const double denom = r > pv ? r : pv;
    const double rel = denom > 0.0 ? __ddiv_rn(dr, denom) : 0.0;
    if (CLOSED && rel <= a.tp) a.va[v] = 0;
    pend = rel > a.tf;
    if (a.np) {
      if (a.np_accumulate) {
        if (pend) a.np[v] = 1;
      } else {
        a.np[v] = pend;
      }
    }
    lowout = od <= a.T;
    if (a.written) a.written[v] = 1;
  }
}

// ---- low in-degree: thread per vertex ----------------------------------------
template <bool FLAGGED, bool CLOSED>
__global__ void __launch_bounds__(kThreads) k_sweep_low(SweepArgs a) {
  double dmax = 0.0;
  unsigned long long proc = 0, edges = 0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads; base < a.n; base += stride) {
    const uint64_t vv = base + threadIdx.x;
    bool pend = false, lowout = false;
    if (vv < a.n) {
      const uint32_t v = (uint32_t)vv;
      const uint64_t b = a.offT[v], e = a.offT[v + 1];
      const uint32_t deg = (uint32_t)(e - b);
      if (deg <= a.T) {
        if (FLAGGED && !a.va[v]) {
          copy_through(a, v);
        } else {
          double c = 0.0;
          uint64_t i = b;
          for (; i + 4 <= e; i += 4) {
            const uint32_t u0 = a.idxT[i], u1 = a.idxT[i + 1], u2 = a.idxT[i + 2],
                           u3 = a.idxT[i + 3];
            const double x0 = a.contrib_prev[u0], x1 = a.contrib_prev[u1],
                         x2 = a.contrib_prev[u2], x3 = a.contrib_prev[u3];
            c = __dadd_rn(c, x0);
            c = __dadd_rn(c, x1);
            c = __dadd_rn(c, x2);
            c = __dadd_rn(c, x3);
          }
          for (; i < e; ++i) c = __dadd_rn(c, a.contrib_prev[a.idxT[i]]);
          finalize<FLAGGED, CLOSED>(a, v, c, dmax, pend, lowout);
          ++proc;
          edges += deg;
        }
      }
    }
    if (FLAGGED && a.pend_low)
      warp_append(pend, lowout, (uint32_t)vv, a.pend_low, a.pend_high, a.red);
  }
  block_reduce_commit(dmax, proc, edges, a.red);
}

// ---- high in-degree: warp-cooperative chunks -----------------------------------
template <bool FLAGGED, bool CLOSED>
__global__ void __launch_bounds__(kThreads) k_sweep_chunks(SweepArgs a) {
  __shared__ double s_x[kWarps][32][kRound + 1];
  __shared__ uint64_t s_b[kWarps][32];
  __shared__ uint32_t s_len[kWarps][32];
  const int w = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  const unsigned half = lane >> 4, hl = lane & 15;
  double dmax = 0.0;
  unsigned long long proc = 0, edges = 0;
  const uint64_t wstride = (uint64_t)gridDim.x * kWarps * 32;
  for (uint64_t cbase = ((uint64_t)blockIdx.x * kWarps + w) * 32; cbase < a.n_chunks;
       cbase += wstride) {
    const uint64_t c = cbase + lane;
    const bool valid = c < a.n_chunks;
    uint32_t v = 0, j = 0;
    uint64_t vb = 0, ve = 0;
    if (valid) {
      const uint2 ent = a.chunks[c];
      v = ent.x;
      j = ent.y;
      vb = a.offT[v];
      ve = a.offT[v + 1];
    }
    const uint64_t b = vb + (uint64_t)kAccumChunk * j;
    const uint64_t e = (b + kAccumChunk < ve) ? b + kAccumChunk : ve;
    const bool aff = valid && (!FLAGGED || a.va[v]);
    const uint32_t len = aff ? (uint32_t)(e - b) : 0u;
    s_b[w][lane] = b;
    s_len[w][lane] = len;
    const unsigned maxlen = __reduce_max_sync(0xffffffffu, len);
    __syncwarp();
    double p = 0.0;
    for (unsigned r0 = 0; r0 < maxlen; r0 += kRound) {
      const unsigned k = r0 + hl;
      // gather phase: step q stages element k of chunks 2q (lanes 0-15) and
      // 2q+1 (lanes 16-31); indices first, then contributions, for MLP.
      uint32_t u[kRound];
#pragma unroll
      for (int q = 0; q < kRound; ++q) {
        const int i = 2 * q + half;
        u[q] = k < s_len[w][i] ? a.idxT[s_b[w][i] + k] : 0xffffffffu;
      }
      double x[kRound];
#pragma unroll
      for (int q = 0; q < kRound; ++q) x[q] = u[q] != 0xffffffffu ? a.contrib_prev[u[q]] : 0.0;
#pragma unroll
      for (int q = 0; q < kRound; ++q) s_x[w][2 * q + half][hl] = x[q];
      __syncwarp();
      // sum phase: each lane walks its own chunk in order
      if (len > r0) {
        const unsigned cnt = (len - r0) < (unsigned)kRound ? (len - r0) : (unsigned)kRound;
        for (unsigned t = 0; t < cnt; ++t) p = __dadd_rn(p, s_x[w][lane][t]);
      }
      __syncwarp();
    }
    bool pend = false, lowout = false;
    if (valid) {
      const uint64_t deg = ve - vb;
      if (deg <= kAccumChunk) {  // single chunk: c = 0.0 + p = p (rank.cpp:72)
        if (!aff) {
          copy_through(a, v);
        } else {
          finalize<FLAGGED, CLOSED>(a, v, p, dmax, pend, lowout);
          ++proc;
          edges += deg;
        }
      } else if (aff) {
        a.partials[c] = p;
      }
    }
    if (FLAGGED && a.pend_low) warp_append(pend, lowout, v, a.pend_low, a.pend_high, a.red);
  }
  block_reduce_commit(dmax, proc, edges, a.red);
}

// ---- multi-chunk vertices: ordered combine of the partials (rank.cpp:72) ------
template <bool FLAGGED, bool CLOSED>
__global__ void __launch_bounds__(kThreads) k_sweep_multi(SweepArgs a) {
  double dmax = 0.0;
  unsigned long long proc = 0, edges = 0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads; base < a.n_multi; base += stride) {
    const uint64_t i = base + threadIdx.x;
    bool pend = false, lowout = false;
    uint32_t v = 0;
    if (i < a.n_multi) {
      const uint2 ent = a.multi[i];
      v = ent.x;
      const uint64_t deg = a.offT[v + 1] - a.offT[v];
      if (FLAGGED && !a.va[v]) {
        copy_through(a, v);
      } else {
        const uint64_t nch = (deg + kAccumChunk - 1) / kAccumChunk;
        double c = 0.0;
        for (uint64_t q = 0; q < nch; ++q) c = __dadd_rn(c, a.partials[(uint64_t)ent.y + q]);
        finalize<FLAGGED, CLOSED>(a, v, c, dmax, pend, lowout);
        ++proc;
        edges += deg;
      }
    }
    if (FLAGGED && a.pend_low) warp_append(pend, lowout, v, a.pend_low, a.pend_high, a.red);
  }
  block_reduce_commit(dmax, proc, edges, a.red);
}

// ---- schedule (partition.cpp:7-61 + chunk table) ----------------------------------
constexpr int kTileItems = 4;
constexpr int kTile = kThreads * kTileItems;  // 1024 vertices per tile

struct Cnt3 {
  unsigned low, chunks, multi;
};
__device__ __forceinline__ Cnt3 add3(Cnt3 x, Cnt3 y) {
  return {x.low + y.low, x.chunks + y.chunks, x.multi + y.multi};
}

__device__ __forceinline__ Cnt3 vertex_counts(const uint64_t* off, uint64_t v, uint32_t n,
                                              uint32_t thr, bool want_chunks) {
  if (v >= n) return {0, 0, 0};
  const uint64_t deg = off[v + 1] - off[v];
  if (deg <= thr) return {1, 0, 0};
  if (!want_chunks) return {0, 0, 0};
  const unsigned nch = (unsigned)((deg + kAccumChunk - 1) / kAccumChunk);
  return {0, nch, nch > 1 ? 1u : 0u};
}

// Exclusive block scan of per-thread Cnt3 (thread order == id order).
__device__ __forceinline__ Cnt3 block_exclusive_scan(Cnt3 x, Cnt3& total) {
  __shared__ Cnt3 s_w[kWarps];
  const unsigned lane = lane_id();
  const int w = threadIdx.x >> 5;
  Cnt3 inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Cnt3 y;
    y.low = __shfl_up_sync(0xffffffffu, inc.low, o);
    y.chunks = __shfl_up_sync(0xffffffffu, inc.chunks, o);
    y.multi = __shfl_up_sync(0xffffffffu, inc.multi, o);
    if ((int)lane >= o) inc = add3(inc, y);
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  Cnt3 pre = {0, 0, 0};
  total = {0, 0, 0};
  for (int i = 0; i < kWarps; ++i) {
    if (i < w) pre = add3(pre, s_w[i]);
    total = add3(total, s_w[i]);
  }
  __syncthreads();
  Cnt3 r = add3(pre, inc);
  return {r.low - x.low, r.chunks - x.chunks, r.multi - x.multi};
}

__global__ void __launch_bounds__(kThreads) k_sched_count(const uint64_t* off, uint32_t n, uint32_t thr,
                                                         bool want_chunks, uint4* tiles) {
  const uint64_t v0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kTileItems;
  Cnt3 s = {0, 0, 0};
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) s = add3(s, vertex_counts(off, v0 + k, n, thr, want_chunks));
  Cnt3 total;
  block_exclusive_scan(s, total);
  if (threadIdx.x == 0) tiles[blockIdx.x] = make_uint4(total.low, total.chunks, total.multi, 0);
}

// Single-block exclusive scan of the tile counts (64-bit chunk totals).
__global__ void k_sched_scan(uint4* tiles, uint64_t ntiles, unsigned long long* totals,
                             unsigned long long* chunk_base) {
  __shared__ unsigned long long s_l[1024], s_c[1024], s_m[1024];
  unsigned long long carry_l = 0, carry_c = 0, carry_m = 0;
  for (uint64_t base = 0; base < ntiles; base += blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const uint4 t = i < ntiles ? tiles[i] : make_uint4(0, 0, 0, 0);
    s_l[threadIdx.x] = t.x;
    s_c[threadIdx.x] = t.y;
    s_m[threadIdx.x] = t.z;
    __syncthreads();
    for (unsigned o = 1; o < blockDim.x; o <<= 1) {  // Hillis-Steele inclusive
      unsigned long long al = 0, ac = 0, am = 0;
      if (threadIdx.x >= o) {
        al = s_l[threadIdx.x - o];
        ac = s_c[threadIdx.x - o];
        am = s_m[threadIdx.x - o];
      }
      __syncthreads();
      s_l[threadIdx.x] += al;
      s_c[threadIdx.x] += ac;
      s_m[threadIdx.x] += am;
      __syncthreads();
    }
    if (i < ntiles) {
      tiles[i] = make_uint4((unsigned)(carry_l + s_l[threadIdx.x] - t.x), 0u,
                            (unsigned)(carry_m + s_m[threadIdx.x] - t.z), 0u);
      chunk_base[i] = carry_c + s_c[threadIdx.x] - t.y;
    }
    __syncthreads();
    carry_l += s_l[blockDim.x - 1];
    carry_c += s_c[blockDim.x - 1];
    carry_m += s_m[blockDim.x - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    totals[0] = carry_l;
    totals[1] = carry_c;
    totals[2] = carry_m;
  }
}

__global__ void __launch_bounds__(kThreads) k_sched_scatter(const uint64_t* off, uint32_t n, uint32_t thr,
                                                           bool want_chunks, const uint4* tiles,
                                                           const unsigned long long* chunk_base,
                                                           const unsigned long long* totals,
                                                           uint32_t* order, uint2* chunks, uint2* multi) {
  const uint64_t v0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kTileItems;
  Cnt3 item[kTileItems];
  Cnt3 s = {0, 0, 0};
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) {
    item[k] = vertex_counts(off, v0 + k, n, thr, want_chunks);
    s = add3(s, item[k]);
  }
  Cnt3 total;
  Cnt3 pre = block_exclusive_scan(s, total);
  const uint4 t = tiles[blockIdx.x];
  uint64_t lowpos = (uint64_t)t.x + pre.low;
  uint64_t cpos = chunk_base[blockIdx.x] + pre.chunks;
  uint64_t mpos = (uint64_t)t.z + pre.multi;
  const uint64_t lowCount = totals[0];
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) {
    const uint64_t v = v0 + k;
    if (v >= n) break;
    if (item[k].low) {
      if (order) order[lowpos] = (uint32_t)v;
      ++lowpos;
    } else {
      // high ids keep ascending order after the low group (partition.cpp:56-58)
      if (order) order[lowCount + (v - lowpos)] = (uint32_t)v;
      if (want_chunks) {
        for (unsigned j = 0; j < item[k].chunks; ++j) chunks[cpos + j] = make_uint2((uint32_t)v, j);
        if (item[k].multi) multi[mpos++] = make_uint2((uint32_t)v, (uint32_t)cpos);
        cpos += item[k].chunks;
      }
    }
  }
}

// ---- init / frontier kernels -------------------------------------------------
__global__ void k_init_ranks(const uint64_t* offF, uint32_t n, const double* init, double uniform,
                             double* r0, double* r1, double* c0, double* c1) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const double r = init ? init[v] : uniform;
    const double c = __ddiv_rn(r, (double)(uint32_t)(offF[v + 1] - offF[v]));
    r0[v] = r;
    if (r1) r1[v] = r;
    c0[v] = c;
    if (c1) c1[v] = c;
  }
}

// initialAffected (frontier.cpp:43-51): dels mark np[u] and va[v]; ins mark
// np[u].  Pending sources go straight to the expansion lists.
__global__ void k_init_affected(const uint64_t* offF, const uint32_t* ds, const uint32_t* dd, uint64_t nd,
                                const uint32_t* is, uint64_t ni, uint8_t* va, uint8_t* np, uint32_t T,
                                uint32_t* pl, uint32_t* ph, SweepRed* red) {
  const uint64_t total = nd + ni;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < total; base += stride) {
    const uint64_t i = base + threadIdx.x;
    bool pend = false, lowout = false;
    uint32_t u = 0;
    if (i < total) {
      if (i < nd) {
        u = ds[i];
        va[dd[i]] = 1;
      } else {
        u = is[i - nd];
      }
      if (np) np[u] = 1;
      pend = true;
      lowout = (offF[u + 1] - offF[u]) <= T;
    }
    if (pl) warp_append(pend, lowout, u, pl, ph, red);
  }
}

__global__ void k_collect_pending(const uint64_t* offF, uint32_t n, const uint8_t* np, uint32_t T,
                                  uint32_t* pl, uint32_t* ph, SweepRed* red) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint64_t v = base + threadIdx.x;
    bool pend = false, lowout = false;
    if (v < n && np[v]) {
      pend = true;
      lowout = (offF[v + 1] - offF[v]) <= T;
    }
    warp_append(pend, lowout, (uint32_t)v, pl, ph, red);
  }
}

// expandAffected (frontier.cpp:55-84) split by out-degree: thread per
// low pending vertex, warp per high pending vertex.  Byte stores of 1 are
// idempotent, so duplicates and races are benign.
__global__ void k_expand_low(const uint64_t* off, const uint32_t* tgt, const uint32_t* list, uint32_t cnt,
                             uint8_t* va) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = list[i];
    const uint64_t b = off[u], e = off[u + 1];
    for (uint64_t k = b; k < e; ++k) va[tgt[k]] = 1;
  }
}
__global__ void k_expand_high(const uint64_t* off, const uint32_t* tgt, const uint32_t* list, uint32_t cnt,
                              uint8_t* va) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  const unsigned lane = lane_id();
  for (uint64_t i = warp; i < cnt; i += nw) {
    const uint32_t u = list[i];
    const uint64_t b = off[u], e = off[u + 1];
    for (uint64_t k = b + lane; k < e; k += 32) va[tgt[k]] = 1;
  }
}

// ---- norms ------------------------------------------------------------------
__global__ void k_linf(const double* a, const double* b, uint64_t n, unsigned long long* out) {
  double m = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double t = fabs(__dsub_rn(a[i], b[i]));
    if (t > m) m = t;
  }
  m = warp_max(m);
  __shared__ double s[kWarps];
  if (lane_id() == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kWarps; ++i) m = fmax(m, s[i]);
    if (m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
}
// blockSum (parallel.hpp:41-59): 4096-element blocks summed sequentially,
// partials combined in block order -> bit-identical to the reference.
__global__ void k_l1_blocks(const double* a, const double* b, uint64_t n, double* partials) {
  const uint64_t nb = (n + 4095) / 4096;
  for (uint64_t blk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; blk < nb;
       blk += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s0 = blk * 4096, e = s0 + 4096 < n ? s0 + 4096 : n;
    double s = 0.0;
    for (uint64_t i = s0; i < e; ++i) s = __dadd_rn(s, fabs(__dsub_rn(a[i], b[i])));
    partials[blk] = s;
  }
}
__global__ void k_l1_final(const double* partials, uint64_t nb, double* out) {
  double t = 0.0;
  for (uint64_t i = 0; i < nb; ++i) t = __dadd_rn(t, partials[i]);
  *out = t;
}

}  // namespace

// ---------------------------------------------------------------------------
Schedule build_schedule(dynpr_context* ctx, const dynpr_graph* g, uint32_t thr, uint32_t* order,
                        bool want_chunks) {
  Schedule s;
  s.threshold = thr;
  const uint32_t n = g->n;
  if (n == 0) return s;
  cudaStream_t st = ctx->stream;
  const uint64_t ntiles = ((uint64_t)n + kTile - 1) / kTile;
  uint4* tiles = ctx->tile_counts.as<uint4>(ntiles);
  auto* cb = ctx->scratch64a.as<unsigned long long>(ntiles + 4);
  unsigned long long* totals = cb + ntiles;
  k_sched_count<<<(unsigned)ntiles, kThreads, 0, st>>>(g->off, n, thr, want_chunks, tiles);
  check_launch();
  k_sched_scan<<<1, 1024, 0, st>>>(tiles, ntiles, totals, cb);
  check_launch();
  count_launch(ctx, 2);
  unsigned long long h[3];
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, totals, sizeof h, cudaMemcpyDeviceToHost, st));
  sync(ctx);
  std::memcpy(h, ctx->pinned, sizeof h);
  s.n_low = (uint32_t)h[0];
  s.n_high = n - s.n_low;
  s.n_chunks = h[1];
  s.n_multi = (uint32_t)h[2];
  uint2* chunks = nullptr;
  uint2* multi = nullptr;
  if (want_chunks) {
    chunks = ctx->sched_chunks.as<uint2>(s.n_chunks + 1);
    multi = ctx->sched_multi.as<uint2>((uint64_t)s.n_multi + 1);
    s.partials = ctx->partials.as<double>(s.n_chunks + 1);
  }
  k_sched_scatter<<<(unsigned)ntiles, kThreads, 0, st>>>(g->off, n, thr, want_chunks, tiles, cb, totals, order,
                                                        chunks, multi);
  check_launch();
  count_launch(ctx);
  s.chunks = chunks;
  s.multi = multi;
  return s;
}

void launch_sweep(dynpr_context* ctx, const SweepArgs& a, bool flagged, bool closed, uint32_t n_low_hint) {
  cudaStream_t st = ctx->stream;
  const unsigned max_blocks = (unsigned)ctx->num_sms * 8;
  (void)n_low_hint;
  const unsigned g_low = grid_for(a.n, kThreads, max_blocks);
  const unsigned g_chunk = grid_for(a.n_chunks, kThreads, max_blocks);
  const unsigned g_multi = grid_for(a.n_multi, kThreads, max_blocks);
#define DYNPR_SWEEP(F, C)                                                        \
  do {                                                                           \
    k_sweep_low<F, C><<<g_low, kThreads, 0, st>>>(a);                            \
    if (a.n_chunks) k_sweep_chunks<F, C><<<g_chunk, kThreads, 0, st>>>(a);       \
    if (a.n_multi) k_sweep_multi<F, C><<<g_multi, kThreads, 0, st>>>(a);         \
  } while (0)
  if (flagged) {
    if (closed) DYNPR_SWEEP(true, true); else DYNPR_SWEEP(true, false);
  } else {
    if (closed) DYNPR_SWEEP(false, true); else DYNPR_SWEEP(false, false);
  }
#undef DYNPR_SWEEP
  check_launch();
  count_launch(ctx, 1 + (a.n_chunks ? 1 : 0) + (a.n_multi ? 1 : 0));
}

void launch_init_ranks(dynpr_context* ctx, const dynpr_graph* gF, const double* init, double uniform, double* r0,
                       double* r1, double* c0, double* c1) {
  if (!gF->n) return;
  k_init_ranks<<<grid_for(gF->n, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(gF->off, gF->n, init,
                                                                                          uniform, r0, r1, c0, c1);
  check_launch();
  count_launch(ctx);
}

void launch_init_affected(dynpr_context* ctx, const dynpr_graph* gF, const uint32_t* ds, const uint32_t* dd,
                          uint64_t nd, const uint32_t* is, uint64_t ni, uint8_t* va, uint8_t* np, uint32_t T,
                          uint32_t* pend_low, uint32_t* pend_high, SweepRed* red) {
  if (nd + ni == 0) return;
  k_init_affected<<<grid_for(nd + ni, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(
      gF->off, ds, dd, nd, is, ni, va, np, T, pend_low, pend_high, red);
  check_launch();
  count_launch(ctx);
}

void launch_collect_pending(dynpr_context* ctx, const dynpr_graph* gF, const uint8_t* np, uint32_t T,
                            uint32_t* pend_low, uint32_t* pend_high, SweepRed* red) {
  if (!gF->n) return;
  k_collect_pending<<<grid_for(gF->n, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(
      gF->off, gF->n, np, T, pend_low, pend_high, red);
  check_launch();
  count_launch(ctx);
}

void launch_expand(dynpr_context* ctx, const dynpr_graph* gF, uint8_t* va, const uint32_t* pend_low,
                   uint32_t n_low, const uint32_t* pend_high, uint32_t n_high) {
  if (n_low) {
    k_expand_low<<<grid_for(n_low, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(gF->off, gF->tgt,
                                                                                            pend_low, n_low, va);
    check_launch();
    count_launch(ctx);
  }
  if (n_high) {
    k_expand_high<<<grid_for((uint64_t)n_high * 32, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(
        gF->off, gF->tgt, pend_high, n_high, va);
    check_launch();
    count_launch(ctx);
  }
}

void launch_linf(dynpr_context* ctx, const double* a, const double* b, uint64_t n, unsigned long long* out_bits) {
  DYNPR_CK(cudaMemsetAsync(out_bits, 0, 8, ctx->stream));
  if (!n) return;
  k_linf<<<grid_for(n, kThreads, ctx->num_sms * 8), kThreads, 0, ctx->stream>>>(a, b, n, out_bits);
  check_launch();
  count_launch(ctx);
}

void launch_l1(dynpr_context* ctx, const double* a, const double* b, uint64_t n, double* partials, double* out) {
  const uint64_t nb = (n + 4095) / 4096;
  if (nb) {
    k_l1_blocks<<<grid_for(nb, 128), 128, 0, ctx->stream>>>(a, b, n, partials);
    check_launch();
  }
  k_l1_final<<<1, 1, 0, ctx->stream>>>(partials, nb, out);
  check_launch();
  count_launch(ctx, 2);
}

}  // namespace dynpr_b200
