// Rank-update sweep, degree partition, frontier and norm kernels
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
// so the ranks, the L-inf delta and every threshold decision are
// bit-identical to the reference CPU library.
//
// Parallel decomposition over the engine layout (layout.cuh), the paper's
// low/high kernel pair recast for the B200 memory system:
//   k_sweep_single  warp per SELL-32 slice of 32 single-segment vertices
//                   (in-degree <= max(T, 256), sorted by in-degree so the
//                   32 lanes have near-equal trip counts); lane = vertex
//   k_sweep_mseg    warp per slice of 32 256-edge chunks of the high
//                   in-degree ("multi") vertices; lane = chunk -> partial
//   k_sweep_mfinal  thread per multi vertex: partials combined in chunk order
// Index loads are coalesced 128-byte lines (lane-interleaved SELL storage,
// streamed past L1); contribution gathers go through the read-only path into
// a relabelled vector whose hot entries are packed at its front.  One fused
// epilogue: closed-loop / plain rank formula, the next sweep's contribution
// r/outdeg (IEEE division, bit-identical to the reference's per-edge
// division), copy-through of unaffected vertices, prune / frontier flags,
// warp-aggregated append of pending vertices to the out-degree-split
// expansion lists, and the L-inf / count reductions finished with one 64-bit
// atomic per block.
//
// Frontier expansion (frontier.cpp:55-84) is direction-optimising: push over
// the relabelled out-CSR (thread per low out-degree vertex, warp per
// 1024-edge item of a high one) when the pending set is small, pull over
// the SELL in-lists of the still-unaffected vertices (early exit on the first
// pending in-neighbour) when pushing would touch more edges.  Both produce
// exactly vertexAffected |= out(pending).
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>

#include "prims.cuh"
#include "sweep.cuh"

namespace dynpr_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

struct Acc {
  double dmax = 0.0;
  unsigned long long proc = 0, edges = 0, pedges = 0;
};

// ---- block reductions ----------------------------------------------------
// (kWarps-sized arrays: with the L1-preferring carveout the SM keeps an 8 KB
// shared-memory configuration, and 1 KB of static shared memory per block
// (+1 KB reserved by the driver) capped the 48-register single-slice kernel
// at 4 blocks per SM -- 32 warps -- instead of its register limit of 5.)
__device__ __forceinline__ void block_reduce_commit(Acc acc, SweepRed* red) {
  __shared__ double s_d[kWarps];
  __shared__ unsigned long long s_p[kWarps], s_e[kWarps], s_q[kWarps];
  acc.dmax = warp_max(acc.dmax);
  acc.proc = warp_sum(acc.proc);
  acc.edges = warp_sum(acc.edges);
  acc.pedges = warp_sum(acc.pedges);
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) {
    s_d[w] = acc.dmax;
    s_p[w] = acc.proc;
    s_e[w] = acc.edges;
    s_q[w] = acc.pedges;
  }
  __syncwarp();  // reconverge the warp after the lane-divergent store
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    unsigned long long p = 0, e = 0, q = 0;
    for (int i = 0; i < kWarps; ++i) {  // every caller runs kThreads-thread blocks
      d = fmax(d, s_d[i]);
      p += s_p[i];
      e += s_e[i];
      q += s_q[i];
    }
    if (d > 0.0) atomicMax(&red->delta_bits, (unsigned long long)__double_as_longlong(d));
    if (p) atomicAdd(&red->processed, p);
    if (e) atomicAdd(&red->edges, e);
    if (q) atomicAdd(&red->pend_edges, q);
  }
}

// Warp-aggregated append of pending vertices (all 32 lanes must call it):
// low out-degree vertices go to `pl` one entry each, the others to `ph` as
// ceil(outdeg / 1024) (vertex, chunk) work items.
__device__ __forceinline__ void warp_append_to(bool pend, bool lowout, uint32_t v, uint32_t od, uint32_t* pl,
                                               uint2* ph, unsigned* cnt_low, unsigned* cnt_high) {
  const unsigned ml = __ballot_sync(kFull, pend && lowout);
  const unsigned items = (pend && !lowout) ? (od + kExpandChunk - 1) / kExpandChunk : 0u;
  const unsigned mh = __ballot_sync(kFull, items != 0);
  if (!(ml | mh)) return;
  const unsigned lane = lane_id();
  unsigned incl = items;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if ((int)lane >= o) incl += y;
  }
  const unsigned total = __shfl_sync(kFull, incl, 31);
  unsigned bl = 0, bh = 0;
  if (lane == 0) {
    if (ml) bl = atomicAdd(cnt_low, (unsigned)__popc(ml));
    if (total) bh = atomicAdd(cnt_high, total);
  }
  bl = __shfl_sync(kFull, bl, 0);
  bh = __shfl_sync(kFull, bh, 0);
  const unsigned lt = (1u << lane) - 1u;
  if (pend && lowout) pl[bl + __popc(ml & lt)] = v;
  for (unsigned j = 0, b = bh + incl - items; j < items; ++j) ph[b + j] = make_uint2(v, j);
}
__device__ __forceinline__ void warp_append(bool pend, bool lowout, uint32_t v, uint32_t od, uint32_t* pl,
                                            uint2* ph, SweepRed* red) {
  warp_append_to(pend, lowout, v, od, pl, ph, &red->pend_low, &red->pend_high);
}

// A new contribution of vertex v: the local buffer and, in a multi-GPU team
// with peer-mapped buffers, every peer's copy (NVLink stores issued from the
// epilogue, so the exchange overlaps the sweep instead of following it).
__device__ __forceinline__ void store_contrib(const SweepArgs& a, uint32_t v, double c) {
  a.contrib_cur[v] = c;
  for (int p = 0; p < a.npeers; ++p) a.peer_cur[p][v] = c;
}

// Unaffected vertex (rank.cpp:90-92): current = previous.  In engine mode
// only vertices written by the previous sweep differ between the buffers.
__device__ __forceinline__ void copy_through(const SweepArgs& a, uint32_t v) {
  if (a.copy_all) {
    a.rank_cur[v] = a.rank_prev[v];
    if (a.contrib_cur) a.contrib_cur[v] = a.contrib_prev[v];
  } else if (const uint8_t w = a.written[v]) {
    a.rank_cur[v] = a.rank_prev[v];
    store_contrib(a, v, fabs(a.contrib_prev[v]));  // (clears an in-sweep-pull pending bit)
    a.written[v] = w - 1;
  }
  if (a.np && !a.np_accumulate) a.np[v] = 0;
}

// The same with the vertex's `written` count and previous rank / contribution
// already loaded (with its flags, one round trip earlier): the split
// single-slice sweep (RMAT-24 DF-P 1e-4 13.51 -> 13.19 ms with the 4-deep
// k_init_ranks; the latency-mode sweep was 2-5% slower with it and keeps
// copy_through).
__device__ __forceinline__ void copy_through_loaded(const SweepArgs& a, uint32_t v, unsigned wr, double pv,
                                                    double cprev) {
  if (a.copy_all) {
    copy_through(a, v);
    return;
  }
  if (wr) {
    a.rank_cur[v] = pv;
    store_contrib(a, v, fabs(cprev));
    a.written[v] = (uint8_t)(wr - 1);
  }
  if (a.np && !a.np_accumulate) a.np[v] = 0;
}
// Is v owed a copy-through (see copy_through)?  Loaded with the flags.
__device__ __forceinline__ unsigned written_of(const SweepArgs& a, uint32_t v, bool valid) {
  return (valid && a.written && !a.copy_all) ? a.written[v] : 0u;
}

// Fused epilogue: rank formula (rank.cpp:97-106), next contribution, delta,
// flags (rank.cpp:108-115).
// `newly`: the vertex became affected in this sweep's in-sweep pull.
template <bool FLAGGED, bool CLOSED>
__device__ __forceinline__ void finalize(const SweepArgs& a, uint32_t v, double c, double pv, uint32_t od,
                                         Acc& acc, bool& pend, bool& lowout, bool newly = false) {
  const double d = (double)od;
  double r;
  if (CLOSED) {
    r = __ddiv_rn(__dadd_rn(a.teleport, __dmul_rn(a.alpha, __dsub_rn(c, __ddiv_rn(pv, d)))),
                  __dsub_rn(1.0, __ddiv_rn(a.alpha, d)));
  } else {
    r = __dadd_rn(a.teleport, __dmul_rn(a.alpha, c));
  }
  a.rank_cur[v] = r;
  const double dr = fabs(__dsub_rn(r, pv));
  if (dr > acc.dmax) acc.dmax = dr;  // NaN never wins, like blockMax (parallel.hpp:66-73)
  bool signbit = false;
  if (FLAGGED) {
    const double denom = r > pv ? r : pv;
    const double rel = denom > 0.0 ? __ddiv_rn(dr, denom) : 0.0;
    if (CLOSED && rel <= a.tp) {
      a.va[v] = 0;
    } else if (newly) {
      a.va[v] = 1;
    }
    pend = rel > a.tf;
    if (a.np) {
      if (a.np_accumulate) {
        if (pend) a.np[v] = 1;
      } else {
        a.np[v] = pend;
      }
    }
    lowout = od <= a.T;
    if (pend) acc.pedges += od;
    signbit = a.pull_fused && pend;
    if (a.written) a.written[v] = signbit ? 2 : 1;
  }
  if (a.contrib_cur) {
    const double q = __ddiv_rn(r, d);
    store_contrib(a, v, signbit ? -q : q);
  }
}

// Index streams bypass L1 (L1::no_allocate) so the gathered contributions
// -- the hot ones packed at the front of the relabelled vector -- keep it.
__device__ __forceinline__ uint4 ld_idx4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// A contribution: the vertex's own (self-loop) value from a register (it
// was loaded coalesced with the vertex's other operands), everything else
// through the read-only path.  A shared-memory cache of the hottest
// contributions was measured and rejected (profiles/r01/README.md): it
// served only ~15% of RMAT-24 gathers and its 1024-thread CTAs halved
// occupancy; random 8-byte gathers top out near 288 G/s from L2
// (profiles/microbench_gather.cu), which is what bounds this sweep.
__device__ __forceinline__ double ld_contrib(const double* __restrict__ contrib, uint32_t u, uint32_t self,
                                             double cself) {
  return u == self ? cself : __ldg(contrib + u);
}

// A single-region segment longer than the flat limit max(T, 256) belongs to
// a chunked vertex (rank.cpp:59-75) that an incrementally derived layout left
// in its single slice (layout.cu): its lane folds the running partial into
// the total at every 256-element boundary -- c = ((0 + p0) + p1) + ..., the
// reference's chunk order exactly.  Never true in a freshly built layout.
__device__ __forceinline__ bool folds(const SweepArgs& a, uint32_t len) {
#ifdef DYNPR_NO_FOLD  // A/B builds only (profiles/ab_static_layouts.py)
  return false;
#endif
  return len > (a.T > kAccumChunk ? a.T : kAccumChunk);
}

// Lane-sequential sum of one SELL-32x4 segment (layout.cuh sell_pos):
// elements 4j..4j+3 of this lane arrive with one 16-byte load.  Index loads
// for the next 8 elements are issued before the adds of the current 8
// (software pipelining); the adds stay in segment order.  `fold`: chunked
// accumulation (see folds()).
// Contributions are summed as |x| (the sign bit may carry an in-sweep-pull
// pending flag, see SweepArgs::pull_fused); NEG also ORs the sign bits of the
// gathered values into *neg (bit 31).
template <bool NEG = false>
__device__ __forceinline__ double segment_sum(const uint32_t* __restrict__ sell, uint64_t base, unsigned lane,
                                              uint32_t len, uint32_t Lw, const double* __restrict__ contrib,
                                              uint32_t self, double cself, unsigned* neg = nullptr,
                                              bool fold = false) {
  unsigned nb = 0;
  const uint32_t* p = sell + base + 4u * lane;  // element k at p + 32*k (k % 4 == 0)
  const uint4 z = make_uint4(0, 0, 0, 0);
  double c = 0.0, tot = 0.0;
  uint4 a = len > 0 ? ld_idx4(p) : z;
  uint4 b = len > 4 ? ld_idx4(p + 128) : z;
  for (uint32_t k = 0; k < Lw; k += 8) {
    const uint32_t u[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    double x[8];
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q)
      x[q] = (k + q < len) ? ld_contrib(contrib, u[q], self, cself) : 0.0;
    a = (k + 8 < len) ? ld_idx4(p + 32ull * (k + 8)) : z;
    b = (k + 12 < len) ? ld_idx4(p + 32ull * (k + 12)) : z;
    if (fold && k != 0 && (k & (kAccumChunk - 1)) == 0 && k < len) {
      tot = __dadd_rn(tot, c);
      c = 0.0;
    }
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
      if (k + q < len) c = __dadd_rn(c, fabs(x[q]));
      if (NEG) nb |= (unsigned)__double2hiint(x[q]);  // (0.0 past the end)
    }
  }
  if (NEG) *neg = nb >> 31;
  return fold ? __dadd_rn(tot, c) : c;
}

// The segment sum of a warp holding a folding lane (folds(): derived layouts
// only, rare): chunked accumulation, c = ((0 + p0) + p1) + ..., with the
// sign-bit OR.  Out of line, so its extra live state does not weigh on the
// register allocation of the common path (the fused sweep spilled 168 B
// instead of 72 B with the fold inlined; RMAT-20 Static 4.67 -> 4.35 ms).
__device__ __noinline__ double segment_sum_folding(const uint32_t* __restrict__ sell, uint64_t base, unsigned lane,
                                                   uint32_t len, uint32_t Lw, const double* __restrict__ contrib,
                                                   uint32_t self, double cself, bool fold, unsigned* neg) {
  const uint32_t* p = sell + base + 4u * lane;
  double c = 0.0, tot = 0.0;
  unsigned nb = 0;
  for (uint32_t k = 0; k < Lw; k += 4) {
    const uint4 w = k < len ? ld_idx4(p + 32ull * k) : make_uint4(0, 0, 0, 0);
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
    double x[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) x[q] = (k + q < len) ? ld_contrib(contrib, u[q], self, cself) : 0.0;
    if (fold && k != 0 && (k & (kAccumChunk - 1)) == 0 && k < len) {
      tot = __dadd_rn(tot, c);
      c = 0.0;
    }
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      if (k + q < len) c = __dadd_rn(c, fabs(x[q]));
      nb |= (unsigned)__double2hiint(x[q]);
    }
  }
  *neg = nb >> 31;
  return fold ? __dadd_rn(tot, c) : c;
}

// Does any element of this lane's SELL segment hit a pending vertex?
__device__ __forceinline__ bool segment_any_pending(const uint32_t* __restrict__ sell, uint64_t base, unsigned lane,
                                                    uint32_t len, const uint8_t* __restrict__ np) {
  const uint32_t* p = sell + base + 4u * lane;
  const uint4 z = make_uint4(0, 0, 0, 0);
  bool found = false;
  for (uint32_t k = 0;; k += 8) {
    const bool active = !found && k < len;
    if (!__any_sync(kFull, active)) break;
    if (active) {
      const uint4 a = ld_idx4(p + 32ull * k);
      const uint4 b = (k + 4 < len) ? ld_idx4(p + 32ull * (k + 4)) : z;
      const uint32_t u[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q)
        if (k + q < len && np[u[q]]) found = true;
    }
  }
  return found;
}

// Device-loop arguments (the cached loop graph, engine.cu): the SweepArgs of
// the solve's two half-iterations live in the constant bank, rewritten per
// solve (stream-ordered), so one instantiated graph serves every snapshot of
// the same launch shape and the kernels still read their arguments as
// constant operands, exactly like by-value kernel parameters.  (Arguments
// staged through shared memory were measured 8-15% slower on RMAT-22/24.)
__constant__ SweepArgs c_loop_args[2];

// Sweep kernels: persistent grids of 256-thread CTAs at full occupancy.
constexpr int kSweepThreads = kThreads;
constexpr int kSweepWarps = kSweepThreads / 32;
// k_sweep_single: slices per dynamic grab, 8 (was 4; measured in the loop
// graph, profiles/r02/s5/*split_grab_ab.txt: Static RMAT-24 55.93 -> 55.62
// ms, RMAT-25 117.7 -> 116.7, RMAT-26 within noise, 2 was 5-7% slower;
// DF-P RMAT-24 1e-6 / 1e-5 / 1e-4 / 1e-3 6.21 -> 6.16, 6.43 -> 6.37,
// 13.06 -> 13.00, 27.47 -> 27.35 ms, RMAT-26 1e-4 61.3 -> 61.0; 16 was
// 10-17% slower).  The latency-mode sweep's light grabs stay at 2 (4 made
// RMAT-20 DF-P 1e-7 19% slower, frontier_grab_ab.txt).
constexpr unsigned kSplitGrab = 8;

// ---- single-segment vertices: warp per 32-vertex slice ------------------------
// In-sweep pull (SweepArgs::pull_fused): this sweep follows an expansion
// decided as a pull.
__device__ __forceinline__ bool pull_now(const SweepArgs& a) {
  return a.pull_fused && a.expand && *a.expand == kExpandPull;
}

template <bool FLAGGED, bool CLOSED>
__device__ __forceinline__ void b_sweep_single(const SweepArgs& a) {
  if (a.done && *a.done) return;
  Acc acc;
  const unsigned lane = lane_id();
  const bool pull = FLAGGED && pull_now(a);
  // slices grabbed dynamically, kSplitGrab at a time (counter in the record)
  for (;;) {
    unsigned g = 0;
    if (lane == 0) g = atomicAdd(&a.red->ticket_light, kSplitGrab);
    g = __shfl_sync(kFull, g, 0);
    const uint64_t s0 = a.ss_lo + g;
    if (s0 >= a.ss_hi) break;
    const uint64_t s1 = s0 + kSplitGrab < a.ss_hi ? s0 + kSplitGrab : a.ss_hi;
    // the grab's slice bases in one load (lane i: slice s0 + i), so a
    // slice's index loads do not wait for its own base load
    const uint64_t sb_lane = s0 + lane < s1 ? a.sbase[s0 + lane] : 0ull;
  for (uint64_t s = s0; s < s1; ++s) {
    const uint64_t sb = __shfl_sync(kFull, sb_lane, (int)(s - s0));
    const uint64_t vv = (uint64_t)a.M + s * 32 + lane;
    const bool valid = vv < a.n;
    const uint32_t v = (uint32_t)vv;
    const uint32_t deg = valid ? a.indeg[v] : 0u;
    bool aff = valid;
    unsigned wr = 0;
    if (FLAGGED) {
      aff = valid && a.va[v];
      wr = written_of(a, v, valid);
    }
    const bool scan = pull && valid && !aff;  // in-sweep pull: any pending in-neighbour?
    const uint32_t len = (aff || scan) ? deg : 0u;
    const uint32_t Lw = __reduce_max_sync(kFull, len);
    double pv = 0.0, cself = 0.0;
    uint32_t od = 0;
    if (aff || scan) {  // prefetch the epilogue operands (and the self-loop term)
      pv = a.rank_prev[v];
      od = a.outdeg[v];
      cself = a.contrib_prev[v];
    } else if (FLAGGED && wr) {  // a copy-through's operands
      pv = a.rank_prev[v];
      cself = a.contrib_prev[v];
    }
    double c = 0.0;
    unsigned neg = 0;
    if (Lw == 1 && a.loops) {  // self-loops only: 0.0 + |cself| (rank.cpp:45-54)
      if (len) {
        c = fabs(cself);
        neg = (unsigned)__double2hiint(cself) >> 31;
      }
    } else if (Lw) {
      // (the split kernel keeps the fold inline: 48 registers either way)
      if (pull)
        c = segment_sum<true>(a.sell_s, sb, lane, len, Lw, a.contrib_prev, v, cself, &neg, folds(a, len));
      else
        c = segment_sum(a.sell_s, sb, lane, len, Lw, a.contrib_prev, v, cself, nullptr, folds(a, len));
    }
    const bool newly = scan && neg;
    bool pend = false, lowout = false;
    if (valid) {
      if (!aff && !newly) {
        copy_through_loaded(a, v, wr, pv, cself);
      } else {
        finalize<FLAGGED, CLOSED>(a, v, c, pv, od, acc, pend, lowout, newly);
        ++acc.proc;
        acc.edges += deg;
      }
    }
    if (FLAGGED && a.pend_low && !(pull && a.lazy_lists)) warp_append(pend, lowout, v, od, a.pend_low, a.pend_high, a.red);
  }
  }
  if (a.npeers) __threadfence_system();  // peer stores visible before the team barrier
  block_reduce_commit(acc, a.red);
}
template <bool FLAGGED, bool CLOSED>
__global__ void __launch_bounds__(kSweepThreads, 5) k_sweep_single(SweepArgs a) {
  b_sweep_single<FLAGGED, CLOSED>(a);
}
template <bool FLAGGED, bool CLOSED, int H>
__global__ void __launch_bounds__(kSweepThreads, 5) k_sweep_single_c() {
  b_sweep_single<FLAGGED, CLOSED>(c_loop_args[H]);
}

// ---- multi vertices: warp per slice of 32 chunks -> partials -------------------
template <bool FLAGGED>
__device__ __forceinline__ void b_sweep_mseg(const SweepArgs& a) {
  if (a.done && *a.done) return;
  const unsigned lane = lane_id();
  const bool pull = FLAGGED && pull_now(a);
  for (;;) {  // slices grabbed dynamically (counter in the record)
    unsigned g = 0;
    if (lane == 0) g = atomicAdd(&a.red->ticket_heavy, 1u);
    const uint64_t s = a.ms_lo + __shfl_sync(kFull, g, 0);
    if (s >= a.ms_hi) break;
    const uint64_t seg = s * 32 + lane;
    uint32_t len = 0, v = 0xffffffffu;
    if (seg < a.n_mseg) {
      len = a.mseg_len[seg];
      v = a.mseg_v[seg];
      if (v < a.v_lo || v >= a.v_hi) len = 0;  // another rank's vertex
      if (FLAGGED && !pull && !a.va[v]) len = 0;
    }
    const uint32_t Lw = __reduce_max_sync(kFull, len);
    if (!Lw) continue;
    // (a multi vertex's self-loop is one gather among >256: not special-cased)
    if (pull) {  // the chunk's "any pending source" rides in the partial's sign bit
      unsigned neg = 0;
      const double c =
          segment_sum<true>(a.sell_m, a.mbase[s], lane, len, Lw, a.contrib_prev, 0xffffffffu, 0.0, &neg);
      if (len) a.partials[seg] = neg ? -c : c;
    } else {
      const double c = segment_sum(a.sell_m, a.mbase[s], lane, len, Lw, a.contrib_prev, 0xffffffffu, 0.0);
      if (len) a.partials[seg] = c;
    }
  }
}
template <bool FLAGGED>
__global__ void __launch_bounds__(kSweepThreads) k_sweep_mseg(SweepArgs a) {
  b_sweep_mseg<FLAGGED>(a);
}
template <bool FLAGGED, int H>
__global__ void __launch_bounds__(kSweepThreads) k_sweep_mseg_c() {
  b_sweep_mseg<FLAGGED>(c_loop_args[H]);
}

// ---- multi vertices: ordered combine (rank.cpp:72) + epilogue --------------------
// Ordered sum of n partials by a whole warp (rank.cpp:72): one coalesced load
// per 32 partials, then a shuffle-broadcast sequential sum whose shuffles are
// independent of the add chain (full groups unrolled), so the critical path
// is n dependent DADDs instead of n dependent loads.
// Partials are summed as |x|; *neg = OR of their sign bits (in-sweep pull).
__device__ __forceinline__ double warp_ordered_sum(const double* __restrict__ p, uint32_t n, bool* neg) {
  const unsigned lane = lane_id();
  double sum = 0.0;
  unsigned nb = 0;
  uint32_t g = 0;
  for (; g + 32 <= n; g += 32) {
    const double x = p[g + lane];
    nb |= (unsigned)__double2hiint(x);
#pragma unroll
    for (int j = 0; j < 32; ++j) sum = __dadd_rn(sum, fabs(__shfl_sync(kFull, x, j)));
  }
  if (g < n) {
    const double x = g + lane < n ? p[g + lane] : 0.0;
    nb |= (unsigned)__double2hiint(x);
    for (uint32_t j = 0; j < n - g; ++j) sum = __dadd_rn(sum, fabs(__shfl_sync(kFull, x, j)));
  }
  *neg = (__reduce_or_sync(kFull, nb) >> 31) != 0;
  return sum;
}

constexpr uint32_t kWarpCombineChunks = 32;  // multi vertices with more partials are combined by a warp

template <bool FLAGGED, bool CLOSED>
__device__ __forceinline__ void b_sweep_mfinal(const SweepArgs& a) {
  if (a.done && *a.done) return;
  Acc acc;
  const bool pull = FLAGGED && pull_now(a);
  const uint64_t vend = a.M < a.v_hi ? a.M : a.v_hi;
  // the multi vertices are sorted by in-degree (descending): [0, Mb) have
  // more than kWarpCombineChunks partials
  __shared__ uint32_t s_mb;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = a.M;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (a.indeg[mid] > kWarpCombineChunks * kAccumChunk) lo = mid + 1; else hi = mid;
    }
    s_mb = lo;
  }
  __syncwarp();  // reconverge the warp after the lane-divergent store
  __syncthreads();
  const uint64_t mb = s_mb;
  // phase 1: warp per heavy multi vertex
  {
    const uint64_t lo = a.v_lo, hi = mb < vend ? mb : vend;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
    for (uint64_t vv = lo + warp; vv < hi; vv += nw) {
      const uint32_t v = (uint32_t)vv;
      bool pend = false, lowout = false;
      uint32_t od = 0;
      const bool aff = !FLAGGED || a.va[v];
      if (!aff && !pull) {
        if (lane_id() == 0) copy_through(a, v);
      } else {
        const uint32_t deg = a.indeg[v];
        const uint32_t pb = a.pbase[v];
        bool neg = false;
        const double c = warp_ordered_sum(a.partials + pb, (deg + kAccumChunk - 1) / kAccumChunk, &neg);
        const bool newly = !aff && neg;
        if (lane_id() == 0) {
          if (!aff && !newly) {
            copy_through(a, v);
          } else {
            od = a.outdeg[v];
            finalize<FLAGGED, CLOSED>(a, v, c, a.rank_prev[v], od, acc, pend, lowout, newly);
            ++acc.proc;
            acc.edges += deg;
          }
        }
      }
      if (FLAGGED && a.pend_low && !(pull && a.lazy_lists)) warp_append(pend, lowout, v, od, a.pend_low, a.pend_high, a.red);
    }
  }
  // phase 2: thread per remaining multi vertex, partials loaded 8 ahead
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t first = a.v_lo > mb ? a.v_lo : mb;
  for (uint64_t base = first + (uint64_t)blockIdx.x * kThreads; base < vend; base += stride) {
    const uint64_t vv = base + threadIdx.x;
    bool pend = false, lowout = false;
    const uint32_t v = (uint32_t)vv;
    uint32_t od = 0;
    if (vv < vend) {
      const bool aff = !FLAGGED || a.va[v];
      if (!aff && !pull) {
        copy_through(a, v);
      } else {
        const uint32_t deg = a.indeg[v];
        const uint32_t nch = (deg + kAccumChunk - 1) / kAccumChunk;
        const double* p = a.partials + a.pbase[v];
        double c = 0.0;
        unsigned nb = 0;
        for (uint32_t q = 0; q < nch; q += 8) {
          double x[8];
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j) x[j] = q + j < nch ? p[q + j] : 0.0;
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j) {
            if (q + j < nch) c = __dadd_rn(c, fabs(x[j]));
            nb |= (unsigned)__double2hiint(x[j]);
          }
        }
        const bool newly = !aff && (nb >> 31);
        if (!aff && !newly) {
          copy_through(a, v);
        } else {
          od = a.outdeg[v];
          finalize<FLAGGED, CLOSED>(a, v, c, a.rank_prev[v], od, acc, pend, lowout, newly);
          ++acc.proc;
          acc.edges += deg;
        }
      }
    }
    if (FLAGGED && a.pend_low && !(pull && a.lazy_lists)) warp_append(pend, lowout, v, od, a.pend_low, a.pend_high, a.red);
  }
  if (a.npeers) __threadfence_system();  // peer stores visible before the team barrier
  block_reduce_commit(acc, a.red);
}
template <bool FLAGGED, bool CLOSED>
__global__ void __launch_bounds__(kThreads) k_sweep_mfinal(SweepArgs a) {
  b_sweep_mfinal<FLAGGED, CLOSED>(a);
}
template <bool FLAGGED, bool CLOSED, int H>
__global__ void __launch_bounds__(kThreads) k_sweep_mfinal_c() {
  b_sweep_mfinal<FLAGGED, CLOSED>(c_loop_args[H]);
}

// ---- fused sweep: one kernel, dynamically scheduled ----------------------------
// The three-kernel sweep above serialises the multi-chunk slices, the
// single-vertex slices and the ordered combine; on graphs that do not fill
// the GPU many times over the sweep time is then the sum of the longest lane
// chains of each kernel (a 256-edge segment is 32 dependent gather rounds).
// The fused kernel runs all of it in one launch:
//  * heavy items first -- every multi-chunk slice, then the single slices whose
//    largest segment exceeds kHeavyDeg -- dealt round-robin to the resident
//    blocks (per-block counters), so the long chains start together at the
//    beginning of the sweep, spread over all SMs (a per-warp trace showed
//    that first-come grabbing piled several hub chains onto one SM, whose
//    request queue then set the sweep time), and gather with a 16-deep
//    pipeline; then the light single slices in global grabs of kLightGrab;
//  * a multi vertex is finished by the warp that completes its last chunk
//    (per-vertex completion counter, threadfence + atomic), which combines
//    the partials in chunk order (rank.cpp:72) with a warp-wide load and a
//    shuffle-broadcast sequential sum, and runs the epilogue.
// Every vertex's sum and epilogue are exactly those of the split kernels.
constexpr unsigned kLightGrab = 2;
// Lanes per segment in the heavy items (segment_sum_group): 2 on the most
// latency-bound graphs (at most kGroupSlicesPerWarp slices per resident warp:
// the heavy chains halve, RMAT-18 static 2.94 -> 2.51 ms), 1 above (the extra
// shuffles and spills cost 15-20% on RMAT-20/22; profiles/r02/README.md).
// DYNPR_HEAVY_LANES=1|2 overrides.
constexpr uint64_t kGroupSlicesPerWarp = 3;
// Above this many slices per resident warp the sweep is throughput-bound and
// the split kernels are used.
constexpr uint64_t kSplitSlicesPerWarp = 64;
constexpr unsigned kMaxBlocks = 4096;  // persistent grids are <= 8 x SMs

// Debug timeline (DYNPR_TRACE=1): per warp of the last fused sweep, {smid,
// start, end, heavy items | light items << 32, first heavy item, end of the
// heavy phase} in globaltimer ns; read with dynpr_debug_sweep_trace.
constexpr int kTraceWarps = 148 * 64;
__device__ unsigned long long g_trace[kTraceWarps * 6];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// (|x| sums and the optional sign-bit OR as in segment_sum)
template <int Q, bool NEG = false>
__device__ __forceinline__ double segment_sum_deep(const uint32_t* __restrict__ sell, uint64_t base, unsigned lane,
                                                   uint32_t len, uint32_t Lw, const double* __restrict__ contrib,
                                                   uint32_t self, double cself, unsigned* neg = nullptr) {
  constexpr uint32_t D = 4 * Q;  // elements in flight per lane
  unsigned nb = 0;
  const uint32_t* p = sell + base + 4u * lane;
  const uint4 z = make_uint4(0, 0, 0, 0);
  double c = 0.0;
  uint4 ix[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) ix[j] = (4u * j < len) ? ld_idx4(p + 128ull * j) : z;
  for (uint32_t k = 0; k < Lw; k += D) {
    double x[D];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const uint32_t u[4] = {ix[j].x, ix[j].y, ix[j].z, ix[j].w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        x[4 * j + q] = (k + 4 * j + q < len) ? ld_contrib(contrib, u[q], self, cself) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < Q; ++j) ix[j] = (k + D + 4 * j < len) ? ld_idx4(p + 32ull * (k + D + 4 * j)) : z;
#pragma unroll
    for (uint32_t q = 0; q < D; ++q) {
      if (k + q < len) c = __dadd_rn(c, fabs(x[q]));
      if (NEG) nb |= (unsigned)__double2hiint(x[q]);
    }
  }
  if (NEG) *neg = nb >> 31;
  return c;
}

// G lanes per segment (column `col` of a SELL slice) for the heavy items of
// the latency-mode sweep: in every round of 16G elements the lane of role r
// gathers elements [16r, 16r + 16) of the round, and the owner (role 0) adds
// its own 16 and then, in order, each other role's 16 received by shuffles
// -- the reference's sequential order with G times fewer dependent gather
// rounds on the chain (a 256-element segment: 16 rounds at G = 1).  Only
// the owner's return value is the sum; *neg is the group's sign-bit OR.
template <int G, bool NEG>
__device__ __forceinline__ double segment_sum_group(const uint32_t* __restrict__ sell, uint64_t base, unsigned col,
                                                    unsigned role, uint32_t len, uint32_t Lw,
                                                    const double* __restrict__ contrib, uint32_t self,
                                                    double cself, unsigned* neg) {
  const uint32_t* p = sell + base + 4u * col;  // element k at p + 32*k (k % 4 == 0)
  const uint4 z = make_uint4(0, 0, 0, 0);
  const unsigned owner = lane_id() - role;
  double c = 0.0;
  unsigned nb = 0;
  uint4 ix[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) ix[j] = (16u * role + 4u * j < len) ? ld_idx4(p + 32ull * (16u * role + 4u * j)) : z;
  for (uint32_t k = 0; k < Lw; k += 16u * G) {
    const uint32_t kb = k + 16u * role;
    double x[16];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t u[4] = {ix[j].x, ix[j].y, ix[j].z, ix[j].w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        x[4 * j + q] = (kb + 4 * j + q < len) ? ld_contrib(contrib, u[q], self, cself) : 0.0;
    }
    const uint32_t kn = kb + 16u * G;
#pragma unroll
    for (int j = 0; j < 4; ++j) ix[j] = (kn + 4u * j < len) ? ld_idx4(p + 32ull * (kn + 4u * j)) : z;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (NEG) nb |= (unsigned)__double2hiint(x[q]);
      if (role == 0 && k + q < len) c = __dadd_rn(c, fabs(x[q]));
    }
#pragma unroll
    for (int r = 1; r < G; ++r) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double y = __shfl_sync(kFull, x[q], owner + r);
        if (role == 0 && k + 16u * r + q < len) c = __dadd_rn(c, fabs(y));
      }
    }
  }
  if (NEG) {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) nb |= __shfl_xor_sync(kFull, nb, o);
    *neg = nb >> 31;
  }
  return c;
}

// One single-region slice (the body of k_sweep_single).
// `pull`: in-sweep pull (SweepArgs::pull_fused) -- unaffected lanes gather
// too and become affected on a pending source.
// G > 1: the heavy-item form -- part `part` of the slice, its 32/G columns
// with G lanes each (segment_sum_group); the owner lanes finish the vertices.
template <bool FLAGGED, bool CLOSED, int Q, int G = 1>
__device__ __forceinline__ void single_slice(const SweepArgs& a, uint64_t s, unsigned lane, Acc& acc, bool pull,
                                             unsigned part = 0) {
  const unsigned col = G == 1 ? lane : part * (32u / G) + lane / G;
  const unsigned role = G == 1 ? 0u : lane % G;
  const uint64_t vv = (uint64_t)a.M + s * 32 + col;
  const bool valid = vv < a.n;
  const uint32_t v = (uint32_t)vv;
  const uint32_t deg = valid ? a.indeg[v] : 0u;
  bool aff = valid;
  if (FLAGGED) aff = valid && a.va[v];
  const bool scan = FLAGGED && pull && valid && !aff;
  const uint32_t len = (aff || scan) ? deg : 0u;
  const uint32_t Lw = __reduce_max_sync(kFull, len);
  double pv = 0.0, cself = 0.0;
  uint32_t od = 0;
  if (aff || scan) {
    pv = a.rank_prev[v];
    od = a.outdeg[v];
    cself = a.contrib_prev[v];
  }
  double c = 0.0;
  unsigned neg = 0;
  if (Lw == 1 && a.loops) {  // self-loops only (see b_sweep_single)
    if (len) {
      c = fabs(cself);
      neg = (unsigned)__double2hiint(cself) >> 31;
    }
  } else if (Lw) {
    const bool fold = folds(a, len);
    if (__any_sync(kFull, fold))  // (every lane of a group computes its column's sum)
      c = segment_sum_folding(a.sell_s, a.sbase[s], col, len, Lw, a.contrib_prev, v, cself, fold, &neg);
    else if (G == 1)  // (frontier sweeps always OR the sign bits: one instantiation, fewer spills)
      c = segment_sum_deep<Q, FLAGGED>(a.sell_s, a.sbase[s], lane, len, Lw, a.contrib_prev, v, cself, &neg);
    else
      c = segment_sum_group<G, FLAGGED>(a.sell_s, a.sbase[s], col, role, len, Lw, a.contrib_prev, v, cself, &neg);
  }
  const bool newly = scan && neg;
  bool pend = false, lowout = false;
  if (valid && role == 0) {
    if (!aff && !newly) {
      copy_through(a, v);
    } else {
      finalize<FLAGGED, CLOSED>(a, v, c, pv, od, acc, pend, lowout, newly);
      ++acc.proc;
      acc.edges += deg;
    }
  }
  if (FLAGGED && a.pend_low && !(pull && a.lazy_lists)) warp_append(pend, lowout, v, od, a.pend_low, a.pend_high, a.red);
}

// One multi-chunk slice: 32 chunk partials; the warp that completes a
// vertex's last chunk combines and finalises it.
template <bool FLAGGED, bool CLOSED, int Q, int G = 1>
__device__ __forceinline__ void multi_slice(const SweepArgs& a, uint64_t s, unsigned lane, Acc& acc, bool pull,
                                            unsigned part = 0) {
  const unsigned col = G == 1 ? lane : part * (32u / G) + lane / G;
  const unsigned role = G == 1 ? 0u : lane % G;
  const uint64_t seg = s * 32 + col;
  uint32_t len = 0, v = 0xffffffffu;
  if (seg < a.n_mseg) {
    v = a.mseg_v[seg];
    len = a.mseg_len[seg];
    if (v < a.v_lo || v >= a.v_hi) {
      len = 0;  // another rank's vertex
    } else if (FLAGGED && !pull && !a.va[v]) {
      len = 0;
      if (seg == a.pbase[v] && role == 0) copy_through(a, v);  // first chunk's owner does the copy-through
    }
  }
  const uint32_t Lw = __reduce_max_sync(kFull, len);
  if (!Lw) return;
  double c;
  {  // (a pull sweep's chunk carries "any pending source" in the partial's sign bit)
    unsigned neg = 0;
    if (G == 1)
      c = segment_sum_deep<Q, FLAGGED>(a.sell_m, a.mbase[s], lane, len, Lw, a.contrib_prev, 0xffffffffu, 0.0, &neg);
    else
      c = segment_sum_group<G, FLAGGED>(a.sell_m, a.mbase[s], col, role, len, Lw, a.contrib_prev, 0xffffffffu, 0.0,
                                        &neg);
    if (FLAGGED && pull && neg) c = -c;
  }
  bool last = false;
  if (len && role == 0) {
    __stcg(a.partials + seg, c);
    __threadfence();
    const uint32_t nch = (a.indeg[v] + kAccumChunk - 1) / kAccumChunk;
    last = atomicAdd(a.mcount + v, 1u) == nch - 1;
    if (last) __threadfence();
  }
  unsigned lm = __ballot_sync(kFull, last);
  if (!lm) return;
  __syncwarp();
  double cfin = 0.0;
  bool negfin = false;
  while (lm) {
    const int L = __ffs(lm) - 1;
    lm &= lm - 1;
    const uint32_t w = __shfl_sync(kFull, v, L);
    // (chunk count from the in-degree: a derived layout's chunks of w need
    // not be followed by w + 1's, layout.cu build_incremental)
    const uint32_t pb = a.pbase[w], nch = (a.indeg[w] + kAccumChunk - 1) / kAccumChunk;
    double sum = 0.0;
    unsigned nb = 0;
    for (uint32_t g = 0; g < nch; g += 32) {
      const double x = (g + lane < nch) ? __ldcg(a.partials + pb + g + lane) : 0.0;
      nb |= (unsigned)__double2hiint(x);
      const uint32_t cnt = nch - g < 32 ? nch - g : 32;
      for (uint32_t j = 0; j < cnt; ++j) sum = __dadd_rn(sum, fabs(__shfl_sync(kFull, x, j)));
    }
    nb = __reduce_or_sync(kFull, nb);
    if ((int)lane == L) {
      cfin = sum;
      negfin = (nb >> 31) != 0;
      a.mcount[w] = 0;  // ready for the next sweep
    }
  }
  bool pend = false, lowout = false;
  uint32_t od = 0;
  if (last) {
    const bool aff = !FLAGGED || !pull || a.va[v];
    const bool newly = !aff && negfin;
    if (!aff && !newly) {
      copy_through(a, v);
    } else {
      od = a.outdeg[v];
      finalize<FLAGGED, CLOSED>(a, v, cfin, a.rank_prev[v], od, acc, pend, lowout, newly);
      ++acc.proc;
      acc.edges += a.indeg[v];
    }
  }
  if (FLAGGED && a.pend_low && !(pull && a.lazy_lists)) warp_append(pend, lowout, v, od, a.pend_low, a.pend_high, a.red);
}

template <bool FLAGGED, bool CLOSED, int QH, int G>
__device__ __forceinline__ void fused_body(const SweepArgs& a) {
  if (a.done && *a.done) return;
  Acc acc;
  const unsigned lane = lane_id();
  const bool pull = FLAGGED && pull_now(a);
  const uint64_t n_ms = a.ms_hi - a.ms_lo;
  const uint64_t hs_hi = a.ss_heavy < a.ss_hi ? a.ss_heavy : a.ss_hi;
  const uint64_t n_hs = hs_hi > a.ss_lo ? hs_hi - a.ss_lo : 0;
  const uint64_t n_heavy = (n_ms + n_hs) * G;  // items: (slice, part of G)
  const unsigned long long t0 = a.trace ? gtimer() : 0ull;
  unsigned long long nh = 0, nl = 0, first = ~0ull, th = 0;
  // heavy items are dealt round-robin to the (all resident) blocks -- item =
  // block + grid * k, k from a per-block counter -- so the long chains are
  // spread over the SMs instead of piling onto whichever warps grab first
  for (;;) {
    unsigned k = 0;
    if (lane == 0) k = atomicAdd(a.tick_sm + blockIdx.x, 1u);
    k = __shfl_sync(kFull, k, 0);
    const uint64_t t = (uint64_t)blockIdx.x + (uint64_t)gridDim.x * k;
    if (t >= n_heavy) break;
    ++nh;
    if (first == ~0ull) first = t;
    const uint64_t item = t / G;
    const unsigned part = (unsigned)(t % G);
    if (item < n_ms)
      multi_slice<FLAGGED, CLOSED, QH, G>(a, a.ms_lo + item, lane, acc, pull, part);
    else
      single_slice<FLAGGED, CLOSED, QH, G>(a, a.ss_lo + (item - n_ms), lane, acc, pull, part);
  }
  if (a.trace) th = gtimer();
  const uint64_t l_lo = a.ss_lo + n_hs;
  const uint64_t n_light = a.ss_hi > l_lo ? a.ss_hi - l_lo : 0;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&a.red->ticket_light, kLightGrab);
    t = __shfl_sync(kFull, t, 0);
    if (t >= n_light) break;
    const uint64_t e = t + kLightGrab < n_light ? t + kLightGrab : n_light;
    nl += e - t;
    for (uint64_t i = t; i < e; ++i) single_slice<FLAGGED, CLOSED, 2>(a, l_lo + i, lane, acc, pull);
  }
  if (a.trace && lane == 0) {
    const uint64_t w = ((uint64_t)blockIdx.x * kSweepThreads + threadIdx.x) / 32;
    if (w < kTraceWarps) {
      unsigned long long* r = g_trace + 6 * w;
      r[0] = smid();
      r[1] = t0;
      r[2] = gtimer();
      r[3] = nh | (nl << 32);
      r[4] = first;
      r[5] = th;
    }
  }
  if (a.npeers) __threadfence_system();  // peer stores visible before the team barrier
  block_reduce_commit(acc, a.red);
  // every warp of the block is past its last grab: the block's heavy-item
  // counter is zero again for the next sweep (no memset per sweep)
  if (threadIdx.x == 0) a.tick_sm[blockIdx.x] = 0;
}

// 16-deep heavy chains at 4 CTAs per SM.  (A 5-CTA, 8-deep variant was
// measured: it spills and is no faster on large graphs, where the split
// kernels win -- profiles/ab_probe.py.)
template <bool FLAGGED, bool CLOSED, int G>
__global__ void __launch_bounds__(kSweepThreads, 4) k_sweep_fused(SweepArgs a) {
  fused_body<FLAGGED, CLOSED, 4, G>(a);
}
template <bool FLAGGED, bool CLOSED, int H, int G>
__global__ void __launch_bounds__(kSweepThreads, 4) k_sweep_fused_c() {
  fused_body<FLAGGED, CLOSED, 4, G>(c_loop_args[H]);
}

// ---- pull expansion over the SELL in-lists ------------------------------------------
__device__ __forceinline__ void b_pull_single(const SweepArgs& a) {
  if (a.expand && *a.expand != kExpandPull) return;
  const unsigned lane = lane_id();
  for (;;) {  // slices grabbed dynamically, kSplitGrab at a time
    unsigned g = 0;
    if (lane == 0) g = atomicAdd(&a.red->ticket_pull, kSplitGrab);
    const uint64_t s0 = a.ss_lo + __shfl_sync(kFull, g, 0);
    if (s0 >= a.ss_hi) break;
    const uint64_t s1 = s0 + kSplitGrab < a.ss_hi ? s0 + kSplitGrab : a.ss_hi;
  for (uint64_t s = s0; s < s1; ++s) {
    const uint64_t vv = (uint64_t)a.M + s * 32 + lane;
    const bool need = vv < a.n && !a.va[vv];
    const uint32_t len = need ? a.indeg[vv] : 0u;
    if (!__any_sync(kFull, len != 0)) continue;
    if (segment_any_pending(a.sell_s, a.sbase[s], lane, len, a.np)) a.va[vv] = 1;
  }
  }
}
__global__ void __launch_bounds__(kThreads) k_pull_single(SweepArgs a) { b_pull_single(a); }
template <int H>
__global__ void __launch_bounds__(kThreads) k_pull_single_c() {
  b_pull_single(c_loop_args[H]);
}
__device__ __forceinline__ void b_pull_mseg(const SweepArgs& a) {
  if (a.expand && *a.expand != kExpandPull) return;
  const unsigned lane = lane_id();
  const uint64_t nw = (uint64_t)gridDim.x * kWarps;
  for (uint64_t s = a.ms_lo + ((uint64_t)blockIdx.x * kThreads + threadIdx.x) / 32; s < a.ms_hi; s += nw) {
    const uint64_t seg = s * 32 + lane;
    uint32_t len = 0, v = 0;
    if (seg < a.n_mseg) {
      v = a.mseg_v[seg];
      if (v >= a.v_lo && v < a.v_hi && !a.va[v]) len = a.mseg_len[seg];
    }
    if (!__any_sync(kFull, len != 0)) continue;
    if (segment_any_pending(a.sell_m, a.mbase[s], lane, len, a.np)) a.va[v] = 1;
  }
}
__global__ void __launch_bounds__(kThreads) k_pull_mseg(SweepArgs a) { b_pull_mseg(a); }
template <int H>
__global__ void __launch_bounds__(kThreads) k_pull_mseg_c() {
  b_pull_mseg(c_loop_args[H]);
}

// ---- stable degree partition (partition.cpp:7-61) ------------------------------------
constexpr int kTileItems = 4;
constexpr int kTile = kThreads * kTileItems;  // 1024 vertices per tile

__device__ __forceinline__ unsigned block_exclusive_scan(unsigned x, unsigned& total) {
  __shared__ unsigned s_w[kWarps];
  const unsigned lane = lane_id();
  const int w = threadIdx.x >> 5;
  unsigned inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, inc, o);
    if ((int)lane >= o) inc += y;
  }
  if (lane == 31) s_w[w] = inc;
  __syncwarp();  // reconverge the warp after the lane-divergent store
  __syncthreads();
  unsigned pre = 0;
  total = 0;
  for (int i = 0; i < kWarps; ++i) {
    if (i < w) pre += s_w[i];
    total += s_w[i];
  }
  __syncthreads();
  return pre + inc - x;
}

__global__ void __launch_bounds__(kThreads) k_part_count(const uint64_t* off, uint32_t n, uint32_t thr,
                                                        unsigned* tiles) {
  const uint64_t v0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kTileItems;
  unsigned s = 0;
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) s += (v0 + k < n) && (off[v0 + k + 1] - off[v0 + k] <= thr);
  unsigned total;
  block_exclusive_scan(s, total);
  if (threadIdx.x == 0) tiles[blockIdx.x] = total;
}

// Single-block exclusive scan of the tile counts.
__global__ void k_part_scan(unsigned* tiles, uint64_t ntiles, unsigned long long* total_out) {
  __shared__ unsigned long long s[1024];
  unsigned long long carry = 0;
  for (uint64_t base = 0; base < ntiles; base += blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const unsigned t = i < ntiles ? tiles[i] : 0u;
    s[threadIdx.x] = t;
    __syncthreads();
    for (unsigned o = 1; o < blockDim.x; o <<= 1) {
      const unsigned long long add = threadIdx.x >= o ? s[threadIdx.x - o] : 0ull;
      __syncthreads();
      s[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < ntiles) tiles[i] = (unsigned)(carry + s[threadIdx.x] - t);
    __syncthreads();
    carry += s[blockDim.x - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = carry;
}

__global__ void __launch_bounds__(kThreads) k_part_scatter(const uint64_t* off, uint32_t n, uint32_t thr,
                                                          const unsigned* tiles,
                                                          const unsigned long long* total, uint32_t* order) {
  const uint64_t v0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kTileItems;
  bool low[kTileItems];
  unsigned s = 0;
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) {
    low[k] = (v0 + k < n) && (off[v0 + k + 1] - off[v0 + k] <= thr);
    s += low[k];
  }
  unsigned tot;
  uint64_t lowpos = (uint64_t)tiles[blockIdx.x] + block_exclusive_scan(s, tot);
  const uint64_t lowCount = *total;
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) {
    const uint64_t v = v0 + k;
    if (v >= n) break;
    if (low[k]) {
      order[lowpos++] = (uint32_t)v;
    } else {
      order[lowCount + (v - lowpos)] = (uint32_t)v;  // high ids ascending after the low group
    }
  }
}

// ---- init / frontier kernels -------------------------------------------------
// init: the previous ranks in old-id order (gathered through perm), or null
// for uniform; r1 / c1 may be null when the first sweep writes every vertex.
__global__ void k_init_ranks(const uint32_t* outdeg, const uint32_t* perm, uint32_t n, const double* init,
                             double uniform, double* r0, double* r1, double* c0, double* c1) {
  // 4 vertices per thread per round, so 4 of the (random) old-order rank
  // gathers are in flight at once
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v0 < n; v0 += 4 * stride) {
    double r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t v = v0 + j * stride;
      r[j] = v < n ? (init ? init[perm[v]] : uniform) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t v = v0 + j * stride;
      if (v >= n) break;
      const double c = __ddiv_rn(r[j], (double)outdeg[v]);
      r0[v] = r[j];
      if (r1) r1[v] = r[j];
      c0[v] = c;
      if (c1) c1[v] = c;
    }
  }
}

// initialAffected (frontier.cpp:43-51): dels mark np[u] and va[v]; ins mark
// np[u] (ids mapped through `inv` into the flag space when given).
__global__ void k_init_affected(const uint32_t* inv, const uint32_t* ds, const uint32_t* dd, uint64_t nd,
                                const uint32_t* is, uint64_t ni, uint8_t* va, uint8_t* np) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nd + ni;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u;
    if (i < nd) {
      u = ds[i];
      const uint32_t v = dd[i];
      va[inv ? inv[v] : v] = 1;
    } else {
      u = is[i - nd];
    }
    np[inv ? inv[u] : u] = 1;
  }
}

// Pending flags -> expansion work lists (out-degree from `outdeg` when given,
// else from the CSR offsets).
__global__ void k_collect_pending(const uint32_t* outdeg, const uint64_t* off, uint32_t n, const uint8_t* np,
                                  uint32_t T, uint32_t* pl, uint2* ph, SweepRed* red) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint64_t v = base + threadIdx.x;
    bool pend = false, lowout = false;
    uint32_t od = 0;
    if (v < n && np[v]) {
      pend = true;
      od = outdeg ? outdeg[v] : (uint32_t)(off[v + 1] - off[v]);
      lowout = od <= T;
    }
    warp_append(pend, lowout, (uint32_t)v, od, pl, ph, red);
  }
}

// Push expansion (frontier.cpp:55-84) split by out-degree: thread per low
// pending vertex, warp per 1024-edge item of a high one.  Byte stores of 1
// are idempotent; the read-before-write keeps dense frontiers
// from turning into L2 write traffic.  (An 8-deep variant with more loads in
// flight per thread was measured slower: profiles/r01/README.md.)
__device__ __forceinline__ void expand_low_body(Rows rows, const uint32_t* list, uint64_t cnt, uint8_t* va) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = list[i];
    const uint32_t* r = rows.row(u);
    const uint64_t len = rows.len(u);
    // 8 targets, then their 8 flags, then the stores: 2 dependent round
    // trips per 8 edges instead of per edge (a byte store may alias the
    // target list, so the compiler cannot hoist the next loads by itself)
    for (uint64_t k = 0; k < len; k += 8) {
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = k + q < len ? __ldg(r + k + q) : 0xffffffffu;
      uint8_t f[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) f[q] = w[q] != 0xffffffffu ? va[w[q]] : 1;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (!f[q]) va[w[q]] = 1;
    }
  }
}
#ifndef DYNPR_EXPAND_DEPTH
#define DYNPR_EXPAND_DEPTH 4
#endif
// edges per lane per round of a 1024-edge item (8 measured no faster:
// profiles/r02/expand_batch_ab.txt)
constexpr int kExpandDepth = DYNPR_EXPAND_DEPTH;
__device__ __forceinline__ void expand_high_body(Rows rows, const uint2* items, uint64_t cnt, uint8_t* va) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  const unsigned lane = lane_id();
  for (uint64_t i = warp; i < cnt; i += nw) {
    const uint2 it = items[i];
    const uint32_t* r = rows.row(it.x);
    const uint64_t len = rows.len(it.x);
    const uint64_t b = (uint64_t)kExpandChunk * it.y;
    const uint64_t e = b + kExpandChunk < len ? b + kExpandChunk : len;
    for (uint64_t k = b + lane; k < e; k += 32 * kExpandDepth) {
      uint32_t w[kExpandDepth];
#pragma unroll
      for (int q = 0; q < kExpandDepth; ++q) w[q] = k + 32 * q < e ? __ldg(r + k + 32 * q) : 0xffffffffu;
      uint8_t f[kExpandDepth];
#pragma unroll
      for (int q = 0; q < kExpandDepth; ++q) f[q] = w[q] != 0xffffffffu ? va[w[q]] : 1;
#pragma unroll
      for (int q = 0; q < kExpandDepth; ++q)
        if (!f[q]) va[w[q]] = 1;
    }
  }
}
__global__ void k_expand_low(Rows rows, const uint32_t* list, uint32_t cnt, uint8_t* va, const unsigned* dcnt,
                             const int* gate) {
  if (gate && *gate != kExpandPush && *gate != kExpandPushCollect) return;
  expand_low_body(rows, list, dcnt ? dcnt[0] : cnt, va);
}
__global__ void k_expand_high(Rows rows, const uint2* items, uint32_t cnt, uint8_t* va, const unsigned* dcnt,
                              const int* gate) {
  if (gate && *gate != kExpandPush && *gate != kExpandPushCollect) return;
  expand_high_body(rows, items, dcnt ? dcnt[1] : cnt, va);
}
// device-loop variants: arguments from the constant-bank slot of half H
template <int H>
__global__ void k_expand_low_c(const unsigned* counts, const int* gate) {
  const SweepArgs* ap = &c_loop_args[H];
  if (gate && *gate != kExpandPush && *gate != kExpandPushCollect) return;
  expand_low_body(Rows{ap->begF, ap->outdeg, ap->tgtF}, ap->pend_low, counts[0], ap->va);
}
template <int H>
__global__ void k_expand_high_c(const unsigned* counts, const int* gate) {
  const SweepArgs* ap = &c_loop_args[H];
  if (gate && *gate != kExpandPush && *gate != kExpandPushCollect) return;
  expand_high_body(Rows{ap->begF, ap->outdeg, ap->tgtF}, ap->pend_high, counts[1], ap->va);
}

// ---- device-driven loop bookkeeping (engine.cpp:71-92) --------------------------------
// Per-iteration trace of the last device-loop solve (read with
// dynpr_debug_loop_trace): {globaltimer ns at the end of the iteration's
// sweep, gathered edges, processed vertices, pending out-edges | expansion
// direction << 62}.  One thread writes 32 bytes per iteration.
constexpr int kLoopTraceIters = 1024;
__device__ unsigned long long g_loop_trace[kLoopTraceIters * 4];

__global__ void k_loop_end(LoopCtl* c, SweepRed* red, cudaGraphConditionalHandle h, int set_cond,
                           cudaGraphConditionalHandle hpush, int has_push, cudaGraphConditionalHandle hempty,
                           int has_empty) {
  if (!c->done) {
    // a pull sweep of a lazy-list loop appended no pending lists
    const bool no_lists = c->lazy_lists && c->expand == kExpandPull;
    const SweepRed r = *red;
    *red = SweepRed{};  // zeroed for the next sweep (no memset node per iteration)
    const double delta = __longlong_as_double((long long)r.delta_bits);
    c->iterations += 1;
    c->affected += c->flagged ? r.processed : c->n;
    c->edges += r.edges;
    c->final_delta = delta;
    c->expand = kExpandNone;
    if (c->check && delta <= c->tol) {
      c->converged = 1;
      c->done = 1;
    } else if (c->iterations >= c->max_iter) {
      c->done = 1;  // the reference's trailing expansion cannot change the ranks
    } else if (c->frontier) {
      // direction-optimising expandAffected (same rule as the host loop)
      const unsigned long long pull_bound = c->m > r.edges ? c->m - r.edges : 0ull;
      const unsigned long long cost = c->push_cost > 0 ? (unsigned long long)c->push_cost : 1ull;
      c->expand = r.pend_edges * cost > pull_bound ? kExpandPull : (no_lists ? kExpandPushCollect : kExpandPush);
      c->pend_low = no_lists ? 0u : r.pend_low;
      c->pend_high = no_lists ? 0u : r.pend_high;
      // nothing pending: no expansion; with pruning the affected set may now
      // be empty (checked by the IF node `hempty`)
      if (r.pend_edges == 0) c->expand = kExpandNone;
      c->check_empty = has_empty && c->check && r.pend_edges == 0 ? 1 : 0;
    }
    if (c->iterations <= kLoopTraceIters) {
      unsigned long long* t = g_loop_trace + 4 * (c->iterations - 1);
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      t[0] = now;
      t[1] = r.edges;
      t[2] = r.processed;
      t[3] = r.pend_edges | ((unsigned long long)c->expand << 62);
    }
  }
  if (set_cond) cudaGraphSetConditional(h, c->done ? 0u : 1u);
  if (has_push) {
    const bool push = !c->done && (c->expand == kExpandPush || c->expand == kExpandPushCollect);
    c->pushes += push ? 1u : 0u;
    cudaGraphSetConditional(hpush, push ? 1u : 0u);
  }
  if (has_empty) {
    const bool chk = !c->done && c->check_empty;
    c->empty_checks += chk ? 1u : 0u;
    cudaGraphSetConditional(hempty, chk ? 1u : 0u);
  }
}

// Any vertex still affected (a delta-V byte set)?  16-byte loads; a block
// stops once another found one.
template <int H>
__global__ void k_any_affected(LoopCtl* c) {
  const uint8_t* va = c_loop_args[H].va;  // (the solve's flags, from its argument slot)
  const uint64_t n = c_loop_args[H].n;
  const uint64_t nv = n / 16;
  const uint4* v4 = reinterpret_cast<const uint4*>(va);
  bool found = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv && !found;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 x = v4[i];
    found = (x.x | x.y | x.z | x.w) != 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x < n % 16) found = found || va[nv * 16 + threadIdx.x] != 0;
  if (__syncthreads_or(found) && threadIdx.x == 0) atomicOr(&c->kept, 1u);
}
__global__ void k_empty_finish(LoopCtl* c, cudaGraphConditionalHandle h, int set_cond) {
  if (!c->done && !c->kept) {
    c->iterations += 1;  // all copied through: delta 0 (engine.cpp:79-91)
    c->final_delta = 0.0;
    c->converged = 0.0 <= c->tol ? 1 : 0;
    c->done = 1;
    c->skipped = 1;
    if (c->iterations <= kLoopTraceIters) {
      unsigned long long* t = g_loop_trace + 4 * (c->iterations - 1);
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      t[0] = now;
      t[1] = t[2] = t[3] = 0ull;
    }
  }
  c->kept = 0u;
  c->check_empty = 0;
  if (set_cond) cudaGraphSetConditional(h, c->done ? 0u : 1u);
}

// A push decided after a pull sweep of a lazy-list loop: the pending lists
// were not appended (SweepArgs::lazy_lists); the sweep's pending vertices
// are exactly the negative entries of the contributions it wrote.  The
// counts go straight to the loop state the push kernels read.
__device__ __forceinline__ void collect_signs_body(const SweepArgs& a, unsigned* cnt_low, unsigned* cnt_high) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < a.n; base += stride) {
    const uint64_t v = base + threadIdx.x;
    bool pend = false, lowout = false;
    uint32_t od = 0;
    if (v < a.n && v >= a.v_lo && v < a.v_hi && __double2hiint(a.contrib_cur[v]) < 0) {
      pend = true;
      od = a.outdeg[v];
      lowout = od <= a.T;
    }
    warp_append_to(pend, lowout, (uint32_t)v, od, a.pend_low, a.pend_high, cnt_low, cnt_high);
  }
}
template <int H>
__global__ void k_collect_signs_c(LoopCtl* c) {
  if (c->expand != kExpandPushCollect) return;
  collect_signs_body(c_loop_args[H], &c->pend_low, &c->pend_high);
}
__global__ void k_collect_signs(SweepArgs a, SweepRed* out) { collect_signs_body(a, &out->pend_low, &out->pend_high); }

// ---- markReachable (frontier.cpp:86-121): level-synchronous BFS -------------------
// Claims a flag byte exactly once (the containing 32-bit word is or-ed, the
// byte's old value decides the winner); newly claimed vertices are appended
// to the next frontier with warp-aggregated atomics.
__device__ __forceinline__ bool claim_byte(uint8_t* flags, uint32_t w) {
  if (flags[w]) return false;
  unsigned* word = reinterpret_cast<unsigned*>(flags + (w & ~3u));
  const unsigned sh = (w & 3u) * 8u;
  const unsigned old = atomicOr(word, 1u << sh);
  return ((old >> sh) & 0xffu) == 0u;
}

// Frontier entries are (vertex, 1024-edge chunk) items, so a hub reached
// at some level is scanned by ceil(outdeg / 1024) warps instead of one (a
// warp per frontier vertex left a single warp walking a 4e5-edge RMAT-24 hub
// while the rest of the GPU idled).  Newly claimed vertices append their
// items with a warp-aggregated atomic.
constexpr uint32_t kBfsChunk = 1024;
__device__ __forceinline__ void warp_push_items(bool take, uint32_t w, uint32_t items, uint2* out, unsigned* cnt) {
  const unsigned lane = lane_id();
  unsigned incl = take ? items : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if ((int)lane >= o) incl += y;
  }
  const unsigned total = __shfl_sync(kFull, incl, 31);
  if (!total) return;
  unsigned base = 0;
  if (lane == 0) base = atomicAdd(cnt, total);
  base = __shfl_sync(kFull, base, 0);
  if (take)
    for (unsigned j = 0, b = base + incl - items; j < items; ++j) out[b + j] = make_uint2(w, j);
}

__device__ __forceinline__ uint32_t bfs_items(Rows rows, uint32_t w) {
  const uint64_t d = rows.len(w);
  return d ? (uint32_t)((d + kBfsChunk - 1) / kBfsChunk) : 0u;
}

__global__ void k_bfs_seed(Rows rows, const uint32_t* inv, const uint32_t* seeds, uint64_t ns,
                           uint8_t* flags, uint2* out, unsigned* cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < ns; b += stride) {
    const uint64_t i = b + threadIdx.x;
    uint32_t v = 0, items = 0;
    bool take = false;
    if (i < ns) {
      v = inv ? inv[seeds[i]] : seeds[i];
      take = claim_byte(flags, v);
      if (take) items = bfs_items(rows, v);
    }
    warp_push_items(take && items, v, items, out, cnt);
  }
}

// warp per frontier item: lanes stride over the chunk's out-edges
__global__ void k_bfs_level(Rows rows, const uint2* fr, uint32_t nf, uint8_t* flags, uint2* out, unsigned* cnt) {
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < nf; i += nw) {
    const uint2 it = fr[i];
    const uint32_t* r = rows.row(it.x);
    const uint64_t len = rows.len(it.x);
    const uint64_t b = (uint64_t)kBfsChunk * it.y;
    const uint64_t e = b + kBfsChunk < len ? b + kBfsChunk : len;
    for (uint64_t k0 = b; k0 < e; k0 += 32) {
      const uint64_t k = k0 + lane_id();
      uint32_t w = 0, items = 0;
      bool take = false;
      if (k < e) {
        w = r[k];
        take = claim_byte(flags, w);
        if (take) items = bfs_items(rows, w);
      }
      warp_push_items(take && items, w, items, out, cnt);
    }
  }
}

// ---- team graph fingerprint ----------------------------------------------------
// Order-free sum of position-salted SplitMix64 finalisers of 32-bit words:
// equal arrays give equal sums on every rank, a differing word changes the
// sum (up to 2^-64 collisions).
__device__ __forceinline__ uint64_t fp_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void k_fingerprint(const uint32_t* w, uint64_t count, uint64_t salt, unsigned long long* out) {
  uint64_t h = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    h += fp_mix((i + salt) * 0x9e3779b97f4a7c15ull ^ w[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(kFull, h, o);
  if (lane_id() == 0 && h) atomicAdd(out, (unsigned long long)h);
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
  __syncwarp();  // reconverge the warp after the lane-divergent store
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

// Persistent grid: resident blocks per SM x SMs (queried once per kernel).
// Lanes per heavy segment for a fused sweep over n_slices slices (see
// kGroupSlicesPerWarp).
static int heavy_lanes(dynpr_context* ctx, uint64_t n_slices) {
  const char* e = std::getenv("DYNPR_HEAVY_LANES");
  const int forced = e ? std::atoi(e) : 0;
  if (forced == 1 || forced == 2) return forced;
  return n_slices <= kGroupSlicesPerWarp * (uint64_t)ctx->num_sms * 32 ? 2 : 1;
}

template <class K>
unsigned persistent_grid(dynpr_context* ctx, K kernel, uint64_t work_blocks) {
  constexpr int kSlots = 128;  // > the 36 persistent kernel instantiations
  static const void* keys[kSlots] = {};
  static int vals[kSlots] = {};
  static std::mutex lock;  // contexts on several host threads (LocalTeam, concurrent solves)
  std::lock_guard<std::mutex> guard(lock);
  int per_sm = -1;
  for (int i = 0; i < kSlots && keys[i]; ++i)
    if (keys[i] == (const void*)kernel) per_sm = vals[i];
  if (per_sm < 0) {
    int b = 0;
    // these kernels use little shared memory: give the SM's unified
    // L1/shared SRAM to L1 (it holds the hot contributions)
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaGetLastError();
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b < 1) {
      cudaGetLastError();
      b = 1;
    }
    per_sm = b;
    for (int i = 0; i < kSlots; ++i)
      if (!keys[i]) {
        keys[i] = (const void*)kernel;
        vals[i] = b;
        break;
      }
  }
  const uint64_t cap = (uint64_t)per_sm * ctx->num_sms;
  return (unsigned)(work_blocks < 1 ? 1 : (work_blocks < cap ? work_blocks : cap));
}

}  // namespace

// ---------------------------------------------------------------------------
Schedule build_partition(dynpr_context* ctx, const dynpr_graph* g, uint32_t thr, uint32_t* order) {
  Schedule s;
  s.threshold = thr;
  const uint32_t n = g->n;
  if (n == 0) return s;
  cudaStream_t st = ctx->stream;
  const uint64_t ntiles = ((uint64_t)n + kTile - 1) / kTile;
  unsigned* tiles = ctx->tile_counts.as<unsigned>(ntiles);
  auto* total = ctx->scratch64a.as<unsigned long long>(1);
  k_part_count<<<(unsigned)ntiles, kThreads, 0, st>>>(g->off, n, thr, tiles);
  check_launch();
  k_part_scan<<<1, 1024, 0, st>>>(tiles, ntiles, total);
  check_launch();
  k_part_scatter<<<(unsigned)ntiles, kThreads, 0, st>>>(g->off, n, thr, tiles, total, order);
  check_launch();
  count_launch(ctx, 3);
  unsigned long long h;
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, total, 8, cudaMemcpyDeviceToHost, st));
  sync(ctx);
  std::memcpy(&h, ctx->pinned, 8);
  s.n_low = (uint32_t)h;
  s.n_high = n - s.n_low;
  return s;
}

SweepArgs layout_args(const Layout* L, double* partials) {
  SweepArgs a{};
  a.n = L->n;
  a.M = L->M;
  static const bool no_self_fast = std::getenv("DYNPR_NO_SELF_FAST") != nullptr;  // A/B only
  a.loops = (L->loops && !no_self_fast) ? 1 : 0;
  a.T = L->T;
  a.indeg = L->indeg;
  a.outdeg = L->outdeg;
  a.n_sslices = L->n_sslices;
  a.sbase = L->sbase;
  a.sell_s = L->sell_s;
  a.n_mseg = L->n_mseg;
  a.n_mslices = L->n_mslices;
  a.mbase = L->mbase;
  a.mseg_v = L->mseg_v;
  a.mseg_len = L->mseg_len;
  a.pbase = L->pbase;
  a.sell_m = L->sell_m;
  a.partials = partials;
  static const int trace = std::getenv("DYNPR_TRACE") != nullptr;
  a.trace = trace;
  a.mcount = L->mcount;
  a.ss_heavy = L->n_hslices;
  a.v_lo = 0;
  a.v_hi = L->n;
  a.ss_lo = 0;
  a.ss_hi = L->n_sslices;
  a.ms_lo = 0;
  a.ms_hi = L->n_mslices;
  return a;
}

// in-degree i widened to 64 bits, 0 past the end
struct IndegAt {
  const uint32_t* indeg;
  uint32_t n;
  __device__ __forceinline__ unsigned long long operator()(uint64_t i) const {
    return i < n ? (unsigned long long)indeg[i] : 0ull;
  }
};
// cut[r] (0 < r < world): after the first vertex v whose inclusive in-degree
// prefix reaches r/world of the edges, rounded up to a whole single-region
// slice; n if none does.
__global__ void k_plan_cuts(const unsigned long long* prefix, uint32_t n, uint32_t M, uint64_t m, int world,
                            uint32_t* cut) {
  const int r = (int)threadIdx.x + 1;
  if (r >= world) return;
  const unsigned long long goal = (unsigned long long)m * (unsigned long long)r;
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (prefix[mid] * (unsigned long long)world >= goal) hi = mid; else lo = mid + 1;
  }
  uint32_t c = n;
  if (lo < n) {
    c = lo + 1;
    if (c > M) c = M + ((c - M + 31) / 32) * 32;
    if (c > n) c = n;
  }
  cut[r] = c;
}

std::vector<RankRange> plan_ranges(dynpr_context* ctx, Layout* L, int world) {
  if (L->plan_world == world) return L->plan;
  const uint32_t n = L->n, M = L->M;
  // boundaries at equal shares of the in-edges (each owned edge is one
  // gather): an in-degree prefix scan and one binary search per boundary on
  // the device; only the world + 1 cuts and the multi-vertex chunk bases
  // come back
  std::vector<uint32_t> cut(world + 1, 0), pbase((size_t)M + 1);
  cut[world] = n;
  if (world > 1 && n) {
    auto* prefix = ctx->plan_prefix.as<unsigned long long>((uint64_t)n + 72);
    auto* dcut = reinterpret_cast<uint32_t*>(prefix + n + 1);
    if (world > 128) throw Error(DYNPR_INVALID_ARGUMENT, "team larger than 128 ranks");
    // 64-bit accumulation (m may exceed 2^32); the exclusive prefix over
    // n + 1 entries shifted by one is the inclusive prefix
    prims::scan_exclusive<unsigned long long>(ctx, IndegAt{L->indeg, n}, prefix, (uint64_t)n + 1, ctx->stream);
    k_plan_cuts<<<1, 128, 0, ctx->stream>>>(prefix + 1, n, M, L->m, world, dcut);
    check_launch();
    DYNPR_CK(cudaMemcpyAsync(cut.data() + 1, dcut + 1, (size_t)(world - 1) * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
  }
  DYNPR_CK(cudaMemcpyAsync(pbase.data(), L->pbase, ((size_t)M + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  DYNPR_CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 1; i <= world; ++i)
    if (cut[i] < cut[i - 1]) cut[i] = cut[i - 1];
  std::vector<RankRange> plan(world);
  for (int i = 0; i < world; ++i) {
    RankRange& p = plan[i];
    p.v_lo = cut[i];
    p.v_hi = cut[i + 1];
    p.ss_lo = p.v_lo <= M ? 0 : (p.v_lo - M) / 32;
    p.ss_hi = p.v_hi <= M ? 0 : (p.v_hi - M + 31) / 32;
    if (p.ss_hi < p.ss_lo) p.ss_hi = p.ss_lo;
    const uint32_t mlo = p.v_lo < M ? p.v_lo : M, mhi = p.v_hi < M ? p.v_hi : M;
    p.ms_lo = pbase[mlo] / 32;
    p.ms_hi = (pbase[mhi] + 31) / 32;
    if (mhi <= mlo) p.ms_lo = p.ms_hi = 0;
  }
  L->plan = plan;
  L->plan_world = world;
  return plan;
}

// Persistent grid for the sweep kernels (resident CTAs per SM x SMs).
template <class K>
unsigned sweep_grid(dynpr_context* ctx, K kernel, uint64_t slices, size_t smem) {
  (void)smem;
  return persistent_grid(ctx, kernel, (slices + kSweepWarps - 1) / kSweepWarps);
}

// Fork / join of the context's aux stream (capturable: the aux stream joins
// a capture through the fork event and rejoins through the join event).
static cudaStream_t fork_aux(dynpr_context* ctx) {
  if (!ctx->aux) {
    // highest priority: the multi-chunk slices hold the longest lane chains,
    // so their blocks go first (captured into the loop graph's kernel node)
    int lo = 0, hi = 0;
    DYNPR_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DYNPR_CK(cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, hi));
    DYNPR_CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    DYNPR_CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  DYNPR_CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
  DYNPR_CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
  return ctx->aux;
}
static void join_aux(dynpr_context* ctx) {
  DYNPR_CK(cudaEventRecord(ctx->ev_join, ctx->aux));
  DYNPR_CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
}

// In the device-loop graph the two concurrently launched split kernels share
// every SM: their persistent grids are capped at kMsegPerSm / kSinglePerSm
// blocks per SM
// (both fit one SM's registers), instead of the first launched kernel
// filling the GPU at full occupancy and the other running in its tail.
// The multi-chunk slices are request-bound and need few warps, the single
// slices are latency-bound and take the rest (profiles/r02/grid_ab_*.txt:
// RMAT-24 Static 60.4 -> 56.0 ms, RMAT-26 259.5 -> 256.2, Kronecker-25
// 121.4 -> 118.5).  DYNPR_MSEG_BPS / DYNPR_SINGLE_BPS override (0: no cap).
constexpr unsigned kMsegPerSm = 2, kSinglePerSm = 3;
static void cap_blocks(dynpr_context* ctx, const char* var, unsigned def_bps, unsigned& grid) {
  const char* e = std::getenv(var);
  const unsigned bps = e ? (unsigned)std::strtoul(e, nullptr, 10) : def_bps;
  const unsigned cap = bps * (unsigned)ctx->num_sms;
  if (grid && cap && grid > cap) grid = cap;
}
static void cap_split_grids(dynpr_context* ctx, unsigned& g_mseg, unsigned& g_single) {
  if (!g_mseg || !g_single) return;  // one kernel alone: full occupancy
  cap_blocks(ctx, "DYNPR_MSEG_BPS", kMsegPerSm, g_mseg);
  cap_blocks(ctx, "DYNPR_SINGLE_BPS", kSinglePerSm, g_single);
}

void launch_sweep(dynpr_context* ctx, const SweepArgs& a, bool flagged, bool closed) {
  cudaStream_t st = ctx->stream;
  const uint64_t mv = (a.M < a.v_hi ? a.M : a.v_hi) > a.v_lo ? (a.M < a.v_hi ? a.M : a.v_hi) - a.v_lo : 0;
  const unsigned g_mfinal = grid_for(mv, kThreads);
  const uint64_t n_ms = a.ms_hi - a.ms_lo, n_ss = a.ss_hi - a.ss_lo;
  const size_t smem = 0;
  unsigned launched = 0;
#define DYNPR_SWEEP(F, C)                                                                           \
  do {                                                                                              \
    const bool par = n_ms && n_ss;  /* multi chunks on aux, concurrent with the single slices */   \
    /* (uncapped grids here: the grid caps of the loop graph made the  */                          \
    /* host-driven sweep slower, 0.95 -> 1.16 ms on RMAT-24)            */                          \
    if (n_ms) {                                                                                     \
      cudaStream_t ms = par ? fork_aux(ctx) : st;                                                   \
      k_sweep_mseg<F><<<sweep_grid(ctx, k_sweep_mseg<F>, n_ms, smem), kSweepThreads, smem,          \
                        ms>>>(a);                                                                   \
      ++launched;                                                                                   \
    }                                                                                               \
    if (mv) { /* the ordered combine follows the chunks on the same stream */                     \
      k_sweep_mfinal<F, C><<<g_mfinal, kThreads, 0, par ? ctx->aux : st>>>(a);                     \
      ++launched;                                                                                   \
    }                                                                                               \
    if (n_ss) {                                                                                     \
      k_sweep_single<F, C><<<sweep_grid(ctx, k_sweep_single<F, C>, n_ss, smem), kSweepThreads,      \
                             smem, st>>>(a);                                                        \
      ++launched;                                                                                   \
    }                                                                                               \
    if (par) join_aux(ctx);                                                                         \
  } while (0)
  // Latency-bound graphs (few slices per resident warp) take the fused
  // kernel; throughput-bound ones the split kernels (measured A/B,
  // profiles/ab_probe.py: fused wins 1.2-1.5x on RMAT-18..22, split wins
  // ~3% on RMAT-24).  DYNPR_SWEEP=split|fused overrides.
  const char* mode = std::getenv("DYNPR_SWEEP");
  const std::string m = mode ? mode : "";
  const uint64_t resident_warps = (uint64_t)ctx->num_sms * 32;
  const bool big = (n_ms + n_ss) > kSplitSlicesPerWarp * resident_warps;
  const bool split = m == "split" || (m != "fused" && big);
  if (!split) {
    // one persistent launch; the work counters live in the (zeroed) record
    SweepArgs af = a;
    af.tick_sm = ctx->tick.as<uint32_t>(kMaxBlocks);
    DYNPR_CK(cudaMemsetAsync(af.tick_sm, 0, kMaxBlocks * sizeof(uint32_t), st));
    const uint64_t wb = (n_ms + n_ss + kSweepWarps - 1) / kSweepWarps;
    const bool grouped = heavy_lanes(ctx, n_ms + n_ss) == 2;
#define DYNPR_FUSED(F, C)                                                                      \
  do {                                                                                         \
    if (grouped)                                                                               \
      k_sweep_fused<F, C, 2><<<persistent_grid(ctx, k_sweep_fused<F, C, 2>, wb), kSweepThreads, 0, st>>>(af); \
    else                                                                                       \
      k_sweep_fused<F, C, 1><<<persistent_grid(ctx, k_sweep_fused<F, C, 1>, wb), kSweepThreads, 0, st>>>(af); \
  } while (0)
    if (n_ms + n_ss) {
      if (flagged) {
        if (closed) DYNPR_FUSED(true, true); else DYNPR_FUSED(true, false);
      } else {
        if (closed) DYNPR_FUSED(false, true); else DYNPR_FUSED(false, false);
      }
      ++launched;
    }
#undef DYNPR_FUSED
  } else if (flagged) {
    if (closed) DYNPR_SWEEP(true, true); else DYNPR_SWEEP(true, false);
  } else {
    if (closed) DYNPR_SWEEP(false, true); else DYNPR_SWEEP(false, false);
  }
#undef DYNPR_SWEEP
  check_launch();
  count_launch(ctx, launched);
}


// ---- indirect launches for the cached device-loop graph ------------------------------
// Same kernel choice as launch_sweep; every grid is fixed here (before any
// capture), so a plan plus the device argument buffer fully describe the
// launches and equal plans can share one instantiated graph.
template <class K>
static unsigned pgrid(dynpr_context* ctx, K k, uint64_t work_blocks) {
  return persistent_grid(ctx, k, work_blocks);
}

SweepPlan plan_sweep(dynpr_context* ctx, const SweepArgs& a, bool flagged, bool closed) {
  SweepPlan p{};
  p.flagged = flagged;
  p.closed = closed;
  const uint64_t mv = (a.M < a.v_hi ? a.M : a.v_hi) > a.v_lo ? (a.M < a.v_hi ? a.M : a.v_hi) - a.v_lo : 0;
  const uint64_t n_ms = a.ms_hi - a.ms_lo, n_ss = a.ss_hi - a.ss_lo;
  const char* mode = std::getenv("DYNPR_SWEEP");
  const std::string m = mode ? mode : "";
  const uint64_t resident_warps = (uint64_t)ctx->num_sms * 32;
  const bool big = (n_ms + n_ss) > kSplitSlicesPerWarp * resident_warps;
  p.split = m == "split" || (m != "fused" && big);
  p.grouped = !p.split && heavy_lanes(ctx, n_ms + n_ss) == 2;
  const uint64_t wms = (n_ms + kSweepWarps - 1) / kSweepWarps, wss = (n_ss + kSweepWarps - 1) / kSweepWarps;
#define DYNPR_PLAN(F, C)                                                                 \
  do {                                                                                   \
    if (!p.split) {                                                                      \
      if (n_ms + n_ss)                                                                   \
        p.g_fused = p.grouped ? pgrid(ctx, k_sweep_fused_c<F, C, 0, 2>, (n_ms + n_ss + kSweepWarps - 1) / kSweepWarps) \
                              : pgrid(ctx, k_sweep_fused_c<F, C, 0, 1>, (n_ms + n_ss + kSweepWarps - 1) / kSweepWarps); \
    } else {                                                                             \
      if (n_ms) p.g_mseg = pgrid(ctx, k_sweep_mseg_c<F, 0>, wms);                        \
      if (n_ss) p.g_single = pgrid(ctx, k_sweep_single_c<F, C, 0>, wss);                 \
      cap_split_grids(ctx, p.g_mseg, p.g_single);                                        \
      if (mv) p.g_mfinal = grid_for(mv, kThreads);                                       \
    }                                                                                    \
  } while (0)
  if (flagged) {
    if (closed) DYNPR_PLAN(true, true); else DYNPR_PLAN(true, false);
  } else {
    if (closed) DYNPR_PLAN(false, true); else DYNPR_PLAN(false, false);
  }
#undef DYNPR_PLAN
  p.pull_fused = a.pull_fused;
  if (n_ms) p.g_pull_m = pgrid(ctx, k_pull_mseg_c<0>, (n_ms + kWarps - 1) / kWarps);
  if (n_ss) p.g_pull_s = pgrid(ctx, k_pull_single_c<0>, (n_ss + kWarps - 1) / kWarps);
  return p;
}

template <int H>
static void launch_sweep_c(dynpr_context* ctx, const SweepPlan& p, uint32_t* tick) {
  cudaStream_t st = ctx->stream;
  unsigned launched = 0;
#define DYNPR_IND(F, C)                                                                          \
  do {                                                                                           \
    if (!p.split) {                                                                              \
      if (p.g_fused) {                                                                           \
        (void)tick; /* zero between sweeps: each block resets its own counter */                \
        if (p.grouped) k_sweep_fused_c<F, C, H, 2><<<p.g_fused, kSweepThreads, 0, st>>>();       \
        else k_sweep_fused_c<F, C, H, 1><<<p.g_fused, kSweepThreads, 0, st>>>();                 \
        ++launched;                                                                              \
      }                                                                                          \
    } else {                                                                                     \
      const bool par = p.g_mseg && p.g_single;                                                  \
      /* in the captured graph: the chunks + combine on the origin stream, the */                 \
      /* single slices on the aux branch (forked after the chunk launch)       */                 \
      cudaStream_t ss = par ? fork_aux(ctx) : st;                                                \
      if (p.g_mseg) {                                                                            \
        k_sweep_mseg_c<F, H><<<p.g_mseg, kSweepThreads, 0, st>>>();                              \
        ++launched;                                                                              \
      }                                                                                          \
      if (p.g_mfinal) {                                                                          \
        k_sweep_mfinal_c<F, C, H><<<p.g_mfinal, kThreads, 0, st>>>();                            \
        ++launched;                                                                              \
      }                                                                                          \
      if (p.g_single) { k_sweep_single_c<F, C, H><<<p.g_single, kSweepThreads, 0, ss>>>(); ++launched; } \
      if (par) join_aux(ctx);                                                                    \
    }                                                                                            \
  } while (0)
  if (p.flagged) {
    if (p.closed) DYNPR_IND(true, true); else DYNPR_IND(true, false);
  } else {
    if (p.closed) DYNPR_IND(false, true); else DYNPR_IND(false, false);
  }
#undef DYNPR_IND
  check_launch();
  count_launch(ctx, launched);
}
void launch_sweep_ind(dynpr_context* ctx, const SweepPlan& p, int half, uint32_t* tick) {
  if (half) launch_sweep_c<1>(ctx, p, tick); else launch_sweep_c<0>(ctx, p, tick);
}

void launch_pull_ind(dynpr_context* ctx, const SweepPlan& p, int half) {
  cudaStream_t st = ctx->stream;
  unsigned launched = 0;
  if (p.g_pull_m) {
    if (half) k_pull_mseg_c<1><<<p.g_pull_m, kThreads, 0, st>>>(); else k_pull_mseg_c<0><<<p.g_pull_m, kThreads, 0, st>>>();
    ++launched;
  }
  if (p.g_pull_s) {
    if (half) k_pull_single_c<1><<<p.g_pull_s, kThreads, 0, st>>>(); else k_pull_single_c<0><<<p.g_pull_s, kThreads, 0, st>>>();
    ++launched;
  }
  check_launch();
  count_launch(ctx, launched);
}

void launch_expand_ind(dynpr_context* ctx, int half, LoopCtl* dc, cudaStream_t stream) {
  const unsigned g = (unsigned)ctx->num_sms * 16;
  const unsigned* counts = &dc->pend_low;
  const int* gate = &dc->expand;
  // (returns at once unless a lazy-list loop pushes after a pull sweep)
  if (half) k_collect_signs_c<1><<<g, kThreads, 0, stream>>>(dc);
  else k_collect_signs_c<0><<<g, kThreads, 0, stream>>>(dc);
  count_launch(ctx);
  if (half) {
    k_expand_low_c<1><<<g, kThreads, 0, stream>>>(counts, gate);
    k_expand_high_c<1><<<g, kThreads, 0, stream>>>(counts, gate);
  } else {
    k_expand_low_c<0><<<g, kThreads, 0, stream>>>(counts, gate);
    k_expand_high_c<0><<<g, kThreads, 0, stream>>>(counts, gate);
  }
  check_launch();
  count_launch(ctx, 2);
}

bool sweep_is_split(dynpr_context* ctx, const Layout* L) {
  const char* mode = std::getenv("DYNPR_SWEEP");
  const std::string m = mode ? mode : "";
  const uint64_t resident_warps = (uint64_t)ctx->num_sms * 32;
  const bool big = (L->n_mslices + L->n_sslices) > kSplitSlicesPerWarp * resident_warps;
  return m == "split" || (m != "fused" && big);
}

bool is_priority_sweep_kernel(const void* f) {
  return f == (const void*)k_sweep_mseg_c<false, 0> || f == (const void*)k_sweep_mseg_c<false, 1> ||
         f == (const void*)k_sweep_mseg_c<true, 0> || f == (const void*)k_sweep_mseg_c<true, 1>;
}

void upload_loop_args(dynpr_context* ctx, const SweepArgs* host_pinned_half2) {
  DYNPR_CK(cudaMemcpyToSymbolAsync(c_loop_args, host_pinned_half2, 2 * sizeof(SweepArgs), 0, cudaMemcpyHostToDevice,
                                   ctx->stream));
}

uint32_t* sweep_tick(dynpr_context* ctx) {
  if (!ctx->tick.p) {  // zeroed once; the fused sweep leaves it zero
    uint32_t* t = ctx->tick.as<uint32_t>(kMaxBlocks);
    DYNPR_CK(cudaMemsetAsync(t, 0, ctx->tick.cap, ctx->stream));
  }
  return ctx->tick.as<uint32_t>(kMaxBlocks);
}

void prepare_sweep_launch(dynpr_context* ctx) {
  sweep_tick(ctx);
  persistent_grid(ctx, k_sweep_fused<false, false, 1>, 1);
  persistent_grid(ctx, k_sweep_fused<true, false, 1>, 1);
  persistent_grid(ctx, k_sweep_fused<false, true, 1>, 1);
  persistent_grid(ctx, k_sweep_fused<true, true, 1>, 1);
  persistent_grid(ctx, k_sweep_fused<false, false, 2>, 1);
  persistent_grid(ctx, k_sweep_fused<true, false, 2>, 1);
  persistent_grid(ctx, k_sweep_fused<false, true, 2>, 1);
  persistent_grid(ctx, k_sweep_fused<true, true, 2>, 1);
  persistent_grid(ctx, k_sweep_mseg<false>, 1);
  persistent_grid(ctx, k_sweep_mseg<true>, 1);
  persistent_grid(ctx, k_sweep_single<false, false>, 1);
  persistent_grid(ctx, k_sweep_single<true, false>, 1);
  persistent_grid(ctx, k_sweep_single<false, true>, 1);
  persistent_grid(ctx, k_sweep_single<true, true>, 1);
  persistent_grid(ctx, k_pull_mseg, 1);
  persistent_grid(ctx, k_pull_single, 1);
}

void launch_pull_expand(dynpr_context* ctx, const SweepArgs& a) {
  cudaStream_t st = ctx->stream;
  unsigned launched = 0;
  const uint64_t n_ms = a.ms_hi - a.ms_lo, n_ss = a.ss_hi - a.ss_lo;
  if (n_ms) {
    k_pull_mseg<<<persistent_grid(ctx, k_pull_mseg, (n_ms + kWarps - 1) / kWarps), kThreads, 0, st>>>(a);
    ++launched;
  }
  if (n_ss) {
    k_pull_single<<<persistent_grid(ctx, k_pull_single, (n_ss + kWarps - 1) / kWarps), kThreads, 0, st>>>(a);
    ++launched;
  }
  check_launch();
  count_launch(ctx, launched);
}

void launch_init_ranks(dynpr_context* ctx, const Layout* L, const double* init_old, double uniform, double* r0,
                       double* r1, double* c0, double* c1) {
  if (!L->n) return;
  k_init_ranks<<<grid_for(L->n, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(
      L->outdeg, L->perm, L->n, init_old, uniform, r0, r1, c0, c1);
  check_launch();
  count_launch(ctx);
}

void launch_init_affected(dynpr_context* ctx, const uint32_t* inv, const uint32_t* ds, const uint32_t* dd,
                          uint64_t nd, const uint32_t* is, uint64_t ni, uint8_t* va, uint8_t* np) {
  if (nd + ni == 0) return;
  k_init_affected<<<grid_for(nd + ni, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(inv, ds, dd, nd,
                                                                                               is, ni, va, np);
  check_launch();
  count_launch(ctx);
}

void launch_collect_pending(dynpr_context* ctx, const uint32_t* outdeg, const uint64_t* off, uint32_t n,
                            const uint8_t* np, uint32_t T, uint32_t* pend_low, uint2* pend_high, SweepRed* red) {
  if (!n) return;
  k_collect_pending<<<grid_for(n, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(
      outdeg, off, n, np, T, pend_low, pend_high, red);
  check_launch();
  count_launch(ctx);
}

void launch_expand(dynpr_context* ctx, Rows rows, uint8_t* va, const uint32_t* pend_low, uint32_t n_low,
                   const uint2* pend_high, uint32_t n_high) {
  if (n_low) {
    k_expand_low<<<grid_for(n_low, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(rows, pend_low, n_low,
                                                                                            va, nullptr, nullptr);
    check_launch();
    count_launch(ctx);
  }
  if (n_high) {
    k_expand_high<<<grid_for((uint64_t)n_high * 32, kThreads, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(
        rows, pend_high, n_high, va, nullptr, nullptr);
    check_launch();
    count_launch(ctx);
  }
}

void launch_empty_check(dynpr_context* ctx, LoopCtl* c, int half, cudaStream_t stream, cudaGraphConditionalHandle h,
                        int set_cond) {
  if (half) k_any_affected<1><<<ctx->num_sms * 4, kThreads, 0, stream>>>(c);
  else k_any_affected<0><<<ctx->num_sms * 4, kThreads, 0, stream>>>(c);
  k_empty_finish<<<1, 1, 0, stream>>>(c, h, set_cond);
  check_launch();
  count_launch(ctx, 2);
}

void launch_loop_end(dynpr_context* ctx, LoopCtl* c, SweepRed* red, cudaGraphConditionalHandle h,
                     int set_cond, cudaGraphConditionalHandle hpush, int has_push, cudaGraphConditionalHandle hempty,
                     int has_empty) {
  k_loop_end<<<1, 1, 0, ctx->stream>>>(c, red, h, set_cond, hpush, has_push, hempty, has_empty);
  check_launch();
  count_launch(ctx);
}

__global__ void k_set_int(int* p, int v) { *p = v; }
void launch_set_expand(dynpr_context* ctx, int* p, int v) {
  k_set_int<<<1, 1, 0, ctx->stream>>>(p, v);
  check_launch();
  count_launch(ctx);
}

void launch_collect_signs(dynpr_context* ctx, const SweepArgs& a, SweepRed* out) {
  DYNPR_CK(cudaMemsetAsync(out, 0, sizeof(SweepRed), ctx->stream));
  k_collect_signs<<<(unsigned)ctx->num_sms * 16, kThreads, 0, ctx->stream>>>(a, out);
  check_launch();
  count_launch(ctx);
}

void launch_expand_dev(dynpr_context* ctx, Rows rows, uint8_t* va, const uint32_t* pend_low, const uint2* pend_high,
                       const unsigned* counts, const int* gate) {
  const unsigned g = (unsigned)ctx->num_sms * 16;
  k_expand_low<<<g, kThreads, 0, ctx->stream>>>(rows, pend_low, 0, va, counts, gate);
  check_launch();
  k_expand_high<<<g, kThreads, 0, ctx->stream>>>(rows, pend_high, 0, va, counts, gate);
  check_launch();
  count_launch(ctx, 2);
}

uint64_t mark_reachable(dynpr_context* ctx, Rows rows, uint32_t n, uint64_t m,
                        const uint32_t* inv, const uint32_t* seeds, uint64_t ns, uint8_t* flags) {
  cudaStream_t st = ctx->stream;
  auto* cnt = reinterpret_cast<unsigned*>(ctx->scratch32a.as<unsigned>(2));
  uint64_t items_total = 0;
  if (!ns || !n) return 0;
  const uint64_t cap = (uint64_t)n + m / kBfsChunk + 1;  // every vertex's items, once
  uint2* fa = ctx->bfs_a.as<uint2>(cap);
  uint2* fb = ctx->bfs_b.as<uint2>(cap);
  DYNPR_CK(cudaMemsetAsync(cnt, 0, 4, st));
  k_bfs_seed<<<grid_for(ns, kThreads, ctx->num_sms * 16), kThreads, 0, st>>>(rows, inv, seeds, ns, flags, fa, cnt);
  check_launch();
  count_launch(ctx);
  for (;;) {
    unsigned nf = 0;
    DYNPR_CK(cudaMemcpyAsync(ctx->pinned, cnt, 4, cudaMemcpyDeviceToHost, st));
    sync(ctx);
    std::memcpy(&nf, ctx->pinned, 4);
    items_total += nf;
    if (!nf) break;
    DYNPR_CK(cudaMemsetAsync(cnt, 0, 4, st));
    k_bfs_level<<<grid_for((uint64_t)nf * 32, kThreads, ctx->num_sms * 16), kThreads, 0, st>>>(rows, fa, nf, flags,
                                                                                           fb, cnt);
    check_launch();
    count_launch(ctx);
    std::swap(fa, fb);
  }
  return items_total;
}

void launch_fingerprint(dynpr_context* ctx, const uint32_t* words, uint64_t count, uint64_t salt,
                        unsigned long long* acc) {
  if (!count) return;
  k_fingerprint<<<grid_for(count, kThreads, ctx->num_sms * 8), kThreads, 0, ctx->stream>>>(words, count, salt, acc);
  check_launch();
  count_launch(ctx);
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

extern "C" dynpr_status dynpr_debug_loop_trace(uint64_t* out, uint64_t cap, uint64_t* count) {
  dynpr_b200::NvtxRange nvtx__("dynpr_debug_loop_trace");
  return dynpr_b200::api_guard([&] {
    const uint64_t n = 4ull * dynpr_b200::kLoopTraceIters;
    if (count) *count = n;
    if (out && cap) DYNPR_CK(cudaMemcpyFromSymbol(out, dynpr_b200::g_loop_trace, (cap < n ? cap : n) * 8));
  });
}

extern "C" dynpr_status dynpr_debug_sweep_trace(uint64_t* out, uint64_t cap, uint64_t* count) {
  return dynpr_b200::api_guard([&] {
    const uint64_t n = 6ull * dynpr_b200::kTraceWarps;
    if (count) *count = n;
    if (out && cap) DYNPR_CK(cudaMemcpyFromSymbol(out, dynpr_b200::g_trace, (cap < n ? cap : n) * 8));
  });
}
