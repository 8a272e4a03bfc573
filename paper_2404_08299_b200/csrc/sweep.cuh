// Internal interface between the sweep kernels (sweep.cu) and the engines
// (engine.cu).  Not part of the public C-ABI.
#pragma once

#include "common.cuh"
#include "layout.cuh"

namespace dynpr_b200 {

// Edges per partial sum for high in-degree vertices (rank.cpp:42 kAccumChunk).
constexpr uint32_t kAccumChunk = 256;

// Largest team whose peer buffers the sweep epilogue writes (one B200 box).
constexpr int kMaxPeers = 8;

// Stable degree partition of one graph (partition.cpp:7-61), used by the
// partitionByDegree entry point.
struct Schedule {
  uint32_t threshold = 0;
  uint32_t n_low = 0;
  uint32_t n_high = 0;
};
Schedule build_partition(dynpr_context* ctx, const dynpr_graph* g, uint32_t thr, uint32_t* order);

// Out-rows of a graph for push expansion / markReachable: a canonical CSR
// (deg null: row u = tgt[beg[u] .. beg[u+1])) or the engine layout's
// copy-on-write relabelled forward graph (row u = deg[u] words from
// tgt + beg[u], beg a 64-bit word offset that may wrap below tgt).
struct Rows {
  const uint64_t* beg;
  const uint32_t* deg;
  const uint32_t* tgt;
  __device__ __forceinline__ const uint32_t* row(uint32_t u) const { return tgt + beg[u]; }
  __device__ __forceinline__ uint64_t len(uint32_t u) const {
    return deg ? (uint64_t)deg[u] : beg[u + 1] - beg[u];
  }
};

struct SweepArgs {
  // engine layout (new-id space)
  uint32_t n, M, T;
  const uint32_t* indeg;
  const uint32_t* outdeg;
  uint64_t n_sslices;
  const uint64_t* sbase;
  const uint32_t* sell_s;
  uint64_t n_mseg, n_mslices;
  const uint64_t* mbase;
  const uint32_t* mseg_v;
  const uint32_t* mseg_len;
  const uint32_t* pbase;
  const uint32_t* sell_m;
  double* partials;
  uint32_t* tick_sm;     // fused sweep: per-block heavy-item counters (zeroed before each sweep)
  uint32_t* mcount;      // per multi vertex chunk-completion counters (fused sweep)
  uint64_t ss_heavy;     // single slices [0, ss_heavy) are heavy (layout n_hslices)
  int trace;     // debug: record per-warp timelines of the fused sweep (DYNPR_TRACE)
  // every in-list holds its own vertex: an in-degree-1 segment is the
  // self-loop alone, summed from the vertex's own contribution (no index or
  // gather load)
  int loops;
  // iteration state
  double alpha, teleport, tf, tp;
  const double* rank_prev;
  double* rank_cur;
  const double* contrib_prev;  // rank_prev[u] / outdeg(u), gathered
  double* contrib_cur;         // rank_cur[v] / outdeg(v), or null
  uint8_t* va;                 // vertexAffected (flagged mode)
  uint8_t* np;                 // neighborsPending, or null (engine mode)
  uint8_t* written;            // "buffers differ" flag, or null
  uint32_t* pend_low;          // pending list, out-degree <= T (or null)
  uint2* pend_high;            // (vertex, 1024-edge chunk) items, out-degree > T
  SweepRed* red;
  int np_accumulate;  // updateRanks primitive: np |= pend, untouched otherwise
  // In-sweep pull (device loop): each new contribution carries
  // its vertex's pending decision in the sign bit (contributions are >= 0,
  // every gather sums |x|), and a sweep that follows a pull-mode expansion
  // decision gathers the in-lists of the unaffected vertices too -- a vertex
  // with a pending in-neighbour is affected (frontier.cpp:55-84) and its sum
  // is already in hand.  `written` then counts the copy-throughs still owed
  // (2 after a pending write: the older buffer's sign bit must be cleared).
  int pull_fused;
  // With pull_fused: a pull sweep does not append the push-expansion lists
  // (the next expansion is usually a pull again); a push decided after it
  // collects them from the contributions' sign bits (k_collect_signs_c).
  int lazy_lists;
  int copy_all;       // updateRanks primitive: copy-through every unaffected
  // owned work (multi-GPU rank; the whole graph on one GPU): vertices
  // [v_lo, v_hi), single slices [ss_lo, ss_hi), multi slices [ms_lo, ms_hi)
  uint32_t v_lo, v_hi;
  uint64_t ss_lo, ss_hi, ms_lo, ms_hi;
  // fused exchange (multi-GPU team with peer-mapped contribution buffers):
  // the other ranks' copies of contrib_cur, written alongside the local one
  int npeers;
  double* peer_cur[kMaxPeers];
  // device-driven loop (engine.cu run_device_loop): every kernel of an
  // iteration returns at once when *done is set; the pull kernels run only
  // when *expand == kExpandPull.  Null in the host-driven loop.
  const int* done;
  const int* expand;
  // relabelled forward graph for the device loop's push expansion
  // (Rows{begF, outdeg, tgtF})
  const uint64_t* begF;
  const uint32_t* tgtF;
};

// Device-driven convergence loop state (convergeLoop's bookkeeping,
// engine.cpp:71-92, kept on the device so no iteration waits on the host).
enum { kExpandNone = 0, kExpandPush = 1, kExpandPull = 2, kExpandPushCollect = 3 };
struct LoopCtl {
  int done, converged, iterations, max_iter;
  int check, frontier, flagged, expand;
  int lazy_lists;        // pull sweeps skip the pending-list appends (SweepArgs::lazy_lists)
  int push_cost;         // direction rule: push when push_cost * pending out-edges <= unaffected in-edges
  unsigned pend_low, pend_high;  // push-expansion list sizes of the last sweep
  unsigned pushes;               // push expansions run (their IF bodies executed)
  unsigned empty_checks;         // DF-P end-game checks run (their IF bodies executed)
  int check_empty;               // no vertex pending after the sweep: is any still affected?
  unsigned kept;                 // (k_any_affected: some vertex still affected)
  int skipped;                   // the last iteration was accounted without its (empty) sweep
  double tol, final_delta;
  unsigned long long affected, edges, m, n;
};
// One iteration's bookkeeping (single thread): count, delta, convergence,
// max-iterations, expansion direction; `set_cond` also sets the WHILE
// node's condition to !done, `has_push` the IF node `hpush` (around the push
// expansion) to "a push follows".
void launch_loop_end(dynpr_context* ctx, LoopCtl* c, SweepRed* red, cudaGraphConditionalHandle h,
                     int set_cond, cudaGraphConditionalHandle hpush = 0, int has_push = 0,
                     cudaGraphConditionalHandle hempty = 0, int has_empty = 0);
// DF-P end game (the body of the IF node `hempty` that k_loop_end arms when a
// sweep leaves no vertex pending): if no vertex is still affected either,
// the next iteration would affect nothing -- it is accounted without its
// sweep (iterations + 1, delta 0, converged, LoopCtl::skipped) and the loop
// ends; `set_cond` also clears the WHILE node's condition `h`.
void launch_empty_check(dynpr_context* ctx, LoopCtl* c, int half, cudaStream_t stream, cudaGraphConditionalHandle h,
                        int set_cond);
// Push expansion with device-resident list sizes (counts[0] low, counts[1]
// high), optionally gated on *gate == kExpandPush; fixed grids.
void launch_expand_dev(dynpr_context* ctx, Rows rows, uint8_t* va,
                       const uint32_t* pend_low, const uint2* pend_high, const unsigned* counts, const int* gate);

// Edge-balanced partition of the layout's vertex space over `world` ranks
// (SURVEY 8e): contiguous new-id ranges, aligned to 32-vertex slices in the
// single region; computed on the host once per (layout, world) and cached.
std::vector<RankRange> plan_ranges(dynpr_context* ctx, Layout* L, int world);

SweepArgs layout_args(const Layout* L, double* partials);

// One synchronous sweep: single-segment slices, multi-segment slices,
// ordered combine of the multi-vertex partials.
void launch_sweep(dynpr_context* ctx, const SweepArgs& a, bool flagged, bool closed);
// Launch plan of one sweep for the cached device-loop graph: kernel choice
// (fused / split) and every grid.  Plans compare bytewise.
struct SweepPlan {
  int flagged, closed, split, pull_fused, grouped;
  unsigned g_fused, g_mseg, g_single, g_mfinal, g_pull_m, g_pull_s;
};
SweepPlan plan_sweep(dynpr_context* ctx, const SweepArgs& a, bool flagged, bool closed);
// The sweep / pull / push-expansion launches of a plan for half-iteration
// `half` (0: R0->R1, 1: R1->R0), reading their SweepArgs from the constant
// bank (upload_loop_args, stream-ordered), for capture into the loop graph.
void launch_sweep_ind(dynpr_context* ctx, const SweepPlan& p, int half, uint32_t* tick);
void launch_pull_ind(dynpr_context* ctx, const SweepPlan& p, int half);
void launch_expand_ind(dynpr_context* ctx, int half, LoopCtl* dc, cudaStream_t stream);
void upload_loop_args(dynpr_context* ctx, const SweepArgs* host_pinned_half2);
// The multi-chunk sweep kernels, whose nodes get the highest launch priority
// in the loop graph (they run concurrently with the single-vertex kernel).
bool is_priority_sweep_kernel(const void* f);
// Whether a whole-graph sweep of this layout takes the split kernels.
bool sweep_is_split(dynpr_context* ctx, const Layout* L);
uint32_t* sweep_tick(dynpr_context* ctx);
// Allocates the sweep launch workspace and resolves every kernel's persistent
// grid, so launch_sweep / launch_pull_expand can be stream-captured.
void prepare_sweep_launch(dynpr_context* ctx);

// rank / contribution initialisation in new-id order: r = init_old[perm[v]]
// (the previous ranks in old-id order) or `uniform`; c = r / outdeg; r1 / c1
// (copies) may be null.
void launch_init_ranks(dynpr_context* ctx, const Layout* L, const double* init_old, double uniform, double* r0,
                       double* r1, double* c0, double* c1);

// Frontier (frontier.cpp).  initialAffected marks the batch endpoints
// (ids mapped through `inv` when given); collect_pending turns pending flags
// into expansion lists (out-degree from `outdeg` when given, else `off`);
// push expansion over a CSR (off/tgt); pull expansion over the layout.
void launch_init_affected(dynpr_context* ctx, const uint32_t* inv, const uint32_t* ds, const uint32_t* dd,
                          uint64_t nd, const uint32_t* is, uint64_t ni, uint8_t* va, uint8_t* np);
void launch_collect_pending(dynpr_context* ctx, const uint32_t* outdeg, const uint64_t* off, uint32_t n,
                            const uint8_t* np, uint32_t T, uint32_t* pend_low, uint2* pend_high, SweepRed* red);
void launch_expand(dynpr_context* ctx, Rows rows, uint8_t* va,
                   const uint32_t* pend_low, uint32_t n_low, const uint2* pend_high, uint32_t n_high);
void launch_pull_expand(dynpr_context* ctx, const SweepArgs& a);
// Host-loop lazy lists: the pending vertices of the sweep that wrote
// a.contrib_cur (negative entries) -> a.pend_low / a.pend_high, counts into
// out->pend_low / pend_high (zeroed here).
void launch_collect_signs(dynpr_context* ctx, const SweepArgs& a, SweepRed* out);
// *p = v on the stream (the host loop's expansion decision for the next sweep)
void launch_set_expand(dynpr_context* ctx, int* p, int v);

// markReachable (frontier.cpp:86-121): flags |= everything reachable from
// the seeds over the CSR (off, tgt; m edges); seed ids mapped through `inv`
// when given.  Level-synchronous; frontier items are (vertex, 1024-edge
// chunk).  Returns the number of frontier items processed.
uint64_t mark_reachable(dynpr_context* ctx, Rows rows, uint32_t n, uint64_t m,
                        const uint32_t* inv, const uint32_t* seeds, uint64_t ns, uint8_t* flags);

// Norms (rank.cpp:142-152).
// adds the fingerprint of `count` 32-bit words to *acc (team graph identity check)
void launch_fingerprint(dynpr_context* ctx, const uint32_t* words, uint64_t count, uint64_t salt,
                        unsigned long long* acc);
void launch_linf(dynpr_context* ctx, const double* a, const double* b, uint64_t n, unsigned long long* out_bits);
void launch_l1(dynpr_context* ctx, const double* a, const double* b, uint64_t n, double* partials, double* out);

}  // namespace dynpr_b200
