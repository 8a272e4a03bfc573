// Engine layout of a (gT, gF) graph pair: the device format the sweep
// kernels read.  Built once per immutable graph snapshot and cached on the
// transpose handle (keyed by the forward graph's id and the degree
// threshold), like the CSR itself.
//
//  * Vertices are relabelled: new id = rank of the vertex when sorted by
//    in-degree descending (stable by old id).  Per-vertex arrays (ranks,
//    contributions, flags, degrees) live in new-id order, so the hot,
//    high-degree vertices -- whose contributions are gathered most -- are
//    packed at the front of the contribution vector (L2 locality).
//  * Every vertex's in-neighbour list is split into the reference's
//    accumulation segments (rank.cpp:42-75): one flat segment when
//    in-degree <= max(T, 256), else 256-edge chunks ("multi" vertices,
//    the prefix [0, M) of new ids).
//  * Segments are stored SELL-32 (sliced ELLPACK, slice = one warp): element
//    k of the 32 segments of slice s sits at base[s] + 32*k + lane, column ids
//    already relabelled, each segment keeping the reference's ascending-old-id
//    order.  A warp walks 32 segments in lock step with fully coalesced index
//    loads and every lane sums its own segment in order -- the reference's
//    accumulation order, bit for bit, with no shared-memory staging.
//  * For the frontier engines the forward graph is also relabelled (rows and
//    columns) for push expansion in new-id space; derived snapshots share
//    its untouched rows copy-on-write.
#pragma once

#include "common.cuh"

namespace dynpr_b200 {

// SELL-32x4 interleave: element k of lane i of a slice starting at `base`
// lives at base + 128*(k/4) + 4*i + k%4, so a lane fetches 4 consecutive
// elements with one 16-byte load and a warp load covers 512 contiguous bytes.
// Slice lengths are padded to a multiple of 4.
__host__ __device__ __forceinline__ uint64_t sell_pos(uint64_t base, uint32_t lane, uint32_t k) {
  return base + 128ull * (k >> 2) + 4u * lane + (k & 3u);
}

// One rank's share of the sweep work (multi-GPU): vertices [v_lo, v_hi),
// single-region slices [ss_lo, ss_hi), multi-region slices [ms_lo, ms_hi).
struct RankRange {
  uint32_t v_lo, v_hi;
  uint64_t ss_lo, ss_hi, ms_lo, ms_hi;
};

// Single-region slices whose first (largest) segment is longer than this are
// "heavy": the fused sweep schedules them one at a time, first, together with
// the multi-vertex chunk slices (their lane chains set the sweep's latency).
constexpr uint32_t kHeavyDeg = 64;

struct Layout {
  dynpr_context* ctx = nullptr;
  uint32_t n = 0;
  uint64_t m = 0;
  uint32_t T = 0;
  uint64_t gF_id = 0;
  uint32_t* perm = nullptr;    // new -> old
  uint32_t* inv = nullptr;     // old -> new
  uint32_t* indeg = nullptr;   // new order
  uint32_t* outdeg = nullptr;  // new order
  uint32_t M = 0;              // multi-segment vertices are [0, M)
  bool loops = false;          // every in-list holds its own vertex (gT carries all self-loops)
  // single-segment region: vertices [M, n), slice s = vertices M+32s..+31
  uint64_t n_sslices = 0;
  uint64_t n_hslices = 0;      // leading single slices with in-degree > kHeavyDeg
  uint64_t* sbase = nullptr;   // n_sslices + 1
  uint32_t* sell_s = nullptr;
  // multi region: segments in (vertex, chunk) order
  uint64_t n_mseg = 0;
  uint64_t n_mslices = 0;
  uint64_t* mbase = nullptr;   // n_mslices + 1
  uint32_t* mseg_v = nullptr;  // vertex of segment
  uint32_t* mseg_len = nullptr;
  uint32_t* pbase = nullptr;   // first segment of multi vertex v (M + 1)
  uint32_t* sell_m = nullptr;
  // Multi-GPU team layouts hold only this rank's rows: sell_s / sell_m are
  // then virtual bases (valid for the owned slices [own.ss_lo, own.ss_hi) /
  // [own.ms_lo, own.ms_hi) only) into the allocations below (SURVEY 8e:
  // per-rank in-CSR rows; the O(n) vertex arrays stay whole).
  bool owned = false;
  RankRange own{};
  // SELL storage this layout reads.  A layout derived incrementally
  // (layout.cu build_incremental) shares its parent's slices copy-on-write:
  // sell_s / sell_m stay the root build's base pointers and sbase / mbase of
  // re-built slices point into later blocks (64-bit offsets relative to the
  // base, wrapping when a block sits below it), so the blocks of the whole
  // chain stay alive with every layout that reads them.
  std::vector<std::shared_ptr<uint32_t>> blocks;
  uint64_t sell_words = 0;  // SELL words held on this rank (both regions, incl. shared)
  uint64_t dead_segs = 0;   // multi-region segments retired by derivations (len 0)
  uint32_t* mcount = nullptr;  // per multi vertex: chunks finished this sweep (0 between sweeps)
  // relabelled forward graph (frontier engines): row v = outdeg[v] words at
  // tgtF + begF[v] (a 64-bit word offset from the shared base, wrapping when
  // a derived layout's block sits below it).  A full build stores the rows in
  // CSR order (begF = exclusive scan of outdeg, n + 1 entries); a derived
  // layout re-points only the rows the batch touched (copy-on-write, the
  // blocks held in `blocks`)
  bool has_forward = false;
  uint64_t* begF = nullptr;
  uint32_t* tgtF = nullptr;
  uint64_t fwd_words = 0;  // forward words allocated along this layout's chain
  double build_ms = 0.0;       // device time of the last (re)build
  // multi-GPU partition cache (sweep.cu plan_ranges)
  int plan_world = 0;
  std::vector<RankRange> plan;
  // content fingerprint of the graph pair (team identity check), 0 = not yet
  uint64_t fingerprint = 0;
  // derivations since the last full build (layout.cu build_incremental)
  int generation = 0;
  ~Layout();
};

// What an incremental layout build needs (graph.cu apply_batch_pair): the
// parent pair's layout and the rows the batch touched, old ids, in the
// pool of `ctx`.  rows_T: in-lists that changed (batch destinations),
// rows_F: out-lists (batch sources).
struct LayoutSeed {
  dynpr_context* ctx = nullptr;
  std::shared_ptr<Layout> parent;
  uint64_t gF_id = 0;  // the new forward snapshot of the pair
  uint32_t* rows_T = nullptr;
  uint64_t n_T = 0;
  uint32_t* rows_F = nullptr;
  uint64_t n_F = 0;
  ~LayoutSeed();
};
std::shared_ptr<Layout> share_layout(Layout* L);

// Returns the cached layout of (gT, gF, T), building it if needed.  When
// `need_forward` the relabelled forward CSR is built too.  On a team context
// (multi-GPU) the layout holds only the calling rank's rows.
Layout* get_layout(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF, uint32_t T,
                   bool need_forward);
void destroy_layout(Layout* L);

// new-id order <-> old-id order
void launch_gather_perm_f64(dynpr_context* ctx, const Layout* L, const double* src_old, double* dst_new);
void launch_gather_perm_u8(dynpr_context* ctx, const Layout* L, const uint8_t* src_old, uint8_t* dst_new);
void launch_scatter_inv_f64(dynpr_context* ctx, const Layout* L, const double* src_new, double* dst_old);
void launch_scatter_inv_u8(dynpr_context* ctx, const Layout* L, const uint8_t* src_new, uint8_t* dst_old);

}  // namespace dynpr_b200
