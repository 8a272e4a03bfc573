// Internal interface between the sweep kernels (sweep.cu) and the engines
// (engine.cu).  Not part of the public C-ABI.
#pragma once

#include "common.cuh"

namespace dynpr_b200 {

// Edges per partial sum for high in-degree vertices (rank.cpp:42 kAccumChunk).
constexpr uint32_t kAccumChunk = 256;

// Degree schedule of one graph: the reference's in-degree partition
// (partition.cpp:7-61) extended with the 256-edge chunk table that the
// warp-cooperative high-degree kernel walks.
struct Schedule {
  uint32_t threshold = 0;
  uint32_t n_low = 0;     // vertices with degree <= threshold (lowCount)
  uint32_t n_high = 0;
  uint64_t n_chunks = 0;  // chunks over high vertices
  uint32_t n_multi = 0;   // high vertices with more than one chunk
  const uint2* chunks = nullptr;  // (vertex, chunk index j)
  const uint2* multi = nullptr;   // (vertex, first chunk)
  double* partials = nullptr;     // one per chunk
};

struct SweepArgs {
  const uint64_t* offT;  // in-CSR (transpose) offsets
  const uint32_t* idxT;  // in-neighbour ids, ascending per slice
  const uint64_t* offF;  // forward offsets (out-degree source)
  uint32_t n;
  uint32_t T;            // lowDegreeThreshold
  double alpha, teleport, tf, tp;
  const double* rank_prev;
  double* rank_cur;
  const double* contrib_prev;  // rank_prev[u] / outdeg(u), gathered
  double* contrib_cur;         // rank_cur[v] / outdeg(v), or null
  uint8_t* va;                 // vertexAffected (flagged mode)
  uint8_t* np;                 // neighborsPending, or null (engine mode)
  uint8_t* written;            // "buffers differ" flag, or null
  uint32_t* pend_low;          // pending list, out-degree <= T (or null)
  uint32_t* pend_high;         // pending list, out-degree  > T
  SweepRed* red;
  const uint2* chunks;
  uint64_t n_chunks;
  const uint2* multi;
  uint32_t n_multi;
  double* partials;
  int np_accumulate;  // updateRanks primitive: np |= pend, untouched otherwise
  int copy_all;       // updateRanks primitive: copy-through every unaffected
};

// Builds the schedule of `g` by degree threshold `thr` (3 kernels: tile
// counts, scan, stable scatter).  When `order` is non-null the full
// partition order (low group then high group) is also written there.
Schedule build_schedule(dynpr_context* ctx, const dynpr_graph* g, uint32_t thr,
                        uint32_t* order, bool want_chunks);

// One synchronous sweep (low kernel + chunk kernel + multi-chunk finalize).
void launch_sweep(dynpr_context* ctx, const SweepArgs& a, bool flagged,
                  bool closed, uint32_t n_low_hint);

// rank[v] = contrib... initialisation: r0 = value or copy of `init`.
void launch_init_ranks(dynpr_context* ctx, const dynpr_graph* gF,
                       const double* init, double uniform, double* r0,
                       double* r1, double* c0, double* c1);

// Frontier (frontier.cpp): batch seeding and push expansion.
void launch_init_affected(dynpr_context* ctx, const dynpr_graph* gF,
                          const uint32_t* ds, const uint32_t* dd, uint64_t nd,
                          const uint32_t* is, uint64_t ni, uint8_t* va,
                          uint8_t* np, uint32_t T, uint32_t* pend_low,
                          uint32_t* pend_high, SweepRed* red);
void launch_collect_pending(dynpr_context* ctx, const dynpr_graph* gF,
                            const uint8_t* np, uint32_t T, uint32_t* pend_low,
                            uint32_t* pend_high, SweepRed* red);
void launch_expand(dynpr_context* ctx, const dynpr_graph* gF, uint8_t* va,
                   const uint32_t* pend_low, uint32_t n_low,
                   const uint32_t* pend_high, uint32_t n_high);

// Norms (rank.cpp:142-152).
void launch_linf(dynpr_context* ctx, const double* a, const double* b,
                 uint64_t n, unsigned long long* out_bits);
void launch_l1(dynpr_context* ctx, const double* a, const double* b, uint64_t n,
               double* partials, double* out);

}  // namespace dynpr_b200
