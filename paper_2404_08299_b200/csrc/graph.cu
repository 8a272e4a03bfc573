// Device CSR construction and batch ingest (north_star subsystems 1 and 5).
//
// Replaces graph.cpp:56-203 of the reference:
//   buildCsr      graph.cpp:56-68   -> radix sort of packed (u,v) keys + unique
//   transpose     graph.cpp:70-83   -> stable radix sort of (v -> u) pairs
//   addSelfLoops  graph.cpp:85-111  -> applyBatch with an empty batch
//                                      (the reference's own identity,
//                                      test_graph.cpp:92-97)
//   applyBatch    graph.cpp:113-203 -> sort/unique batch, per-vertex delta,
//                                      scan, bulk tile copy of untouched
//                                      slices + warp-parallel merge of the
//                                      touched ones
// Every result is byte-identical to the reference CsrGraph (sorted,
// deduplicated slices) and validation errors carry the reference messages.
#include <atomic>

#include <cub/cub.cuh>

#include "common.cuh"
#include "layout.cuh"

namespace dynpr_b200 {

namespace {

constexpr unsigned long long kNone = ~0ull;

// ---------------------------------------------------------------------------
// SplitMix64 / deriveSeed (rng.hpp:14-19,44-47) for the RMAT generator.
__device__ __forceinline__ uint64_t splitmix_next(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void k_rmat(uint64_t count, uint32_t scale, double t1, double t2,
                       double t3, uint64_t seed, uint32_t* src, uint32_t* dst) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s0 = seed ^ (0xD1B54A32D192ED03ULL * (i + 1));
    uint64_t st = splitmix_next(s0);  // deriveSeed(seed, i)
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      const double r = (double)(splitmix_next(st) >> 11) * 0x1.0p-53;
      const uint32_t bu = r >= t2;
      const uint32_t bv = (r >= t1 && r < t2) || r >= t3;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    src[i] = u;
    dst[i] = v;
  }
}

// First list index whose endpoints fall outside [0, n) (graph.cpp:13-20
// reports the first offending pair in list order).
__global__ void k_first_bad_id(const uint32_t* s, const uint32_t* d,
                               uint64_t cnt, uint32_t n,
                               unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (s[i] >= n || d[i] >= n) atomicMin(first, (unsigned long long)i);
}
__global__ void k_first_self_pair(const uint32_t* s, const uint32_t* d,
                                  uint64_t cnt, unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (s[i] == d[i]) atomicMin(first, (unsigned long long)i);
}

__global__ void k_pack(const uint32_t* s, const uint32_t* d, uint64_t cnt,
                       int sb, uint64_t* keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = ((uint64_t)s[i] << sb) | d[i];
}

// offsets[w] for sorted source ids: every position i in [0, m] fills the
// offsets of the sources strictly after key[i-1]'s source up to key[i]'s.
__global__ void k_offsets_from_keys64(const uint64_t* keys, uint64_t m, int sb,
                                      uint32_t n, uint64_t* off) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t prev = i == 0 ? -1 : (int64_t)(keys[i - 1] >> sb);
    const int64_t cur = i == m ? (int64_t)n : (int64_t)(keys[i] >> sb);
    for (int64_t w = prev + 1; w <= cur; ++w) off[w] = i;
  }
}
__global__ void k_offsets_from_keys32(const uint32_t* keys, uint64_t m,
                                      uint32_t n, uint64_t* off) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t prev = i == 0 ? -1 : (int64_t)keys[i - 1];
    const int64_t cur = i == m ? (int64_t)n : (int64_t)keys[i];
    for (int64_t w = prev + 1; w <= cur; ++w) off[w] = i;
  }
}
__global__ void k_unpack_low(const uint64_t* keys, uint64_t m, uint64_t mask,
                             uint32_t* tgt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    tgt[i] = (uint32_t)(keys[i] & mask);
}

// Warp per vertex: write the source id of every edge of its slice.
__global__ void k_expand_sources(const uint64_t* off, uint32_t n,
                                 uint32_t* src) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t v = warp; v < n; v += nwarps) {
    const uint64_t b = off[v], e = off[v + 1];
    for (uint64_t i = b + lane; i < e; i += 32) src[i] = (uint32_t)v;
  }
}

__global__ void k_has_edge(const uint64_t* off, const uint32_t* tgt,
                           uint32_t s, uint32_t t, int* out) {
  const uint64_t b = off[s], e = off[s + 1];
  const uint64_t p = lower_bound_dev<uint32_t, uint64_t>(tgt, b, e, t);
  *out = (p < e && tgt[p] == t) ? 1 : 0;
}

// CsrGraph ctor validation (graph.cpp:38-48): per vertex, the first failing
// check in the reference's order; the global answer is the lowest vertex.
// Also records whether every vertex carries its self-loop.
// CsrGraph constructor validation (graph.cpp:30-49), edge-parallel.
// Pass 1 (vertex per thread, vertices < vlim): first vertex with decreasing
// offsets -> err[0]; marks the first edge of every non-empty row in a bitmap;
// self-loop presence by binary search.  Pass 2 (edges < elim, 4 per thread,
// coalesced): first edge whose target is out of range (code 2) or not above
// its in-row predecessor (code 3) -> err[1] = i << 2 | code.  The reference
// reports the first violation in (vertex, edge) order; the host combines the
// two passes into exactly that one.
__global__ void k_validate_rows(const uint64_t* off, const uint32_t* tgt, uint32_t vlim, uint64_t m,
                                unsigned* rowstart, unsigned long long* err, int* all_loops) {
  bool loops = true;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < vlim;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = off[v], e = off[v + 1];
    if (b > e) {
      atomicMin(err, v);
      loops = false;
      continue;
    }
    if (e > m || b == e) {
      loops = false;
      continue;
    }
    atomicOr(rowstart + (b >> 5), 1u << (b & 31));
    uint64_t lo = b, hi = e;  // lower_bound of v
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (tgt[mid] < (uint32_t)v) lo = mid + 1; else hi = mid;
    }
    if (lo == e || tgt[lo] != (uint32_t)v) loops = false;
  }
  if (!__all_sync(0xffffffffu, loops) && (threadIdx.x & 31) == 0) atomicExch(all_loops, 0);
}

__global__ void k_validate_edges(const uint32_t* tgt, uint64_t elim, uint32_t n, const unsigned* rowstart,
                                 unsigned long long* err) {
  const uint64_t nq = (elim + 3) / 4;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = 4 * q;
    uint32_t t[5];
    t[0] = i0 ? tgt[i0 - 1] : 0u;
    if (i0 + 4 <= elim) {
      const uint4 w = *reinterpret_cast<const uint4*>(tgt + i0);
      t[1] = w.x; t[2] = w.y; t[3] = w.z; t[4] = w.w;
    } else {
      for (int k = 0; k < 4; ++k) t[k + 1] = i0 + k < elim ? tgt[i0 + k] : 0u;
    }
    const unsigned rs = (rowstart[i0 >> 5] >> (i0 & 31)) & 0xfu;  // i0 % 4 == 0: same word
    for (int k = 0; k < 4 && i0 + k < elim; ++k) {
      const uint64_t i = i0 + k;
      int code = 0;
      if (t[k + 1] >= n) code = 2;
      else if (i > 0 && !((rs >> k) & 1u) && t[k] >= t[k + 1]) code = 3;
      if (code) {
        atomicMin(err, (i << 2) | code);
        break;
      }
    }
  }
}

// ---- applyBatch kernels ----------------------------------------------------
__global__ void k_overlap(const uint64_t* ins, uint64_t ni, const uint64_t* dels,
                          uint64_t nd, int* flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ni;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = lower_bound_dev<uint64_t, uint64_t>(dels, 0, nd, ins[i]);
    if (p < nd && dels[p] == ins[i]) atomicExch(flag, 1);
  }
}

__device__ __forceinline__ bool slice_has(const uint64_t* off, const uint32_t* tgt,
                                          uint32_t u, uint32_t v) {
  const uint64_t b = off[u], e = off[u + 1];
  const uint64_t p = lower_bound_dev<uint32_t, uint64_t>(tgt, b, e, v);
  return p < e && tgt[p] == v;
}

// Unique deletions: found ones shrink their source slice, absent ones are
// tallied as missing (graph.cpp:174-191).
__global__ void k_del_effect(const uint64_t* dels, uint64_t nd, int sb,
                             uint64_t mask, const uint64_t* off,
                             const uint32_t* tgt, uint8_t* found,
                             unsigned* ddel, uint8_t* touched,
                             unsigned long long* missing) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nd;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(dels[i] >> sb), v = (uint32_t)(dels[i] & mask);
    const bool f = slice_has(off, tgt, u, v);
    found[i] = f;
    if (f) {
      atomicAdd(&ddel[u], 1u);
      touched[u] = 1;
    } else {
      atomicAdd(missing, 1ull);
    }
  }
}
// Unique insertions: present ones are duplicates (graph.cpp:168-171).
__global__ void k_ins_effect(const uint64_t* ins, uint64_t ni, int sb,
                             uint64_t mask, const uint64_t* off,
                             const uint32_t* tgt, uint8_t* fresh,
                             unsigned* dins, uint8_t* touched,
                             uint8_t* loop_ins, unsigned long long* dup) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ni;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(ins[i] >> sb), v = (uint32_t)(ins[i] & mask);
    const bool present = slice_has(off, tgt, u, v);
    fresh[i] = !present;
    if (present) {
      atomicAdd(dup, 1ull);
    } else {
      atomicAdd(&dins[u], 1u);
      touched[u] = 1;
      if (u == v) loop_ins[u] = 1;
    }
  }
}
// Vertices lacking their loop get one (graph.cpp:155-163,193).
__global__ void k_need_loop(const uint64_t* off, const uint32_t* tgt, uint32_t n,
                            const uint8_t* loop_ins, uint8_t* need,
                            uint8_t* touched) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const bool has = slice_has(off, tgt, (uint32_t)v, (uint32_t)v);
    const bool nl = !has && !loop_ins[v];
    need[v] = nl;
    if (nl) touched[v] = 1;
  }
}
__global__ void k_new_degrees(const uint64_t* off, uint32_t n,
                              const unsigned* ddel, const unsigned* dins,
                              const uint8_t* need, uint64_t* noff) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (v == n) { noff[v] = 0; continue; }
    noff[v] = (off[v + 1] - off[v]) - ddel[v] + dins[v] + need[v];
  }
}

// Untouched slices keep their content and only shift: a warp per 32-vertex
// tile copies the whole contiguous range when no vertex of the tile is
// touched (the common case), else slice by slice skipping touched ones.
// Copy of one CSR row range [b, e) to d..: 16-byte stores at 16-byte
// aligned destinations, the source realigned in registers -- each lane loads
// one aligned 16-byte source block, takes its neighbour's with a shuffle and
// funnels the four words the destination block needs (the source/destination
// shift is arbitrary: it is the running balance of inserted and deleted
// edges).  Heads, tails and short ranges go 4 bytes at a time.
__device__ __forceinline__ uint4 funnel4(uint4 a, uint4 b, unsigned r) {
  switch (r) {
    case 1: return make_uint4(a.y, a.z, a.w, b.x);
    case 2: return make_uint4(a.z, a.w, b.x, b.y);
    case 3: return make_uint4(a.w, b.x, b.y, b.z);
    default: return a;
  }
}
__device__ __forceinline__ void warp_copy_words(const uint32_t* __restrict__ tgt, uint32_t* __restrict__ ntgt,
                                                uint64_t b, uint64_t e, uint64_t d, unsigned lane) {
  for (uint64_t i = b + lane; i < e; i += 32 * 8) {
    uint32_t x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = i + 32 * q < e ? __ldcs(tgt + i + 32 * q) : 0u;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (i + 32 * q < e) __stcs(ntgt + d + (i + 32 * q - b), x[q]);
  }
}
__device__ __forceinline__ void warp_copy_range(const uint32_t* __restrict__ tgt, uint32_t* __restrict__ ntgt,
                                                uint64_t b, uint64_t e, uint64_t d, unsigned lane) {
  if (e - b < 512) {
    warp_copy_words(tgt, ntgt, b, e, d, lane);
    return;
  }
  const uint64_t head = (4 - (d & 3)) & 3;  // words until the destination is 16-byte aligned
  const uint64_t S = b + head, D = d + head;
  const unsigned r = (unsigned)(S & 3);
  const uint64_t A = S - r;  // aligned source block of the first destination block
  // vector blocks j with source blocks j and j + 1 both inside [A, e)
  const uint64_t nblk = (e - A) / 4 >= 1 ? (e - A) / 4 - 1 : 0;
  const uint4* src4 = reinterpret_cast<const uint4*>(tgt + A);
  uint4* dst4 = reinterpret_cast<uint4*>(ntgt + D);
  if (lane < head) ntgt[d + lane] = tgt[b + lane];
  constexpr int U = 4;  // blocks in flight per lane (2 KB per warp)
  for (uint64_t j0 = 0; j0 < nblk; j0 += 32 * U) {
    uint4 a[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint64_t j = j0 + 32 * q + lane;
      a[q] = j < nblk ? __ldcs(src4 + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint64_t j = j0 + 32 * q + lane;
      // block j + 1: the next lane's block, lane 0's of the next group for
      // lane 31; loaded directly at the end of the round or of the range
      const unsigned srcl = (lane + 1) & 31;
      const uint4 from = (lane == 0 && q + 1 < U) ? a[q + 1 < U ? q + 1 : q] : a[q];  // lane 31 reads lane 0's
      uint4 nx;
      nx.x = __shfl_sync(0xffffffffu, from.x, srcl);
      nx.y = __shfl_sync(0xffffffffu, from.y, srcl);
      nx.z = __shfl_sync(0xffffffffu, from.z, srcl);
      nx.w = __shfl_sync(0xffffffffu, from.w, srcl);
      if (j < nblk && ((lane == 31 && q + 1 == U) || j + 1 >= nblk)) nx = __ldcs(src4 + j + 1);
      if (j < nblk) __stcs(dst4 + j, funnel4(a[q], nx, r));
    }
  }
  // tail: the words after the last vector block
  warp_copy_words(tgt, ntgt, S + 4 * nblk, e, D + 4 * nblk, lane);
}


// Untouched rows as runs: the rows between two consecutive touched rows
// keep their slices and their order, so each run is ONE contiguous copy with
// a constant source/destination shift.  Runs are cut into kRunPiece-word
// pieces, warp per piece (grid-stride over the pieces), which keeps every
// warp streaming ~32 KB instead of re-reading row metadata every 32 rows.
constexpr uint64_t kRunPiece = 8192;
__global__ void k_run_pieces(const uint32_t* T, const unsigned long long* nt_ptr, uint32_t n, const uint64_t* off,
                             uint32_t* pieces) {
  const uint64_t nt = *nt_ptr;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= nt + 1;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (j <= nt) {
      const uint64_t a = j == 0 ? 0 : (uint64_t)T[j - 1] + 1;
      const uint64_t b = j == nt ? n : T[j];
      const uint64_t words = b > a ? off[b] - off[a] : 0;
      c = (uint32_t)((words + kRunPiece - 1) / kRunPiece);
    }
    pieces[j] = c;  // entry nt + 1 stays 0: the exclusive scan's total
  }
}
__global__ void k_copy_runs(const uint32_t* T, const unsigned long long* nt_ptr, const uint32_t* pstart, uint32_t n,
                            const uint64_t* off, const uint32_t* tgt, const uint64_t* noff, uint32_t* ntgt) {
  const uint64_t nt = *nt_ptr;
  const uint32_t total = pstart[nt + 1];
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x / 32;
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t t = warp; t < total; t += nwarps) {
    const uint64_t j = upper_bound_u32(pstart, nt + 2, (uint32_t)t) - 1;  // run of piece t
    const uint64_t k = t - pstart[j];
    const uint64_t a = j == 0 ? 0 : (uint64_t)T[j - 1] + 1;
    const uint64_t b = j == nt ? n : T[j];
    const uint64_t sb = off[a] + k * kRunPiece, se0 = off[b];
    const uint64_t se = sb + kRunPiece < se0 ? sb + kRunPiece : se0;
    warp_copy_range(tgt, ntgt, sb, se, noff[a] + k * kRunPiece, lane);
  }
}

// Merge work items of the touched rows: a row of old degree d is split into
// max(1, ceil(d / kMergeChunk)) items so a touched hub (RMAT-24: ~4e5 edges)
// is spread over many warps instead of serialising one.
constexpr uint64_t kMergeChunk = 2048;
__global__ void k_merge_items(const uint8_t* touched, const uint64_t* off, uint32_t n, uint32_t* items) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (v < n && touched[v]) {
      const uint64_t d = off[v + 1] - off[v];
      c = d > kMergeChunk ? (uint32_t)((d + kMergeChunk - 1) / kMergeChunk) : 1u;
    }
    items[v] = c;
  }
}

// Rows with batch entries: every surviving old target and every fresh
// insertion is written at its final position (old index - deletions before
// it + insertions before it + the re-ensured self-loop when it precedes),
// so the items of one row are independent.  Item t -> row through the
// exclusive scan `istart` (n + 1 entries, istart[n] = total items).
__global__ void k_merge_touched(const uint32_t* istart, uint32_t n,
                                const uint64_t* off, const uint32_t* tgt,
                                const uint64_t* noff, uint32_t* ntgt,
                                const uint64_t* dp, uint64_t ndp,
                                const uint64_t* nw, uint64_t nnw, int sb,
                                uint64_t mask, const uint8_t* need) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x / 32;
  const uint32_t total = istart[n];
  for (uint64_t t = warp; t < total; t += nwarps) {
    // row u: the last u with istart[u] <= t (rows with no items share a start)
    const uint32_t u = (uint32_t)(upper_bound_u32(istart, (uint64_t)n + 1, (uint32_t)t) - 1);
    const uint64_t c = t - istart[u];
    const uint64_t so = off[u], se = off[u + 1], base = noff[u];
    const uint64_t cb = so + c * kMergeChunk, ce = cb + kMergeChunk < se ? cb + kMergeChunk : se;
    const uint64_t klo = (uint64_t)u << sb, khi = ((uint64_t)u + 1) << sb;
    const uint64_t dlo = lower_bound_dev<uint64_t, uint64_t>(dp, 0, ndp, klo);
    const uint64_t dhi = lower_bound_dev<uint64_t, uint64_t>(dp, dlo, ndp, khi);
    const uint64_t nlo = lower_bound_dev<uint64_t, uint64_t>(nw, 0, nnw, klo);
    const uint64_t nhi = lower_bound_dev<uint64_t, uint64_t>(nw, nlo, nnw, khi);
    const bool nl = need[u];
    for (uint64_t k = cb - so + lane; k < ce - so; k += 32) {
      const uint32_t x = tgt[so + k];
      const uint64_t key = klo | x;
      const uint64_t q = lower_bound_dev<uint64_t, uint64_t>(dp, dlo, dhi, key);
      if (q < dhi && dp[q] == key) continue;
      const uint64_t r = lower_bound_dev<uint64_t, uint64_t>(nw, nlo, nhi, key) - nlo;
      ntgt[base + k - (q - dlo) + r + ((nl && u < x) ? 1 : 0)] = x;
    }
    if (c != 0) continue;
    for (uint64_t k = lane; k < nhi - nlo; k += 32) {
      const uint64_t key = nw[nlo + k];
      const uint32_t x = (uint32_t)(key & mask);
      const uint64_t s = lower_bound_dev<uint32_t, uint64_t>(tgt, so, se, x) - so;
      const uint64_t q = lower_bound_dev<uint64_t, uint64_t>(dp, dlo, dhi, key) - dlo;
      ntgt[base + s - q + k + ((nl && u < x) ? 1 : 0)] = x;
    }
    if (nl && lane == 0) {
      const uint64_t key = klo | u;
      const uint64_t s = lower_bound_dev<uint32_t, uint64_t>(tgt, so, se, u) - so;
      const uint64_t q = lower_bound_dev<uint64_t, uint64_t>(dp, dlo, dhi, key) - dlo;
      const uint64_t r = lower_bound_dev<uint64_t, uint64_t>(nw, nlo, nhi, key) - nlo;
      ntgt[base + s - q + r] = u;
    }
  }
}

// ---- helpers -------------------------------------------------------------
int key_shift(uint32_t n) {
  int sb = bits_for(n ? n - 1 : 0);
  return sb < 1 ? 1 : sb;
}

unsigned long long read_u64(dynpr_context* ctx, const unsigned long long* d) {
  unsigned long long h;
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, d, sizeof h, cudaMemcpyDeviceToHost,
                           ctx->stream));
  sync(ctx);
  std::memcpy(&h, ctx->pinned, sizeof h);
  return h;
}

unsigned long long* scratch_u64(dynpr_context* ctx, DevBuf& b, int count,
                                unsigned long long init) {
  auto* p = b.as<unsigned long long>(count);
  std::vector<unsigned long long> h(count, init);
  DYNPR_CK(cudaMemcpyAsync(p, h.data(), count * sizeof(unsigned long long),
                           cudaMemcpyHostToDevice, ctx->stream));
  sync(ctx);  // h is pageable and leaves scope
  return p;
}

std::pair<uint32_t, uint32_t> fetch_pair(dynpr_context* ctx, const uint32_t* d_s,
                                         const uint32_t* d_d, const uint32_t* h_s,
                                         const uint32_t* h_d, uint64_t i) {
  if (h_s && h_d) return {h_s[i], h_d[i]};
  uint32_t a = 0, b = 0;
  DYNPR_CK(cudaMemcpy(&a, d_s + i, 4, cudaMemcpyDeviceToHost));
  DYNPR_CK(cudaMemcpy(&b, d_d + i, 4, cudaMemcpyDeviceToHost));
  return {a, b};
}

void check_ids(dynpr_context* ctx, const uint32_t* d_s, const uint32_t* d_d,
               uint64_t cnt, uint32_t n, const char* what, const uint32_t* h_s,
               const uint32_t* h_d) {
  if (!cnt) return;
  auto* first = scratch_u64(ctx, ctx->scratch64b, 1, kNone);
  k_first_bad_id<<<grid_for(cnt, 256, 4096), 256, 0, ctx->stream>>>(d_s, d_d, cnt, n, first);
  check_launch();
  count_launch(ctx);
  const unsigned long long i = read_u64(ctx, first);
  if (i != kNone) {
    auto [u, v] = fetch_pair(ctx, d_s, d_d, h_s, h_d, i);
    invalid(std::string(what) + ": vertex id out of range (" + std::to_string(u) +
            "," + std::to_string(v) + ") for |V|=" + std::to_string(n));
  }
}

template <class F>
void cub_call(dynpr_context* ctx, F&& f) {
  size_t bytes = 0;
  DYNPR_CK(f(nullptr, bytes));
  void* tmp = ctx->cub_tmp.ensure(bytes);
  DYNPR_CK(f(tmp, bytes));
}

// Sorts + dedupes packed keys; returns the unique count (keys end in `out`).
uint64_t sort_unique(dynpr_context* ctx, uint64_t* keys, uint64_t* alt,
                     uint64_t cnt, int end_bit, uint64_t** out) {
  if (cnt == 0) {
    *out = keys;
    return 0;
  }
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  cub_call(ctx, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, db, cnt, 0, end_bit, ctx->stream);
  });
  uint64_t* sorted = db.Current();
  uint64_t* uniq = db.Alternate();
  auto* num = reinterpret_cast<unsigned long long*>(ctx->scratch64a.as<unsigned long long>(1));
  cub_call(ctx, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, sorted, uniq, num, (int64_t)cnt, ctx->stream);
  });
  *out = uniq;
  return read_u64(ctx, num);
}

}  // namespace

// True when any (s[i], d[i]) falls outside [0, n) (frontier.cpp:24-29).
bool any_bad_ids(dynpr_context* ctx, const uint32_t* d_s, const uint32_t* d_d, uint64_t cnt, uint32_t n) {
  if (!cnt) return false;
  auto* first = scratch_u64(ctx, ctx->scratch64b, 1, kNone);
  k_first_bad_id<<<grid_for(cnt, 256, 4096), 256, 0, ctx->stream>>>(d_s, d_d, cnt, n, first);
  check_launch();
  count_launch(ctx);
  return read_u64(ctx, first) != kNone;
}

// ---------------------------------------------------------------------------
dynpr_graph* new_graph_struct(dynpr_context* ctx, uint32_t n) {
  static std::atomic<uint64_t> next_id{1};
  auto* g = new dynpr_graph();
  g->id = next_id.fetch_add(1);
  g->ctx = ctx;
  g->n = n;
  if (ctx) ctx->live_graphs.fetch_add(1);
  return g;
}

dynpr_graph* make_graph(dynpr_context* ctx, uint32_t n, uint64_t m) {
  dynpr_graph* g = new_graph_struct(ctx, n);
  g->m = m;
  try {
    g->off = pool_alloc_n<uint64_t>(ctx, (uint64_t)n + 1);
    g->tgt = pool_alloc_n<uint32_t>(ctx, m ? m : 1);
  } catch (...) {
    destroy_graph(g);
    throw;
  }
  return g;
}

void destroy_graph(dynpr_graph* g) {
  if (!g) return;
  g->layout.reset();  // (freed through the context's pool: before its teardown)
  g->seed.reset();
  dynpr_context* ctx = g->ctx;
  pool_free(ctx, g->off);
  pool_free(ctx, g->tgt);
  delete g;
  // the context's own destroy came first: its teardown waited for us
  if (ctx && ctx->live_graphs.fetch_sub(1) == 1 && ctx->closing.load() && !ctx->torn_down.exchange(true))
    context_teardown(ctx);
}

// buildCsr on device from device edge arrays (validation already done).
static dynpr_graph* build_from_device_edges(dynpr_context* ctx, uint32_t n,
                                            const uint32_t* d_s,
                                            const uint32_t* d_d, uint64_t cnt) {
  const int sb = key_shift(n);
  const uint64_t mask = (sb >= 64) ? ~0ull : ((1ull << sb) - 1);
  uint64_t* keys = ctx->stage_c.as<uint64_t>(cnt ? cnt : 1);
  uint64_t* alt = ctx->stage_d.as<uint64_t>(cnt ? cnt : 1);
  if (cnt) {
    k_pack<<<grid_for(cnt, 256, 1 << 16), 256, 0, ctx->stream>>>(d_s, d_d, cnt, sb, keys);
    check_launch();
    count_launch(ctx);
  }
  uint64_t* uniq = nullptr;
  const uint64_t m = sort_unique(ctx, keys, alt, cnt, 2 * sb, &uniq);
  dynpr_graph* g = make_graph(ctx, n, m);
  k_offsets_from_keys64<<<grid_for(m + 1, 256, 1 << 16), 256, 0, ctx->stream>>>(uniq, m, sb, n, g->off);
  check_launch();
  if (m) {
    k_unpack_low<<<grid_for(m, 256, 1 << 16), 256, 0, ctx->stream>>>(uniq, m, mask, g->tgt);
    check_launch();
  }
  count_launch(ctx, 2);
  sync(ctx);
  return g;
}

// Rows of `touched` (flags, n entries) listed in order, and every run of
// untouched rows between them copied from (off, tgt) to (noff, ntgt) in
// 8K-word pieces: the part of a CSR rebuild that is a plain copy.  `nt` =
// device count of touched rows; the list is left in ctx->run_list.
uint32_t* copy_untouched_rows(dynpr_context* ctx, const uint8_t* touched, uint32_t n, const uint64_t* off,
                              const uint32_t* tgt, const uint64_t* noff, uint32_t* ntgt, unsigned long long* nt) {
  cudaStream_t st = ctx->stream;
  uint32_t* T = ctx->run_list.as<uint32_t>((uint64_t)n + 1);
  uint32_t* pcs = ctx->run_pieces.as<uint32_t>((uint64_t)n + 3);
  cub::CountingInputIterator<uint32_t> iota(0);
  cub_call(ctx, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, iota, touched, T, nt, (int64_t)n, st);
  });
  k_run_pieces<<<grid_for((uint64_t)n + 2, 256, 1 << 16), 256, 0, st>>>(T, nt, n, off, pcs);
  check_launch();
  cub_call(ctx, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, pcs, pcs, (int64_t)n + 3, st);
  });
  k_copy_runs<<<(unsigned)ctx->num_sms * 32, 256, 0, st>>>(T, nt, pcs, n, off, tgt, noff, ntgt);
  check_launch();
  count_launch(ctx, 2);
  return T;
}

void graph_apply_batch_impl(dynpr_context* ctx, const dynpr_graph* g,
                            const uint32_t* d_ds, const uint32_t* d_dd,
                            uint64_t nd, const uint32_t* d_is,
                            const uint32_t* d_id, uint64_t ni, bool validate,
                            const uint32_t* h_ds, const uint32_t* h_dd,
                            const uint32_t* h_is, const uint32_t* h_id,
                            dynpr_graph** out, uint64_t* missing_out,
                            uint64_t* duplicate_out, uint32_t** rows_out,
                            uint64_t* nrows_out) {
  const uint32_t n = g->n;
  cudaStream_t st = ctx->stream;
  if (validate) {  // graph.cpp:116-120, in the reference's order
    check_ids(ctx, d_ds, d_dd, nd, n, "applyBatch deletions", h_ds, h_dd);
    check_ids(ctx, d_is, d_id, ni, n, "applyBatch insertions", h_is, h_id);
    if (nd) {
      auto* first = scratch_u64(ctx, ctx->scratch64b, 1, kNone);
      k_first_self_pair<<<grid_for(nd, 256, 4096), 256, 0, st>>>(d_ds, d_dd, nd, first);
      check_launch();
      count_launch(ctx);
      if (read_u64(ctx, first) != kNone)
        invalid("applyBatch: self-loops cannot be deleted");
    }
  }
  const int sb = key_shift(n);
  const uint64_t mask = (1ull << sb) - 1;
  // sort + unique both lists (graph.cpp:122-127)
  uint64_t* dk = ctx->stage_c.as<uint64_t>(nd + 1);
  uint64_t* dk2 = ctx->stage_d.as<uint64_t>(nd + 1);
  uint64_t* ik = ctx->stage_e.as<uint64_t>(ni + 1);
  uint64_t* ik2 = ctx->stage_f.as<uint64_t>(ni + 1);
  if (nd) {
    k_pack<<<grid_for(nd, 256, 4096), 256, 0, st>>>(d_ds, d_dd, nd, sb, dk);
    check_launch();
    count_launch(ctx);
  }
  if (ni) {
    k_pack<<<grid_for(ni, 256, 4096), 256, 0, st>>>(d_is, d_id, ni, sb, ik);
    check_launch();
    count_launch(ctx);
  }
  uint64_t *du = dk, *iu = ik;
  const uint64_t ndu = sort_unique(ctx, dk, dk2, nd, 2 * sb, &du);
  const uint64_t niu = sort_unique(ctx, ik, ik2, ni, 2 * sb, &iu);
  uint64_t missing = nd - ndu, duplicate = ni - niu;
  if (validate && ndu && niu) {  // graph.cpp:130-138
    auto* flag = reinterpret_cast<int*>(scratch_u64(ctx, ctx->scratch64b, 1, 0));
    k_overlap<<<grid_for(niu, 256, 4096), 256, 0, st>>>(iu, niu, du, ndu, flag);
    check_launch();
    count_launch(ctx);
    if (read_u64(ctx, reinterpret_cast<unsigned long long*>(flag)) != 0)
      invalid("applyBatch: edge appears in both deletions and insertions");
  }
  // per-vertex deltas
  unsigned* ddel = ctx->scratch32a.as<unsigned>(2 * (uint64_t)n + 2);
  unsigned* dins = ddel + n + 1;
  uint8_t* v8 = ctx->scratch8a.as<uint8_t>(3 * (uint64_t)n + 3);
  uint8_t* touched = v8;
  uint8_t* loop_ins = v8 + n + 1;
  uint8_t* need = v8 + 2 * ((uint64_t)n + 1);
  DYNPR_CK(cudaMemsetAsync(ddel, 0, (2 * (uint64_t)n + 2) * sizeof(unsigned), st));
  DYNPR_CK(cudaMemsetAsync(v8, 0, 3 * (uint64_t)n + 3, st));
  auto* counters = scratch_u64(ctx, ctx->scratch64b, 4, 0);  // missing, dup, touched
  uint8_t* found = ctx->stage_a.as<uint8_t>(ndu + niu + 2);
  uint8_t* fresh = found + ndu + 1;
  if (ndu) {
    k_del_effect<<<grid_for(ndu, 256, 8192), 256, 0, st>>>(du, ndu, sb, mask, g->off, g->tgt, found,
                                                           ddel, touched, counters + 0);
    check_launch();
    count_launch(ctx);
  }
  if (niu) {
    k_ins_effect<<<grid_for(niu, 256, 8192), 256, 0, st>>>(iu, niu, sb, mask, g->off, g->tgt, fresh,
                                                           dins, touched, loop_ins, counters + 1);
    check_launch();
    count_launch(ctx);
  }
  if (!g->all_loops && n) {
    k_need_loop<<<grid_for(n, 256, 1 << 16), 256, 0, st>>>(g->off, g->tgt, n, loop_ins, need, touched);
    check_launch();
    count_launch(ctx);
  }
  // new offsets
  dynpr_graph* r = new_graph_struct(ctx, n);
  try {
    r->off = pool_alloc_n<uint64_t>(ctx, (uint64_t)n + 1);
  } catch (...) {
    destroy_graph(r);
    throw;
  }
  k_new_degrees<<<grid_for((uint64_t)n + 1, 256, 1 << 16), 256, 0, st>>>(g->off, n, ddel, dins, need, r->off);
  check_launch();
  count_launch(ctx);
  cub_call(ctx, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, r->off, r->off, (int64_t)n + 1, st);
  });
  uint64_t m_new = 0;
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, r->off + n, 8, cudaMemcpyDeviceToHost, st));
  sync(ctx);
  std::memcpy(&m_new, ctx->pinned, 8);
  r->m = m_new;
  try {
    r->tgt = pool_alloc_n<uint32_t>(ctx, m_new ? m_new : 1);
  } catch (...) {
    destroy_graph(r);
    throw;
  }
  // compact present deletions / fresh insertions
  uint64_t* dp = ctx->stage_d.as<uint64_t>(ndu + 1);
  uint64_t* nw = ctx->stage_f.as<uint64_t>(niu + 1);
  auto* nsel = reinterpret_cast<unsigned long long*>(ctx->scratch64a.as<unsigned long long>(2));
  uint64_t ndp = 0, nnw = 0;
  if (ndu) {
    if (du == dp) {  // sort_unique left the result in stage_d: move it aside
      DYNPR_CK(cudaMemcpyAsync(dk, du, ndu * 8, cudaMemcpyDeviceToDevice, st));
      du = dk;
    }
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, du, found, dp, nsel, (int64_t)ndu, st);
    });
    ndp = read_u64(ctx, nsel);
  }
  if (niu) {
    if (iu == nw) {
      DYNPR_CK(cudaMemcpyAsync(ik, iu, niu * 8, cudaMemcpyDeviceToDevice, st));
      iu = ik;
    }
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, iu, fresh, nw, nsel + 1, (int64_t)niu, st);
    });
    nnw = read_u64(ctx, nsel + 1);
  }
  // copies of the untouched rows + chunked merge of the touched ones
  if (n) {
    uint32_t* istart = ctx->scratch32b.as<uint32_t>((uint64_t)n + 1);
    k_merge_items<<<grid_for((uint64_t)n + 1, 256, 1 << 16), 256, 0, st>>>(touched, g->off, n, istart);
    check_launch();
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, istart, istart, (int64_t)n + 1, st);
    });
    // touched rows in order -> runs of untouched rows -> pieces -> copies
    auto* nt = reinterpret_cast<unsigned long long*>(ctx->scratch64a.as<unsigned long long>(4)) + 2;
    uint32_t* T = copy_untouched_rows(ctx, touched, n, g->off, g->tgt, r->off, r->tgt, nt);
    k_merge_touched<<<(unsigned)ctx->num_sms * 16, 256, 0, st>>>(istart, n, g->off, g->tgt, r->off, r->tgt, dp,
                                                                 ndp, nw, nnw, sb, mask, need);
    check_launch();
    count_launch(ctx, 3);
    if (rows_out) {  // the touched rows, for an incremental engine layout (layout.cu)
      const uint64_t cnt = read_u64(ctx, nt);
      uint32_t* rows = pool_alloc_n<uint32_t>(ctx, cnt ? cnt : 1);
      if (cnt) DYNPR_CK(cudaMemcpyAsync(rows, T, cnt * 4, cudaMemcpyDeviceToDevice, st));
      *rows_out = rows;
      *nrows_out = cnt;
    }
  }
  unsigned long long hc[2];
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, counters, 16, cudaMemcpyDeviceToHost, st));
  sync(ctx);
  std::memcpy(hc, ctx->pinned, 16);
  missing += hc[0];
  duplicate += hc[1];
  r->all_loops = true;
  if (missing_out) *missing_out += missing;
  if (duplicate_out) *duplicate_out += duplicate;
  *out = r;
}

}  // namespace dynpr_b200

using namespace dynpr_b200;

extern "C" {

}  // extern "C"

namespace dynpr_b200 {

// CsrGraph constructor validation (graph.cpp:30-49) of a snapshot whose
// arrays are (being) uploaded on stream `s`: err[0] first row whose offset
// decreases, err[1] first bad edge, err[2] every-row-has-its-loop flag.
// enqueue_csr_validation queues the kernels and the readback into `host`;
// finish_csr_validation waits on `s` and throws the reference's messages
// (re-scanning exactly the rows the reference would have scanned when the
// offsets decrease).
void enqueue_csr_validation(dynpr_context* ctx, dynpr_graph* g, uint32_t vlim, uint64_t elim, cudaStream_t s,
                            unsigned long long* err, unsigned* rowstart, unsigned long long* host) {
  const uint64_t m = g->m;
  const uint64_t words = (m + 31) / 32 + 1;
  const unsigned long long init[3] = {kNone, kNone, 1ull};  // loops flag = 1
  std::memcpy(host, init, sizeof init);
  DYNPR_CK(cudaMemcpyAsync(err, host, sizeof init, cudaMemcpyHostToDevice, s));
  DYNPR_CK(cudaMemsetAsync(rowstart, 0, words * 4, s));
  int* loops = reinterpret_cast<int*>(err + 2);
  if (vlim) {
    k_validate_rows<<<grid_for(vlim, 256, ctx->num_sms * 16), 256, 0, s>>>(g->off, g->tgt, vlim, m, rowstart, err,
                                                                          loops);
    check_launch();
    count_launch(ctx);
  }
  if (elim) {
    k_validate_edges<<<grid_for((elim + 3) / 4, 256, ctx->num_sms * 16), 256, 0, s>>>(g->tgt, elim, g->n, rowstart,
                                                                                      err + 1);
    check_launch();
    count_launch(ctx);
  }
  DYNPR_CK(cudaMemcpyAsync(host, err, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
}

void finish_csr_validation(dynpr_context* ctx, dynpr_graph* g, cudaStream_t s, unsigned long long* err,
                           unsigned* rowstart, unsigned long long* host) {
  DYNPR_CK(cudaStreamSynchronize(s));
  unsigned long long h[3];
  std::memcpy(h, host, sizeof h);
  if (h[0] != kNone) {
    // offsets decrease at v0: the reference scanned only the rows before it,
    // whose edges are [0, off[v0]); rescan exactly those
    const uint32_t v0 = (uint32_t)h[0];
    uint64_t lim = 0;
    DYNPR_CK(cudaMemcpy(&lim, g->off + v0, 8, cudaMemcpyDeviceToHost));
    enqueue_csr_validation(ctx, g, v0, lim < g->m ? lim : g->m, s, err, rowstart, host);
    DYNPR_CK(cudaStreamSynchronize(s));
    std::memcpy(h, host, sizeof h);
    h[0] = v0;
  }
  if (h[1] != kNone) {
    if ((h[1] & 3) == 2) invalid("CsrGraph: target id out of range");
    invalid("CsrGraph: target slices must be sorted and deduplicated");
  }
  if (h[0] != kNone) invalid("CsrGraph: offsets must be non-decreasing");
  g->all_loops = g->n == 0 || (int)(h[2] & 0xffffffffu) == 1;
}

// Host-side part of the constructor checks: offsets.front() == 0 and
// offsets.back() == targets.size().
void check_csr_ends(uint32_t n, const uint64_t* offsets, uint64_t m) {
  uint64_t first = 0, last = 0;
  if (!offsets) invalid("CsrGraph: malformed offsets array");
  if (is_device_ptr(offsets)) {
    DYNPR_CK(cudaMemcpy(&first, offsets, 8, cudaMemcpyDeviceToHost));
    DYNPR_CK(cudaMemcpy(&last, offsets + n, 8, cudaMemcpyDeviceToHost));
  } else {
    first = offsets[0];
    last = offsets[n];
  }
  if (first != 0 || last != m) invalid("CsrGraph: malformed offsets array");
}

DeferredCsr::~DeferredCsr() {
  if (pending && ctx && ctx->side) cudaStreamSynchronize(ctx->side);  // error path: the side work must end first
  if (rowstart) pool_free(ctx, rowstart);
  if (g) destroy_graph(g);
}

// Upload of a host CSR whose targets travel and are validated on the
// context's side stream (after `after` fires), overlapping whatever the
// main stream runs next; finish() joins and throws on invalid input.
void upload_csr_deferred(dynpr_context* ctx, uint32_t n, const uint64_t* offsets, const uint32_t* targets,
                         uint64_t m, cudaEvent_t after, DeferredCsr& d) {
  check_csr_ends(n, offsets, m);
  d.ctx = ctx;
  d.g = make_graph(ctx, n, m);
  d.rowstart = pool_alloc_n<unsigned>(ctx, (m + 31) / 32 + 1);
  d.err = ctx->side_err.as<unsigned long long>(3);
  d.host = reinterpret_cast<unsigned long long*>(static_cast<char*>(ctx->pinned) + 3072);
  DYNPR_CK(cudaMemcpyAsync(d.g->off, offsets, ((size_t)n + 1) * 8, cudaMemcpyDefault, ctx->stream));
  DYNPR_CK(cudaEventRecord(after, ctx->stream));  // the allocations and offsets are ordered before the side work
  cudaStream_t side = side_stream(ctx);
  DYNPR_CK(cudaStreamWaitEvent(side, after, 0));
  if (m) DYNPR_CK(cudaMemcpyAsync(d.g->tgt, targets, m * 4, cudaMemcpyDefault, side));
  enqueue_csr_validation(ctx, d.g, n, m, side, d.err, d.rowstart, d.host);
  d.pending = true;
}

void DeferredCsr::finish() {
  if (!pending) return;
  pending = false;
  finish_csr_validation(ctx, g, side_stream(ctx), err, rowstart, host);
}

cudaStream_t side_stream(dynpr_context* ctx) {
  if (!ctx->side) DYNPR_CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  return ctx->side;
}

}  // namespace dynpr_b200

extern "C" {

dynpr_status dynpr_graph_from_csr(dynpr_context* ctx, uint32_t n,
                                  const uint64_t* offsets,
                                  const uint32_t* targets, uint64_t m,
                                  dynpr_graph** out) {
  NvtxRange nvtx__("dynpr_graph_from_csr");
  return api_guard([&] {
    if (!ctx || !out) invalid("null argument");
    bind_device(ctx);
    check_csr_ends(n, offsets, m);
    dynpr_graph* g = make_graph(ctx, n, m);
    try {
      DYNPR_CK(cudaMemcpyAsync(g->off, offsets, ((size_t)n + 1) * 8, cudaMemcpyDefault, ctx->stream));
      if (m) DYNPR_CK(cudaMemcpyAsync(g->tgt, targets, m * 4, cudaMemcpyDefault, ctx->stream));
      auto* err = ctx->scratch64b.as<unsigned long long>(3);
      unsigned* rowstart = pool_alloc_n<unsigned>(ctx, (m + 31) / 32 + 1);
      auto* host = static_cast<unsigned long long*>(ctx->pinned);
      try {
        enqueue_csr_validation(ctx, g, n, m, ctx->stream, err, rowstart, host);
        finish_csr_validation(ctx, g, ctx->stream, err, rowstart, host);
      } catch (...) {
        pool_free(ctx, rowstart);
        throw;
      }
      pool_free(ctx, rowstart);
    } catch (...) {
      destroy_graph(g);
      throw;
    }
    *out = g;
  });
}

dynpr_status dynpr_graph_build(dynpr_context* ctx, uint32_t n, const uint32_t* src,
                               const uint32_t* dst, uint64_t count, dynpr_graph** out) {
  return api_guard([&] {
    if (!ctx || !out) invalid("null argument");
    bind_device(ctx);
    const uint32_t* ds = stage_in(ctx, ctx->stage_a, src, count);
    const uint32_t* dd = stage_in(ctx, ctx->stage_b, dst, count);
    const bool host = count && !is_device_ptr(src);
    check_ids(ctx, ds, dd, count, n, "buildCsr", host ? src : nullptr, host ? dst : nullptr);
    *out = build_from_device_edges(ctx, n, ds, dd, count);
  });
}

dynpr_status dynpr_graph_add_self_loops(dynpr_context* ctx, const dynpr_graph* g,
                                        dynpr_graph** out) {
  return api_guard([&] {
    if (!ctx || !g || !out) invalid("null argument");
    bind_device(ctx);
    graph_apply_batch_impl(ctx, g, nullptr, nullptr, 0, nullptr, nullptr, 0, false, nullptr, nullptr,
                           nullptr, nullptr, out, nullptr, nullptr);
  });
}

dynpr_status dynpr_graph_transpose(dynpr_context* ctx, const dynpr_graph* g, dynpr_graph** out) {
  NvtxRange nvtx__("dynpr_graph_transpose");
  return api_guard([&] {
    if (!ctx || !g || !out) invalid("null argument");
    bind_device(ctx);
    const uint32_t n = g->n;
    const uint64_t m = g->m;
    dynpr_graph* t = make_graph(ctx, n, m);
    try {
      cudaStream_t st = ctx->stream;
      uint32_t* keys = ctx->stage_a.as<uint32_t>(m + 1);
      uint32_t* keys2 = ctx->stage_b.as<uint32_t>(m + 1);
      uint32_t* vals = reinterpret_cast<uint32_t*>(ctx->stage_c.as<uint32_t>(m + 1));
      if (m) {
        DYNPR_CK(cudaMemcpyAsync(keys, g->tgt, m * 4, cudaMemcpyDeviceToDevice, st));
        k_expand_sources<<<grid_for((uint64_t)n * 32, 256, 1 << 16), 256, 0, st>>>(g->off, n, vals);
        check_launch();
        count_launch(ctx);
        cub::DoubleBuffer<uint32_t> kb(keys, keys2);
        cub::DoubleBuffer<uint32_t> vb(vals, t->tgt);
        const int eb = key_shift(n);
        cub_call(ctx, [&](void* tmp, size_t& b) {
          return cub::DeviceRadixSort::SortPairs(tmp, b, kb, vb, m, 0, eb, st);
        });
        if (vb.Current() != t->tgt)
          DYNPR_CK(cudaMemcpyAsync(t->tgt, vb.Current(), m * 4, cudaMemcpyDeviceToDevice, st));
        k_offsets_from_keys32<<<grid_for(m + 1, 256, 1 << 16), 256, 0, st>>>(kb.Current(), m, n, t->off);
      } else {
        k_offsets_from_keys32<<<1, 256, 0, st>>>(keys, 0, n, t->off);
      }
      check_launch();
      count_launch(ctx);
      sync(ctx);
      t->all_loops = g->all_loops;
    } catch (...) {
      destroy_graph(t);
      throw;
    }
    *out = t;
  });
}

static dynpr_status apply_batch_common(dynpr_context* ctx, const dynpr_graph* gF,
                                       const dynpr_graph* gT, const uint32_t* ds,
                                       const uint32_t* dd, uint64_t nd, const uint32_t* is,
                                       const uint32_t* id, uint64_t ni, dynpr_graph** outF,
                                       dynpr_graph** outT, uint64_t* missing, uint64_t* duplicate) {
  return api_guard([&] {
    if (!ctx || !gF || !outF) invalid("null argument");
    bind_device(ctx);
    // The batch lists get dedicated buffers: stage_a..f are the ingest's own.
    const uint32_t* d_ds = stage_in(ctx, ctx->batch[0], ds, nd);
    const uint32_t* d_dd = stage_in(ctx, ctx->batch[1], dd, nd);
    const uint32_t* d_is = stage_in(ctx, ctx->batch[2], is, ni);
    const uint32_t* d_id = stage_in(ctx, ctx->batch[3], id, ni);
    const bool hd = nd && !is_device_ptr(ds), hi = ni && !is_device_ptr(is);
    // The new pair's engine layout can be derived from the parent's when the
    // parent pair has one (single-GPU layouts; both graphs carry every
    // self-loop, so only the batch's rows change): record the touched rows.
    const bool seeded = gT && gT->layout && !gT->layout->owned && gT->layout->gF_id == gF->id &&
                        gF->all_loops && gT->all_loops && gT->ctx == ctx && gF->ctx == ctx;
    auto seed = seeded ? std::make_shared<LayoutSeed>() : nullptr;
    if (seed) {
      seed->ctx = ctx;
      seed->parent = gT->layout;
    }
    dynpr_graph* f = nullptr;
    graph_apply_batch_impl(ctx, gF, d_ds, d_dd, nd, d_is, d_id, ni, true, hd ? ds : nullptr,
                           hd ? dd : nullptr, hi ? is : nullptr, hi ? id : nullptr, &f, missing,
                           duplicate, seed ? &seed->rows_F : nullptr, seed ? &seed->n_F : nullptr);
    if (gT) {
      dynpr_graph* t = nullptr;
      try {
        // reversed batch on the transpose (ids already validated)
        graph_apply_batch_impl(ctx, gT, d_dd, d_ds, nd, d_id, d_is, ni, false, nullptr, nullptr,
                               nullptr, nullptr, &t, nullptr, nullptr, seed ? &seed->rows_T : nullptr,
                               seed ? &seed->n_T : nullptr);
      } catch (...) {
        destroy_graph(f);
        throw;
      }
      if (seed) {
        seed->gF_id = f->id;
        t->seed = std::move(seed);
      }
      *outT = t;
    }
    *outF = f;
  });
}

dynpr_status dynpr_graph_apply_batch(dynpr_context* ctx, const dynpr_graph* g, const uint32_t* del_src,
                                     const uint32_t* del_dst, uint64_t n_del, const uint32_t* ins_src,
                                     const uint32_t* ins_dst, uint64_t n_ins, dynpr_graph** out,
                                     uint64_t* missing, uint64_t* duplicate) {
  NvtxRange nvtx__("dynpr_graph_apply_batch");
  return apply_batch_common(ctx, g, nullptr, del_src, del_dst, n_del, ins_src, ins_dst, n_ins, out,
                            nullptr, missing, duplicate);
}

dynpr_status dynpr_graph_apply_batch_pair(dynpr_context* ctx, const dynpr_graph* gF,
                                          const dynpr_graph* gT, const uint32_t* del_src,
                                          const uint32_t* del_dst, uint64_t n_del,
                                          const uint32_t* ins_src, const uint32_t* ins_dst,
                                          uint64_t n_ins, dynpr_graph** out_gF, dynpr_graph** out_gT,
                                          uint64_t* missing, uint64_t* duplicate) {
  NvtxRange nvtx__("dynpr_graph_apply_batch_pair");
  if (!gT || !out_gT) {
    set_last_error("null argument");
    return DYNPR_INVALID_ARGUMENT;
  }
  if (gT->n != gF->n || gT->m != gF->m) {
    set_last_error("engine: graph pair is not mutually transposed (count mismatch)");
    return DYNPR_INVALID_ARGUMENT;
  }
  return apply_batch_common(ctx, gF, gT, del_src, del_dst, n_del, ins_src, ins_dst, n_ins, out_gF,
                            out_gT, missing, duplicate);
}

dynpr_status dynpr_graph_info(const dynpr_graph* g, uint32_t* n, uint64_t* m) {
  return api_guard([&] {
    if (!g) invalid("null graph");
    if (n) *n = g->n;
    if (m) *m = g->m;
  });
}

dynpr_status dynpr_graph_download(dynpr_context* ctx, const dynpr_graph* g, uint64_t* offsets,
                                  uint32_t* targets) {
  return api_guard([&] {
    if (!ctx || !g) invalid("null argument");
    bind_device(ctx);
    if (offsets)
      DYNPR_CK(cudaMemcpyAsync(offsets, g->off, ((size_t)g->n + 1) * 8, cudaMemcpyDefault, ctx->stream));
    if (targets && g->m)
      DYNPR_CK(cudaMemcpyAsync(targets, g->tgt, g->m * 4, cudaMemcpyDefault, ctx->stream));
    sync(ctx);
  });
}

dynpr_status dynpr_graph_has_edge(dynpr_context* ctx, const dynpr_graph* g, uint32_t source,
                                  uint32_t target, int* out) {
  return api_guard([&] {
    if (!ctx || !g || !out) invalid("null argument");
    if (source >= g->n) invalid("hasEdge: source out of range");
    bind_device(ctx);
    int* d = reinterpret_cast<int*>(ctx->scratch64b.as<unsigned long long>(1));
    k_has_edge<<<1, 1, 0, ctx->stream>>>(g->off, g->tgt, source, target, d);
    check_launch();
    count_launch(ctx);
    DYNPR_CK(cudaMemcpyAsync(ctx->pinned, d, 4, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    std::memcpy(out, ctx->pinned, 4);
  });
}

dynpr_status dynpr_graph_destroy(dynpr_graph* g) {
  return api_guard([&] {
    if (g && g->ctx) cudaSetDevice(g->ctx->device);
    destroy_graph(g);
  });
}

dynpr_status dynpr_graph_rmat(dynpr_context* ctx, uint32_t scale, uint32_t edge_factor, double a,
                              double b, double c, uint64_t seed, dynpr_graph** out) {
  NvtxRange nvtx__("dynpr_graph_rmat");
  return api_guard([&] {
    if (!ctx || !out) invalid("null argument");
    if (scale < 1 || scale > 31) invalid("rmat: scale must be in [1,31]");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) invalid("rmat: bad probabilities");
    bind_device(ctx);
    const uint32_t n = 1u << scale;
    const uint64_t cnt = (uint64_t)edge_factor << scale;
    uint32_t* s = ctx->stage_a.as<uint32_t>(cnt + 1);
    uint32_t* d = ctx->stage_b.as<uint32_t>(cnt + 1);
    if (cnt) {
      k_rmat<<<grid_for(cnt, 256, 1 << 18), 256, 0, ctx->stream>>>(cnt, scale, a, a + b, a + b + c, seed, s,
                                                                   d);
      check_launch();
      count_launch(ctx);
    }
    dynpr_graph* raw = build_from_device_edges(ctx, n, s, d, cnt);
    // free the generator's staging before the self-loop pass needs memory
    dynpr_graph* looped = nullptr;
    try {
      graph_apply_batch_impl(ctx, raw, nullptr, nullptr, 0, nullptr, nullptr, 0, false, nullptr, nullptr,
                             nullptr, nullptr, &looped, nullptr, nullptr);
    } catch (...) {
      destroy_graph(raw);
      throw;
    }
    destroy_graph(raw);
    *out = looped;
  });
}

}  // extern "C"
