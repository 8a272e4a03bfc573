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

#include "common.cuh"
#include "layout.cuh"
#include "prims.cuh"

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

// Graph500-style vertex scrambling for the Kronecker generator: a seeded
// bijection of [0, 2^scale) (odd multiplications, an added constant and
// xor-shifts, all modulo 2^scale), so hub ids are spread over the id space
// instead of sitting at the small ids RMAT favours.
struct Scramble {
  uint64_t k1, k2, k3, mask;
  uint32_t sh1, sh2;
  __host__ __device__ uint32_t operator()(uint32_t x) const {
    uint64_t y = ((uint64_t)x * k1) & mask;
    y ^= y >> sh1;
    y = (y * k2 + k3) & mask;
    y ^= y >> sh2;
    return (uint32_t)y;
  }
};

// The keys of the bijection from the seed (SplitMix64 stream seeded with
// deriveSeed(seed, 2^40), rng.hpp:44-47); multipliers forced odd.
Scramble kronecker_scramble(uint32_t scale, uint64_t seed) {
  uint64_t st = seed ^ (0xD1B54A32D192ED03ULL * ((1ull << 40) + 1));
  auto next = [&st] {
    uint64_t z = (st += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  };
  st = next();  // deriveSeed(seed, 2^40): the stream's seed
  Scramble sc;
  sc.k1 = next() | 1ull;
  sc.k2 = next() | 1ull;
  sc.k3 = next();
  sc.mask = scale >= 64 ? ~0ull : (1ull << scale) - 1;
  sc.sh1 = (scale + 1) / 2;
  sc.sh2 = (scale + 2) / 3;
  return sc;
}

__global__ void k_rmat(uint64_t count, uint32_t scale, double t1, double t2,
                       double t3, uint64_t seed, uint32_t* src, uint32_t* dst, int scramble, Scramble sc) {
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
    src[i] = scramble ? sc(u) : u;
    dst[i] = scramble ? sc(v) : v;
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
// The ingest is two-phase (see graph_apply_batch_impl): phase A sorts and
// classifies the batch and derives the new offsets without a host round
// trip; one readback of an IngestStatus record then sizes the new target
// array and carries every validation result; phase B copies and merges.
// Per-vertex state (deletion / insertion counts, touched / loop / need
// flags) lives in context arrays that stay zero between ingests: phase B
// clears exactly the touched rows again, so no O(n) memset runs per batch.
struct IngestStatus {
  unsigned long long bad_del, bad_ins, self_del;  // first offending list index (kNone: none)
  unsigned long long overlap;                     // an edge both deleted and inserted
  unsigned long long missing, dup;                // deletions not present / insertions already present
  unsigned long long ndu, nu;                     // unique deletions / unique batch entries
  unsigned long long ndp, nnw;                    // present deletions / fresh insertions
  unsigned long long nt;                          // touched rows
  unsigned long long m_new;                       // edge count of the new snapshot
  unsigned long long nrd, nri, nrm;               // touched rows among the deletions / insertions / both
};

// Per-vertex ingest state of one CSR, zero between ingests.
struct VertexState {
  unsigned* ddel;
  unsigned* dins;
  uint8_t* touched;
  uint8_t* loop_ins;
  uint8_t* need;
};

__global__ void k_status_init(IngestStatus* s) {
  *s = IngestStatus{kNone, kNone, kNone, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
}

// graph.cpp:116-120: ids in range (both lists), no self-loop deletion; the
// first offending index of each kind.
__global__ void k_batch_check(const uint32_t* ds, const uint32_t* dd, uint64_t nd, const uint32_t* is,
                              const uint32_t* id, uint64_t ni, uint32_t n, IngestStatus* st) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nd + ni;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < nd) {
      const uint32_t u = ds[i], v = dd[i];
      if (u >= n || v >= n) atomicMin(&st->bad_del, (unsigned long long)i);
      if (u == v) atomicMin(&st->self_del, (unsigned long long)i);
    } else {
      const uint64_t k = i - nd;
      if (is[k] >= n || id[k] >= n) atomicMin(&st->bad_ins, (unsigned long long)k);
    }
  }
}

// Deletions then insertions as one key list: tag (0 / 1) above the packed
// (u, v).  Out-of-range ids (reported through the status) are clamped so
// the rest of phase A stays in bounds.
__global__ void k_pack_batch(const uint32_t* ds, const uint32_t* dd, uint64_t nd, const uint32_t* is,
                             const uint32_t* id, uint64_t ni, uint32_t n, int sb, uint64_t* keys) {
  const uint32_t top = n ? n - 1 : 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nd + ni;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const bool del = i < nd;
    uint32_t u = del ? ds[i] : is[i - nd], v = del ? dd[i] : id[i - nd];
    u = u < top ? u : top;
    v = v < top ? v : top;
    keys[i] = ((uint64_t)(del ? 0 : 1) << (2 * sb)) | ((uint64_t)u << sb) | v;
  }
}

__device__ __forceinline__ bool slice_has(const uint64_t* off, const uint32_t* tgt,
                                          uint32_t u, uint32_t v) {
  const uint64_t b = off[u], e = off[u + 1];
  const uint64_t p = lower_bound_dev<uint32_t, uint64_t>(tgt, b, e, v);
  return p < e && tgt[p] == v;
}

// Unique batch entries (graph.cpp:122-191): a deletion present in the graph
// shrinks its row, an absent one is missing; an insertion already present
// is a duplicate, a fresh one grows its row; an insertion that is also a
// deletion is the overlap error (graph.cpp:130-138).  keep[i] marks the
// entries the merge applies.
__global__ void k_batch_effect(const uint64_t* keys, const unsigned long long* nu_dev, int sb, const uint64_t* off,
                               const uint32_t* tgt, uint8_t* keep, VertexState vs, IngestStatus* st) {
  const uint64_t nu = *nu_dev;
  const uint64_t tag = 1ull << (2 * sb), mask = (1ull << sb) - 1;
  unsigned long long missing = 0, dup = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nu;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const bool ins = (k & tag) != 0;
    const uint32_t u = (uint32_t)((k >> sb) & mask), v = (uint32_t)(k & mask);
    if (!ins && (i + 1 == nu || (keys[i + 1] & tag))) st->ndu = i + 1;  // last deletion
    const bool present = slice_has(off, tgt, u, v);
    bool kp;
    if (!ins) {
      kp = present;
      if (present) {
        atomicAdd(vs.ddel + u, 1u);
        vs.touched[u] = 1;
      } else {
        ++missing;
      }
    } else {
      kp = !present;
      if (present) {
        ++dup;
      } else {
        atomicAdd(vs.dins + u, 1u);
        vs.touched[u] = 1;
        if (u == v) vs.loop_ins[u] = 1;
      }
      const uint64_t dk = k & ~tag;  // the same edge as a deletion?
      const uint64_t p = lower_bound_dev<uint64_t, uint64_t>(keys, 0, i, dk);
      if (p < i && keys[p] == dk) st->overlap = 1;
    }
    keep[i] = kp;
  }
  missing = warp_sum(missing);
  dup = warp_sum(dup);
  if ((threadIdx.x & 31) == 0) {
    if (missing) atomicAdd(&st->missing, missing);
    if (dup) atomicAdd(&st->dup, dup);
  }
}

// Vertices lacking their loop get one (graph.cpp:155-163,193).
__global__ void k_need_loop(const uint64_t* off, const uint32_t* tgt, uint32_t n, VertexState vs) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const bool nl = !vs.loop_ins[v] && !slice_has(off, tgt, (uint32_t)v, (uint32_t)v);
    if (nl) {
      vs.need[v] = 1;
      vs.touched[v] = 1;
    }
  }
}

// The merge lists: present deletions (tag 0, keep) / fresh insertions (tag
// 1, keep), untagged and still sorted.
struct KeepTag {
  const uint64_t* keys;
  const uint8_t* keep;
  uint64_t tag;
  bool ins;
  __device__ __forceinline__ bool operator()(uint64_t i) const {
    return keep[i] && (((keys[i] & tag) != 0) == ins);
  }
};
struct Untag {
  const uint64_t* keys;
  uint64_t tag;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return keys[i] & ~tag; }
};
// Touched rows from the batch (every row with a loop: only batch sources
// change): the first entry of each row within the sorted deletions
// [0, ndu) or the sorted insertions [ndu, nu), kept if the row changes.
struct RowHead {
  const uint64_t* keys;
  const unsigned long long* ndu;
  const uint8_t* touched;
  int sb;
  uint64_t mask;
  bool ins;
  __device__ __forceinline__ bool operator()(uint64_t i) const {
    const uint64_t d = *ndu;
    if (ins ? i < d : i >= d) return false;
    const uint32_t u = (uint32_t)((keys[i] >> sb) & mask);
    if (i != (ins ? d : 0ull) && (uint32_t)((keys[i - 1] >> sb) & mask) == u) return false;
    return touched[u] != 0;
  }
};
struct RowOf {
  const uint64_t* keys;
  int sb;
  uint64_t mask;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return (uint32_t)((keys[i] >> sb) & mask); }
};
// Merge of the two sorted touched-row lists (duplicates kept adjacent, the
// deletion side first); *nm = na + nb for the unique pass that follows.
__global__ void k_merge_row_lists(const uint32_t* A, const unsigned long long* na_d, const uint32_t* B,
                                  const unsigned long long* nb_d, uint32_t* out, unsigned long long* nm) {
  const uint64_t na = *na_d, nb = *nb_d;
  if (blockIdx.x == 0 && threadIdx.x == 0) *nm = na + nb;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < na + nb;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < na) {
      const uint32_t x = A[i];
      out[i + lower_bound_dev<uint32_t, uint64_t>(B, 0, nb, x)] = x;  // B entries < x
    } else {
      const uint32_t x = B[i - na];
      out[(i - na) + lower_bound_dev<uint32_t, uint64_t>(A, 0, na, x + 1)] = x;  // A entries <= x
    }
  }
}

// Row delta of the j-th touched row (0 past the list).
struct RowDelta {
  const uint32_t* T;
  const unsigned long long* nt;
  VertexState vs;
  __device__ __forceinline__ long long operator()(uint64_t j) const {
    if (j >= *nt) return 0;
    const uint32_t u = T[j];
    return (long long)vs.dins[u] + vs.need[u] - (long long)vs.ddel[u];
  }
};

// New offsets: noff[v] = off[v] + D[#touched rows < v].  Block per 2048
// vertices: cs[c] = #touched rows below chunk c (k_chunk_starts, one
// binary search per chunk), the chunk's touched rows (few) are staged in
// shared memory and each thread counts those below its vertex.
constexpr int kOffChunk = 2048;
__global__ void k_chunk_starts(const uint32_t* T, const unsigned long long* nt_dev, uint64_t nchunks, uint32_t* cs) {
  const uint64_t nt = *nt_dev;
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c <= nchunks;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = c * kOffChunk;
    uint64_t lo = 0, hi = nt;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (T[mid] < x) lo = mid + 1; else hi = mid;
    }
    cs[c] = (uint32_t)lo;
  }
}
__global__ void __launch_bounds__(256) k_new_offsets(const uint64_t* off, uint32_t n, const uint32_t* T,
                                                     const uint32_t* cs, const long long* D, uint64_t* noff,
                                                     IngestStatus* st) {
  __shared__ uint32_t s_t[kOffChunk];
  const uint64_t c0 = (uint64_t)blockIdx.x * kOffChunk;
  const uint64_t c1 = c0 + kOffChunk < (uint64_t)n + 1 ? c0 + kOffChunk : (uint64_t)n + 1;
  const uint32_t j0 = cs[blockIdx.x], k = cs[blockIdx.x + 1] - j0;  // <= kOffChunk (distinct rows)
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) s_t[i] = T[j0 + i];
  __syncthreads();
  for (uint64_t v = c0 + threadIdx.x; v < c1; v += blockDim.x) {
    uint32_t lo = 0, hi = k;  // staged rows < v
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_t[mid] < v) lo = mid + 1; else hi = mid;
    }
    const uint64_t o = (uint64_t)((long long)off[v] + D[j0 + lo]);
    noff[v] = o;
    if (v == n) st->m_new = o;
  }
}

// Phase B: clear the touched rows' state (the zero invariant).
__global__ void k_clear_rows(const uint32_t* T, uint64_t nt, VertexState vs) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nt;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = T[j];
    vs.ddel[u] = 0;
    vs.dins[u] = 0;
    vs.touched[u] = 0;
    vs.loop_ins[u] = 0;
    vs.need[u] = 0;
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
__global__ void k_run_pieces(const uint32_t* T, const unsigned long long* nt_ptr, uint64_t upper, uint32_t n,
                             const uint64_t* off, uint32_t* pieces) {
  const uint64_t nt = *nt_ptr;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < upper + 2;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (j <= nt) {
      const uint64_t a = j == 0 ? 0 : (uint64_t)T[j - 1] + 1;
      const uint64_t b = j == nt ? n : T[j];
      const uint64_t words = b > a ? off[b] - off[a] : 0;
      c = (uint32_t)((words + kRunPiece - 1) / kRunPiece);
    }
    pieces[j] = c;  // entries past nt stay 0: the exclusive scan at nt + 1 is the total
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

// The runs of untouched rows around the ascending touched-row list T (*nt_dev
// entries, at most nt_upper) copied from (off, tgt) to (noff, ntgt); pieces
// holds nt_upper + 3 words of workspace.
void copy_runs(dynpr_context* ctx, const uint32_t* T, const unsigned long long* nt_dev, uint64_t nt_upper, uint32_t n,
               const uint64_t* off, const uint32_t* tgt, const uint64_t* noff, uint32_t* ntgt, uint32_t* pieces) {
  cudaStream_t st = ctx->stream;
  k_run_pieces<<<grid_for(nt_upper + 2, 256, (unsigned)ctx->num_sms * 8), 256, 0, st>>>(T, nt_dev, nt_upper, n, off,
                                                                                       pieces);
  check_launch();
  prims::scan_array<uint32_t>(ctx, pieces, pieces, nt_upper + 2, st);
  k_copy_runs<<<(unsigned)ctx->num_sms * 32, 256, 0, st>>>(T, nt_dev, pieces, n, off, tgt, noff, ntgt);
  check_launch();
  count_launch(ctx, 2);
}

// Merge work items of the touched rows: a row of old degree d is split into
// max(1, ceil(d / kMergeChunk)) items so a touched hub (RMAT-24: ~4e5 edges)
// is spread over many warps instead of serialising one.
constexpr uint64_t kMergeChunk = 2048;
struct RowItems {
  const uint32_t* T;
  const uint64_t* off;
  uint64_t nt;
  __device__ __forceinline__ uint32_t operator()(uint64_t j) const {
    if (j >= nt) return 0;
    const uint64_t d = off[T[j] + 1] - off[T[j]];
    return d > kMergeChunk ? (uint32_t)((d + kMergeChunk - 1) / kMergeChunk) : 1u;
  }
};

// Touched rows: every surviving old target and every fresh insertion is
// written at its final position (old index - deletions before it +
// insertions before it + the re-ensured self-loop when it precedes), so
// the items of one row are independent.  Item t -> touched row j through
// the exclusive scan `istart` (nt + 1 entries).  Old targets are loaded
// kMergeIlp at a time per lane (independent loads in flight; the searches
// in the row's few batch entries then run on registers).
constexpr int kMergeIlp = 8;
__global__ void k_merge_touched(const uint32_t* istart, const uint32_t* T, uint64_t nt, const uint64_t* off,
                                const uint32_t* tgt, const uint64_t* noff, uint32_t* ntgt, const uint64_t* dp,
                                const unsigned long long* ndp_dev, const uint64_t* nw,
                                const unsigned long long* nnw_dev, int sb, uint64_t mask, const uint8_t* need) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x / 32;
  const uint32_t total = istart[nt];
  const uint64_t ndp = *ndp_dev, nnw = *nnw_dev;
  for (uint64_t t = warp; t < total; t += nwarps) {
    const uint64_t j = upper_bound_u32(istart, nt + 1, (uint32_t)t) - 1;
    const uint32_t u = T[j];
    const uint64_t c = t - istart[j];
    const uint64_t so = off[u], se = off[u + 1], base = noff[u];
    const uint64_t cb = so + c * kMergeChunk, ce = cb + kMergeChunk < se ? cb + kMergeChunk : se;
    const uint64_t klo = (uint64_t)u << sb, khi = ((uint64_t)u + 1) << sb;
    const uint64_t dlo = lower_bound_dev<uint64_t, uint64_t>(dp, 0, ndp, klo);
    const uint64_t dhi = lower_bound_dev<uint64_t, uint64_t>(dp, dlo, ndp, khi);
    const uint64_t nlo = lower_bound_dev<uint64_t, uint64_t>(nw, 0, nnw, klo);
    const uint64_t nhi = lower_bound_dev<uint64_t, uint64_t>(nw, nlo, nnw, khi);
    const bool nl = need[u];
    // the batch entries inside the chunk's value range (usually none)
    const uint64_t kf = cb < ce ? (klo | tgt[cb]) : klo, kl = cb < ce ? (klo | tgt[ce - 1]) + 1 : klo;
    const uint64_t d0 = lower_bound_dev<uint64_t, uint64_t>(dp, dlo, dhi, kf);
    const uint64_t d1 = lower_bound_dev<uint64_t, uint64_t>(dp, d0, dhi, kl);
    const uint64_t n0 = lower_bound_dev<uint64_t, uint64_t>(nw, nlo, nhi, kf);
    const uint64_t n1 = lower_bound_dev<uint64_t, uint64_t>(nw, n0, nhi, kl);
    for (uint64_t k0 = cb; k0 < ce; k0 += 32 * kMergeIlp) {
      uint32_t x[kMergeIlp];
#pragma unroll
      for (int q = 0; q < kMergeIlp; ++q) {
        const uint64_t k = k0 + 32 * q + lane;
        x[q] = k < ce ? tgt[k] : 0u;
      }
#pragma unroll
      for (int q = 0; q < kMergeIlp; ++q) {
        const uint64_t k = k0 + 32 * q + lane;
        if (k >= ce) continue;
        const uint64_t key = klo | x[q];
        const uint64_t qd = d1 > d0 ? lower_bound_dev<uint64_t, uint64_t>(dp, d0, d1, key) : d0;
        if (qd < d1 && dp[qd] == key) continue;
        const uint64_t r = (n1 > n0 ? lower_bound_dev<uint64_t, uint64_t>(nw, n0, n1, key) : n0) - nlo;
        ntgt[base + (k - so) - (qd - dlo) + r + ((nl && u < x[q]) ? 1 : 0)] = x[q];
      }
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

// Sorts + dedupes packed keys (end_bit significant bits); returns the unique
// count (keys end in `*out`, one of the two buffers).
uint64_t sort_unique(dynpr_context* ctx, uint64_t* keys, uint64_t* alt, uint64_t cnt, int end_bit, uint64_t** out) {
  if (cnt == 0) {
    *out = keys;
    return 0;
  }
  uint64_t* sorted = prims::radix_sort<uint64_t, uint32_t>(ctx, keys, alt, nullptr, nullptr, cnt, 0, end_bit,
                                                           ctx->stream);
  uint64_t* uniq = sorted == keys ? alt : keys;
  auto* num = ctx->scratch64a.as<unsigned long long>(1);
  prims::unique_sorted<uint64_t>(ctx, sorted, cnt, uniq, num, ctx->stream);
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

namespace {

// Device temporaries of one CSR's ingest, carved from one pool block.
struct IngestPlan {
  const dynpr_graph* g = nullptr;
  dynpr_graph* r = nullptr;
  uint32_t n = 0;
  int sb = 1;
  uint64_t nd = 0, ni = 0, nb = 0, t_cap = 0;
  VertexState vs{};
  void* block = nullptr;
  uint64_t *keys = nullptr, *keys2 = nullptr, *ukeys = nullptr, *dp = nullptr, *nw = nullptr;
  uint8_t* keep = nullptr;
  uint32_t *T = nullptr, *pieces = nullptr, *istart = nullptr, *cs = nullptr;
  long long* D = nullptr;
  IngestStatus* st = nullptr;   // device
  IngestStatus* host = nullptr; // pinned readback slot
};

template <class T>
T* carve(char*& p, uint64_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += ((count * sizeof(T) + 255) / 256) * 256;
  return r;
}

// Per-vertex ingest state `set` (0: the forward CSR, 1: the transpose of a
// pair): zeroed when (re)allocated, kept zero by phase B.
VertexState vertex_state(dynpr_context* ctx, int set, uint32_t n) {
  DevBuf& b = ctx->ingest_state[set];
  const uint64_t words = (uint64_t)n + 1;
  const size_t need = words * (4 + 4 + 1 + 1 + 1) + 64;
  void* before = b.p;
  const size_t cap_before = b.cap;
  char* p = static_cast<char*>(b.ensure(need));
  if (p != before || cap_before < need) DYNPR_CK(cudaMemsetAsync(p, 0, b.cap, ctx->stream));
  VertexState vs;
  vs.ddel = reinterpret_cast<unsigned*>(p);
  vs.dins = vs.ddel + words;
  vs.touched = reinterpret_cast<uint8_t*>(vs.dins + words);
  vs.loop_ins = vs.touched + words;
  vs.need = vs.loop_ins + words;
  return vs;
}

// Phase A: validation (optional), sort + unique + classification of the
// batch, touched rows, their deltas and the new offsets; ends with the
// status record copied to its pinned slot (no host wait).
void ingest_phase_a(dynpr_context* ctx, IngestPlan& P, const dynpr_graph* g, int set, const uint32_t* ds,
                    const uint32_t* dd, uint64_t nd, const uint32_t* is, const uint32_t* id, uint64_t ni,
                    bool validate, IngestStatus* host_slot) {
  cudaStream_t st = ctx->stream;
  const uint32_t n = g->n;
  P.g = g;
  P.n = n;
  P.sb = key_shift(n);
  if (2 * P.sb + 1 > 64) invalid("applyBatch: vertex ids too wide for the batch keys");
  P.nd = nd;
  P.ni = ni;
  P.nb = nd + ni;
  P.vs = vertex_state(ctx, set, n);
  // touched rows: batch sources, plus every row lacking its loop
  P.t_cap = g->all_loops ? (P.nb < (uint64_t)n ? P.nb : (uint64_t)n) : (uint64_t)n;
  const uint64_t nb1 = P.nb + 1, t1 = P.t_cap + 2;
  const uint64_t nchunks1 = ((uint64_t)n + 1 + kOffChunk - 1) / kOffChunk + 1;
  const size_t bytes = 5 * (((nb1 * 8) + 255) / 256) * 256 + ((nb1 + 255) / 256) * 256 +
                       2 * (((t1 * 4) + 255) / 256) * 256 + (((t1 + 1) * 4 + 255) / 256) * 256 +
                       (((t1 * 8) + 255) / 256) * 256 + ((nchunks1 * 4 + 255) / 256) * 256 + 256;
  P.block = pool_alloc(ctx, bytes);
  char* p = static_cast<char*>(P.block);
  P.keys = carve<uint64_t>(p, nb1);
  P.keys2 = carve<uint64_t>(p, nb1);
  P.ukeys = carve<uint64_t>(p, nb1);
  P.dp = carve<uint64_t>(p, nb1);
  P.nw = carve<uint64_t>(p, nb1);
  P.keep = carve<uint8_t>(p, nb1);
  P.T = carve<uint32_t>(p, t1);
  P.istart = carve<uint32_t>(p, t1);
  P.pieces = carve<uint32_t>(p, t1 + 1);
  P.D = carve<long long>(p, t1);
  P.cs = carve<uint32_t>(p, nchunks1);
  P.st = carve<IngestStatus>(p, 1);
  P.host = host_slot;
  k_status_init<<<1, 1, 0, st>>>(P.st);
  if (validate && P.nb) {
    k_batch_check<<<grid_for(P.nb, 256, 4096), 256, 0, st>>>(ds, dd, nd, is, id, ni, n, P.st);
  }
  const uint64_t tag = 1ull << (2 * P.sb);
  unsigned long long* nu = &P.st->nu;
  if (P.nb) {
    k_pack_batch<<<grid_for(P.nb, 256, 4096), 256, 0, st>>>(ds, dd, nd, is, id, ni, n, P.sb, P.keys);
    uint64_t* sorted = prims::radix_sort<uint64_t, uint32_t>(ctx, P.keys, P.keys2, nullptr, nullptr, P.nb, 0,
                                                             2 * P.sb + 1, st);
    prims::unique_sorted<uint64_t>(ctx, sorted, P.nb, P.ukeys, nu, st);
    k_batch_effect<<<grid_for(P.nb, 256, 4096), 256, 0, st>>>(P.ukeys, nu, P.sb, g->off, g->tgt, P.keep, P.vs,
                                                              P.st);
    count_launch(ctx, 2);
  }
  if (!g->all_loops && n) {
    k_need_loop<<<grid_for(n, 256, 1 << 16), 256, 0, st>>>(g->off, g->tgt, n, P.vs);
    count_launch(ctx);
  }
  check_launch();
  unsigned long long* nt = &P.st->nt;
  if (P.t_cap && g->all_loops) {
    // O(batch): the rows the batch changes, from its sorted keys (the
    // deletion and insertion runs merged, then deduplicated) -- not a
    // selection over all n vertices (Kronecker-27: ~0.3 ms per CSR)
    const uint64_t mask = (1ull << P.sb) - 1;
    auto* A = reinterpret_cast<uint32_t*>(P.keys);  // (free after the sort + unique)
    uint32_t* B = A + nb1;
    auto* Mg = reinterpret_cast<uint32_t*>(P.keys2);
    prims::select_if<uint32_t>(ctx, RowHead{P.ukeys, &P.st->ndu, P.vs.touched, P.sb, mask, false},
                               RowOf{P.ukeys, P.sb, mask}, P.nb, A, &P.st->nrd, st, nu);
    prims::select_if<uint32_t>(ctx, RowHead{P.ukeys, &P.st->ndu, P.vs.touched, P.sb, mask, true},
                               RowOf{P.ukeys, P.sb, mask}, P.nb, B, &P.st->nri, st, nu);
    k_merge_row_lists<<<grid_for(P.nb, 256, 4096), 256, 0, st>>>(A, &P.st->nrd, B, &P.st->nri, Mg, &P.st->nrm);
    check_launch();
    count_launch(ctx);
    prims::unique_sorted<uint32_t>(ctx, Mg, 2 * P.nb, P.T, nt, st, &P.st->nrm);
  } else if (P.t_cap) {
    prims::select_if<uint32_t>(ctx, prims::Nonzero<uint8_t>{P.vs.touched}, prims::Iota32{}, n, P.T, nt, st);
  }
  if (P.nb) {
    prims::select_if<uint64_t>(ctx, KeepTag{P.ukeys, P.keep, tag, false}, Untag{P.ukeys, tag}, P.nb, P.dp,
                               &P.st->ndp, st, nu);
    prims::select_if<uint64_t>(ctx, KeepTag{P.ukeys, P.keep, tag, true}, Untag{P.ukeys, tag}, P.nb, P.nw,
                               &P.st->nnw, st, nu);
  }
  // D[j] = sum of the deltas of touched rows 0..j-1 (j <= nt)
  prims::scan_exclusive<long long>(ctx, RowDelta{P.T, nt, P.vs}, P.D, P.t_cap + 1, st);
  P.r = new_graph_struct(ctx, n);
  P.r->off = pool_alloc_n<uint64_t>(ctx, (uint64_t)n + 1);
  const uint64_t nchunks = ((uint64_t)n + 1 + kOffChunk - 1) / kOffChunk;
  k_chunk_starts<<<grid_for(nchunks + 1, 256, 4096), 256, 0, st>>>(P.T, nt, nchunks, P.cs);
  k_new_offsets<<<(unsigned)nchunks, 256, 0, st>>>(g->off, n, P.T, P.cs, P.D, P.r->off, P.st);
  check_launch();
  count_launch(ctx, 2);
  DYNPR_CK(cudaMemcpyAsync(P.host, P.st, sizeof(IngestStatus), cudaMemcpyDeviceToHost, st));
}

// Phase B: the new targets -- runs of untouched rows copied, touched rows
// merged -- and the per-vertex state cleared again.
void ingest_phase_b(dynpr_context* ctx, IngestPlan& P, uint32_t** rows_out, uint64_t* nrows_out) {
  cudaStream_t st = ctx->stream;
  const IngestStatus& h = *P.host;
  dynpr_graph* r = P.r;
  r->m = h.m_new;
  r->tgt = pool_alloc_n<uint32_t>(ctx, r->m ? r->m : 1);
  const uint64_t nt = h.nt;
  copy_runs(ctx, P.T, &P.st->nt, nt, P.n, P.g->off, P.g->tgt, r->off, r->tgt, P.pieces);
  if (nt) {
    prims::scan_exclusive<uint32_t>(ctx, RowItems{P.T, P.g->off, nt}, P.istart, nt + 1, st);
    const uint64_t mask = (1ull << P.sb) - 1;
    k_merge_touched<<<(unsigned)ctx->num_sms * 16, 256, 0, st>>>(P.istart, P.T, nt, P.g->off, P.g->tgt, r->off,
                                                                  r->tgt, P.dp, &P.st->ndp, P.nw, &P.st->nnw, P.sb,
                                                                  mask, P.vs.need);
    k_clear_rows<<<grid_for(nt, 256, 4096), 256, 0, st>>>(P.T, nt, P.vs);
    check_launch();
    count_launch(ctx, 2);
  }
  if (rows_out) {  // the touched rows, for an incremental engine layout (layout.cu)
    uint32_t* rows = pool_alloc_n<uint32_t>(ctx, nt ? nt : 1);
    if (nt) DYNPR_CK(cudaMemcpyAsync(rows, P.T, nt * 4, cudaMemcpyDeviceToDevice, st));
    *rows_out = rows;
    *nrows_out = nt;
  }
  r->all_loops = true;
  pool_free(ctx, P.block);
  P.block = nullptr;
}

// Error path: the result (if any) and the temporaries freed, and the
// per-vertex state zeroed wholesale (phase A may have marked rows that no
// readback listed).
void ingest_abort(dynpr_context* ctx, IngestPlan& P, int set) {
  if (P.r) destroy_graph(P.r);
  P.r = nullptr;
  if (P.block) pool_free(ctx, P.block);
  P.block = nullptr;
  DevBuf& b = ctx->ingest_state[set];
  if (b.p) cudaMemsetAsync(b.p, 0, b.cap, ctx->stream);
  cudaGetLastError();
}

// The reference's error order (graph.cpp:116-138), from the status record.
void ingest_throw_if_invalid(dynpr_context* ctx, const IngestStatus& h, const uint32_t* d_ds, const uint32_t* d_dd,
                             const uint32_t* d_is, const uint32_t* d_id, const uint32_t* h_ds, const uint32_t* h_dd,
                             const uint32_t* h_is, const uint32_t* h_id, uint32_t n) {
  auto bad = [&](const char* what, const uint32_t* ds, const uint32_t* dd, const uint32_t* hs, const uint32_t* hd,
                 unsigned long long i) {
    auto [u, v] = fetch_pair(ctx, ds, dd, hs, hd, i);
    invalid(std::string(what) + ": vertex id out of range (" + std::to_string(u) + "," + std::to_string(v) +
            ") for |V|=" + std::to_string(n));
  };
  if (h.bad_del != kNone) bad("applyBatch deletions", d_ds, d_dd, h_ds, h_dd, h.bad_del);
  if (h.bad_ins != kNone) bad("applyBatch insertions", d_is, d_id, h_is, h_id, h.bad_ins);
  if (h.self_del != kNone) invalid("applyBatch: self-loops cannot be deleted");
  if (h.overlap) invalid("applyBatch: edge appears in both deletions and insertions");
}

}  // namespace

// applyBatch of one CSR or of a mutually transposed pair (the transpose
// receives the reversed batch, ids already validated through the first):
// both phase A's, ONE host wait for both status records, both phase B's.
void graph_apply_batch_multi(dynpr_context* ctx, int count, const dynpr_graph* const* gs,
                             const uint32_t* const* ds, const uint32_t* const* dd, uint64_t nd,
                             const uint32_t* const* is, const uint32_t* const* id, uint64_t ni, bool validate,
                             const uint32_t* h_ds, const uint32_t* h_dd, const uint32_t* h_is,
                             const uint32_t* h_id, dynpr_graph** outs, uint64_t* missing_out,
                             uint64_t* duplicate_out, uint32_t** rows_out, uint64_t* nrows_out) {
  IngestPlan P[2];
  auto* slots = reinterpret_cast<IngestStatus*>(static_cast<char*>(ctx->pinned) + 4096);
  static_assert(2 * sizeof(IngestStatus) <= 1024, "pinned status slots");
  try {
    for (int c = 0; c < count; ++c)
      ingest_phase_a(ctx, P[c], gs[c], c, ds[c], dd[c], nd, is[c], id[c], ni, validate && c == 0, slots + c);
    sync(ctx);
    if (validate) ingest_throw_if_invalid(ctx, *P[0].host, ds[0], dd[0], is[0], id[0], h_ds, h_dd, h_is, h_id,
                                          gs[0]->n);
    for (int c = 0; c < count; ++c)
      ingest_phase_b(ctx, P[c], rows_out ? rows_out + c : nullptr, nrows_out ? nrows_out + c : nullptr);
  } catch (...) {
    for (int c = 0; c < count; ++c) ingest_abort(ctx, P[c], c);
    throw;
  }
  const IngestStatus& h = *P[0].host;
  if (missing_out) *missing_out += (nd - h.ndu) + h.missing;
  if (duplicate_out) *duplicate_out += (ni - (h.nu - h.ndu)) + h.dup;
  for (int c = 0; c < count; ++c) {
    outs[c] = P[c].r;
    P[c].r = nullptr;
  }
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
  graph_apply_batch_multi(ctx, 1, &g, &d_ds, &d_dd, nd, &d_is, &d_id, ni, validate, h_ds, h_dd, h_is, h_id, out,
                          missing_out, duplicate_out, rows_out, nrows_out);
  sync(ctx);
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
        const int eb = key_shift(n);
        uint32_t* vsorted = nullptr;
        uint32_t* ksorted = prims::radix_sort<uint32_t, uint32_t>(ctx, keys, keys2, vals, t->tgt, m, 0, eb, st,
                                                                  &vsorted);
        if (vsorted != t->tgt) DYNPR_CK(cudaMemcpyAsync(t->tgt, vsorted, m * 4, cudaMemcpyDeviceToDevice, st));
        k_offsets_from_keys32<<<grid_for(m + 1, 256, 1 << 16), 256, 0, st>>>(ksorted, m, n, t->off);
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
    // forward + transpose (reversed batch, ids validated through the
    // forward): both phase A's, one host wait, both phase B's
    const int cnt = gT ? 2 : 1;
    const dynpr_graph* gs[2] = {gF, gT};
    const uint32_t* ls[2] = {d_ds, d_dd};
    const uint32_t* ld[2] = {d_dd, d_ds};
    const uint32_t* lis[2] = {d_is, d_id};
    const uint32_t* lid[2] = {d_id, d_is};
    dynpr_graph* outs[2] = {nullptr, nullptr};
    uint32_t* rows[2] = {nullptr, nullptr};
    uint64_t nrows[2] = {0, 0};
    graph_apply_batch_multi(ctx, cnt, gs, ls, ld, nd, lis, lid, ni, true, hd ? ds : nullptr, hd ? dd : nullptr,
                            hi ? is : nullptr, hi ? id : nullptr, outs, missing, duplicate, seed ? rows : nullptr,
                            seed ? nrows : nullptr);
    sync(ctx);  // calls are synchronous on return (the C-ABI contract)
    dynpr_graph* f = outs[0];
    if (gT) {
      dynpr_graph* t = outs[1];
      if (seed) {
        seed->rows_F = rows[0];
        seed->n_F = nrows[0];
        seed->rows_T = rows[1];
        seed->n_T = nrows[1];
        seed->gF_id = f->id;
        t->seed = std::move(seed);
      }
      *outT = t;
    } else if (seed) {
      pool_free(ctx, rows[0]);
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

// Unit-test entry for the device primitives (prims.cuh) on host arrays.
dynpr_status dynpr_debug_prims(dynpr_context* ctx, int op, const void* in, const void* in2, uint64_t count,
                               int bits, void* out, void* out2, uint64_t* out_count) {
  return api_guard([&] {
    if (!ctx) invalid("null context");
    bind_device(ctx);
    cudaStream_t st = ctx->stream;
    const uint64_t c1 = count ? count : 1;
    auto up = [&](const void* h, size_t bytes) {
      void* d = pool_alloc(ctx, bytes ? bytes : 16);
      if (bytes) DYNPR_CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
      return d;
    };
    std::vector<void*> held;
    auto hold = [&](void* p) { held.push_back(p); return p; };
    try {
      auto* num = ctx->scratch64a.as<unsigned long long>(1);
      uint64_t n_out = count;
      switch (op) {
        case 0: {  // radix sort of u64 keys on bits [0, bits)
          auto* k = static_cast<uint64_t*>(hold(up(in, count * 8)));
          auto* k2 = static_cast<uint64_t*>(hold(pool_alloc(ctx, c1 * 8)));
          uint64_t* r = prims::radix_sort<uint64_t, uint32_t>(ctx, k, k2, nullptr, nullptr, count, 0, bits, st);
          if (count) DYNPR_CK(cudaMemcpyAsync(out, r, count * 8, cudaMemcpyDeviceToHost, st));
          break;
        }
        case 1: {  // radix sort of (u32 key, u32 value) pairs on bits [0, bits)
          auto* k = static_cast<uint32_t*>(hold(up(in, count * 4)));
          auto* v = static_cast<uint32_t*>(hold(up(in2, count * 4)));
          auto* k2 = static_cast<uint32_t*>(hold(pool_alloc(ctx, c1 * 4)));
          auto* v2 = static_cast<uint32_t*>(hold(pool_alloc(ctx, c1 * 4)));
          uint32_t* vo = nullptr;
          uint32_t* r = prims::radix_sort<uint32_t, uint32_t>(ctx, k, k2, v, v2, count, 0, bits, st, &vo);
          if (count) {
            DYNPR_CK(cudaMemcpyAsync(out, r, count * 4, cudaMemcpyDeviceToHost, st));
            DYNPR_CK(cudaMemcpyAsync(out2, vo, count * 4, cudaMemcpyDeviceToHost, st));
          }
          break;
        }
        case 2: {  // exclusive scan of u64, total in *out_count
          auto* a = static_cast<uint64_t*>(hold(up(in, count * 8)));
          prims::scan_array<uint64_t>(ctx, a, a, count, st, reinterpret_cast<uint64_t*>(num));
          if (count) DYNPR_CK(cudaMemcpyAsync(out, a, count * 8, cudaMemcpyDeviceToHost, st));
          n_out = read_u64(ctx, num);
          break;
        }
        case 3: {  // indices of the nonzero bytes
          auto* f = static_cast<uint8_t*>(hold(up(in, count)));
          auto* o = static_cast<uint32_t*>(hold(pool_alloc(ctx, c1 * 4)));
          prims::select_if<uint32_t>(ctx, prims::Nonzero<uint8_t>{f}, prims::Iota32{}, count, o, num, st);
          n_out = read_u64(ctx, num);
          if (n_out) DYNPR_CK(cudaMemcpyAsync(out, o, n_out * 4, cudaMemcpyDeviceToHost, st));
          break;
        }
        case 4: {  // unique of sorted u64
          auto* k = static_cast<uint64_t*>(hold(up(in, count * 8)));
          auto* o = static_cast<uint64_t*>(hold(pool_alloc(ctx, c1 * 8)));
          prims::unique_sorted<uint64_t>(ctx, k, count, o, num, st);
          n_out = read_u64(ctx, num);
          if (n_out) DYNPR_CK(cudaMemcpyAsync(out, o, n_out * 8, cudaMemcpyDeviceToHost, st));
          break;
        }
        default:
          invalid("dynpr_debug_prims: unknown op");
      }
      sync(ctx);
      if (out_count) *out_count = n_out;
    } catch (...) {
      for (void* p : held) pool_free(ctx, p);
      throw;
    }
    for (void* p : held) pool_free(ctx, p);
  });
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

static void generate_rmat(dynpr_context* ctx, uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                          uint64_t seed, bool scramble, dynpr_graph** out) {
  if (!ctx || !out) invalid("null argument");
  if (scale < 1 || scale > 31) invalid("rmat: scale must be in [1,31]");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) invalid("rmat: bad probabilities");
  bind_device(ctx);
  const uint32_t n = 1u << scale;
  const uint64_t cnt = (uint64_t)edge_factor << scale;
  uint32_t* s = ctx->stage_a.as<uint32_t>(cnt + 1);
  uint32_t* d = ctx->stage_b.as<uint32_t>(cnt + 1);
  Scramble sc = kronecker_scramble(scale, seed);
  if (cnt) {
    k_rmat<<<grid_for(cnt, 256, 1 << 18), 256, 0, ctx->stream>>>(cnt, scale, a, a + b, a + b + c, seed, s, d,
                                                                 scramble ? 1 : 0, sc);
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
}

dynpr_status dynpr_graph_rmat(dynpr_context* ctx, uint32_t scale, uint32_t edge_factor, double a,
                              double b, double c, uint64_t seed, dynpr_graph** out) {
  NvtxRange nvtx__("dynpr_graph_rmat");
  return api_guard([&] { generate_rmat(ctx, scale, edge_factor, a, b, c, seed, false, out); });
}

dynpr_status dynpr_graph_kronecker(dynpr_context* ctx, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                                   dynpr_graph** out) {
  NvtxRange nvtx__("dynpr_graph_kronecker");
  return api_guard([&] { generate_rmat(ctx, scale, edge_factor, 0.57, 0.19, 0.19, seed, true, out); });
}

}  // extern "C"
