/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Never linked into the product path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * the shared library built from this file (oracle/_build/libdynpr_oracle.so).
 *
 * A sequential plain-C restatement of the reference `dynpr` hot path
 * (/root/reference/proj/src), function by function, each citing the
 * reference file:line it follows.  It reproduces the reference's arithmetic
 * order exactly (flat sums for in-degree <= D_P, 256-edge chunked partial sums
 * above it, no FMA contraction), so its ranks are bit-identical to the
 * reference library's.  Parity of this restatement is PINNED two ways by
 * tests/test_oracle.py: against the golden vectors in tests/golden/ (generated
 * from the reference itself by tests/golden/make_golden.py) and, where
 * oracle/_ref is built, against the reference library directly.
 *
 * Vertex ids uint32, offsets uint64, ranks double, flags uint8
 * (graph.hpp:9,47-48, frontier.hpp:16-17).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dynpr_cuda.h" /* POD dynpr_config / dynpr_stats / dynpr_observer */

static _Thread_local char g_err[512];
static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* orc_last_error(void) { return g_err; }

/* ---- rng.hpp:10-47 ------------------------------------------------------ */
typedef struct { uint64_t state; } orc_rng;
static uint64_t rng_next(orc_rng* r) { /* rng.hpp:14-19 */
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t rng_bounded(orc_rng* r, uint64_t bound) { /* rng.hpp:22-34 */
  unsigned __int128 m = (unsigned __int128)rng_next(r) * bound;
  uint64_t low = (uint64_t)m;
  if (low < bound) {
    const uint64_t threshold = (0 - bound) % bound;
    while (low < threshold) {
      m = (unsigned __int128)rng_next(r) * bound;
      low = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}
static double rng_double(orc_rng* r) { /* rng.hpp:37 */
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) { /* rng.hpp:44-47 */
  orc_rng r = {seed ^ (0xD1B54A32D192ED03ULL * (stream + 1))};
  return rng_next(&r);
}
uint64_t orc_rng_next(uint64_t* state) {
  orc_rng r = {*state};
  uint64_t x = rng_next(&r);
  *state = r.state;
  return x;
}
uint64_t orc_rng_bounded(uint64_t* state, uint64_t bound) {
  orc_rng r = {*state};
  uint64_t x = rng_bounded(&r, bound);
  *state = r.state;
  return x;
}
double orc_rng_double(uint64_t* state) {
  orc_rng r = {*state};
  double x = rng_double(&r);
  *state = r.state;
  return x;
}

/* ---- CsrGraph (graph.hpp:17-49) ---------------------------------------- */
typedef struct {
  uint32_t n;
  uint64_t m;
  uint64_t* off; /* n+1 */
  uint32_t* tgt; /* m */
} orc_graph;

static orc_graph* graph_alloc(uint32_t n, uint64_t m) {
  orc_graph* g = (orc_graph*)calloc(1, sizeof *g);
  g->n = n;
  g->m = m;
  g->off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  g->tgt = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
  return g;
}
void orc_graph_free(orc_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->tgt);
  free(g);
}
void orc_graph_info(const orc_graph* g, uint32_t* n, uint64_t* m) {
  *n = g->n;
  *m = g->m;
}
void orc_graph_download(const orc_graph* g, uint64_t* off, uint32_t* tgt) {
  memcpy(off, g->off, ((size_t)g->n + 1) * sizeof(uint64_t));
  if (g->m) memcpy(tgt, g->tgt, g->m * sizeof(uint32_t));
}
static uint32_t degree(const orc_graph* g, uint32_t v) { /* graph.hpp:28-30 */
  return (uint32_t)(g->off[v + 1] - g->off[v]);
}
static int has_edge(const orc_graph* g, uint32_t s, uint32_t t) {
  /* graph.cpp:51-54 binary search */
  uint64_t lo = g->off[s], hi = g->off[s + 1];
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (g->tgt[mid] < t) lo = mid + 1; else hi = mid;
  }
  return lo < g->off[s + 1] && g->tgt[lo] == t;
}
int orc_has_edge(const orc_graph* g, uint32_t s, uint32_t t) {
  return has_edge(g, s, t);
}

/* CsrGraph ctor validation (graph.cpp:30-49). */
int orc_graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt,
                       uint64_t m, orc_graph** out) {
  if (off[0] != 0 || off[n] != m)
    return set_err(1, "CsrGraph: malformed offsets array");
  for (uint32_t v = 0; v < n; ++v) {
    if (off[v] > off[v + 1])
      return set_err(1, "CsrGraph: offsets must be non-decreasing");
    for (uint64_t i = off[v]; i < off[v + 1]; ++i) {
      if (tgt[i] >= n) return set_err(1, "CsrGraph: target id out of range");
      if (i > off[v] && tgt[i - 1] >= tgt[i])
        return set_err(1,
                       "CsrGraph: target slices must be sorted and deduplicated");
    }
  }
  orc_graph* g = graph_alloc(n, m);
  memcpy(g->off, off, ((size_t)n + 1) * sizeof(uint64_t));
  if (m) memcpy(g->tgt, tgt, m * sizeof(uint32_t));
  *out = g;
  return 0;
}

/* LSD radix sort of 64-bit keys (stand-in for std::sort, graph.cpp:22-26:
 * sorting (u,v) pairs lexicographically == sorting u<<32|v). */
static void radix_sort_u64(uint64_t* a, uint64_t n) {
  if (n < 2) return;
  uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t* src = a;
  uint64_t* dst = tmp;
  for (int shift = 0; shift < 64; shift += 16) {
    uint64_t* cnt = (uint64_t*)calloc(65537, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) cnt[((src[i] >> shift) & 0xFFFF) + 1]++;
    for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
    for (uint64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & 0xFFFF]++] = src[i];
    free(cnt);
    uint64_t* t = src; src = dst; dst = t;
  }
  /* 4 passes: result back in `a` */
  free(tmp);
}
static uint64_t sorted_unique(uint64_t* keys, uint64_t n) {
  radix_sort_u64(keys, n);
  uint64_t w = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (w == 0 || keys[w - 1] != keys[i]) keys[w++] = keys[i];
  return w;
}

static int check_ids(const uint32_t* s, const uint32_t* d, uint64_t count,
                     uint32_t n, const char* what) { /* graph.cpp:13-20 */
  for (uint64_t i = 0; i < count; ++i)
    if (s[i] >= n || d[i] >= n) {
      snprintf(g_err, sizeof g_err,
               "%s: vertex id out of range (%u,%u) for |V|=%u", what, s[i],
               d[i], n);
      return 1;
    }
  return 0;
}

/* buildCsr (graph.cpp:56-68). */
int orc_build_csr(uint32_t n, const uint32_t* s, const uint32_t* d,
                  uint64_t count, orc_graph** out) {
  if (check_ids(s, d, count, n, "buildCsr")) return 1;
  uint64_t* keys = (uint64_t*)malloc((count ? count : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < count; ++i) keys[i] = ((uint64_t)s[i] << 32) | d[i];
  uint64_t m = sorted_unique(keys, count);
  orc_graph* g = graph_alloc(n, m);
  for (uint64_t i = 0; i < m; ++i) g->off[(keys[i] >> 32) + 1]++;
  for (uint32_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
  for (uint64_t i = 0; i < m; ++i) g->tgt[i] = (uint32_t)keys[i];
  free(keys);
  *out = g;
  return 0;
}

/* transpose (graph.cpp:70-83): counting sort, sources ascending. */
orc_graph* orc_transpose(const orc_graph* g) {
  orc_graph* t = graph_alloc(g->n, g->m);
  for (uint64_t i = 0; i < g->m; ++i) t->off[g->tgt[i] + 1]++;
  for (uint32_t v = 0; v < g->n; ++v) t->off[v + 1] += t->off[v];
  uint64_t* cursor = (uint64_t*)malloc(((size_t)g->n + 1) * sizeof(uint64_t));
  memcpy(cursor, t->off, (size_t)g->n * sizeof(uint64_t));
  for (uint32_t u = 0; u < g->n; ++u)
    for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i)
      t->tgt[cursor[g->tgt[i]]++] = u;
  free(cursor);
  return t;
}

/* addSelfLoops (graph.cpp:85-111). */
orc_graph* orc_add_self_loops(const orc_graph* g) {
  const uint32_t n = g->n;
  uint64_t m = 0;
  for (uint32_t v = 0; v < n; ++v) m += degree(g, v) + (has_edge(g, v, v) ? 0 : 1);
  orc_graph* r = graph_alloc(n, m);
  for (uint32_t v = 0; v < n; ++v)
    r->off[v + 1] = r->off[v] + degree(g, v) + (has_edge(g, v, v) ? 0 : 1);
  for (uint32_t v = 0; v < n; ++v) {
    uint64_t w = r->off[v];
    int placed = 0;
    for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
      uint32_t t = g->tgt[i];
      if (!placed && t >= v) {
        if (t != v) r->tgt[w++] = v;
        placed = 1;
      }
      r->tgt[w++] = t;
    }
    if (!placed) r->tgt[w++] = v;
  }
  return r;
}

/* applyBatch (graph.cpp:113-203). */
int orc_apply_batch(const orc_graph* g, const uint32_t* ds, const uint32_t* dd,
                    uint64_t nd, const uint32_t* is, const uint32_t* id,
                    uint64_t ni, orc_graph** out, uint64_t* missing_out,
                    uint64_t* duplicate_out) {
  const uint32_t n = g->n;
  if (check_ids(ds, dd, nd, n, "applyBatch deletions")) return 1;
  if (check_ids(is, id, ni, n, "applyBatch insertions")) return 1;
  for (uint64_t i = 0; i < nd; ++i)
    if (ds[i] == dd[i])
      return set_err(1, "applyBatch: self-loops cannot be deleted");
  uint64_t* dels = (uint64_t*)malloc((nd ? nd : 1) * sizeof(uint64_t));
  uint64_t* ins = (uint64_t*)malloc((ni ? ni : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < nd; ++i) dels[i] = ((uint64_t)ds[i] << 32) | dd[i];
  for (uint64_t i = 0; i < ni; ++i) ins[i] = ((uint64_t)is[i] << 32) | id[i];
  const uint64_t ndu = sorted_unique(dels, nd), niu = sorted_unique(ins, ni);
  uint64_t missing = nd - ndu, duplicate = ni - niu; /* graph.cpp:126-127 */
  { /* overlap check, graph.cpp:130-138 */
    uint64_t di = 0;
    for (uint64_t k = 0; k < niu; ++k) {
      while (di < ndu && dels[di] < ins[k]) ++di;
      if (di < ndu && dels[di] == ins[k]) {
        free(dels); free(ins);
        return set_err(1, "applyBatch: edge appears in both deletions and insertions");
      }
    }
  }
  uint64_t cap = g->m + niu + n;
  uint32_t* merged = (uint32_t*)malloc((cap ? cap : 1) * sizeof(uint32_t));
  uint64_t* off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t mm = 0, di = 0, ii = 0;
  for (uint32_t v = 0; v < n; ++v) { /* graph.cpp:147-195 */
    const uint64_t sliceStart = mm;
    uint64_t s = g->off[v];
    const uint64_t se = g->off[v + 1];
    uint64_t dEnd = di, iEnd = ii;
    while (dEnd < ndu && (dels[dEnd] >> 32) == v) ++dEnd;
    while (iEnd < niu && (ins[iEnd] >> 32) == v) ++iEnd;
    int loopPlaced = 0;
    while (s < se || ii < iEnd) {
      uint32_t t;
      if (ii >= iEnd || (s < se && g->tgt[s] <= (uint32_t)ins[ii])) {
        t = g->tgt[s];
        if (ii < iEnd && (uint32_t)ins[ii] == t) { ++ii; ++duplicate; }
        ++s;
        while (di < dEnd && (uint32_t)dels[di] < t) { ++missing; ++di; }
        if (di < dEnd && (uint32_t)dels[di] == t) { ++di; continue; }
      } else {
        t = (uint32_t)ins[ii];
        ++ii;
      }
      if (!loopPlaced && t >= v) { /* push(), graph.cpp:156-162 */
        if (t != v) merged[mm++] = v;
        loopPlaced = 1;
      }
      merged[mm++] = t;
    }
    while (di < dEnd) { ++missing; ++di; }
    ii = iEnd;
    if (!loopPlaced) merged[mm++] = v;
    off[v + 1] = mm - sliceStart;
  }
  for (uint32_t v = 0; v < n; ++v) off[v + 1] += off[v];
  orc_graph* r = (orc_graph*)calloc(1, sizeof *r);
  r->n = n; r->m = mm; r->off = off; r->tgt = merged;
  free(dels); free(ins);
  if (missing_out) *missing_out += missing;
  if (duplicate_out) *duplicate_out += duplicate;
  *out = r;
  return 0;
}

/* partitionByDegree (partition.cpp:7-61): stable, low (deg <= thr) first. */
void orc_partition(const orc_graph* g, uint32_t thr, uint32_t* order,
                   uint32_t* low) {
  uint32_t w = 0;
  for (uint32_t v = 0; v < g->n; ++v) if (degree(g, v) <= thr) order[w++] = v;
  *low = w;
  for (uint32_t v = 0; v < g->n; ++v) if (degree(g, v) > thr) order[w++] = v;
}

/* updateRanks (rank.cpp:79-140).  Results do not depend on the dispatch
 * order, only on which accumulation (flat vs 256-chunked) applies, which is
 * decided by in-degree <= lowDegreeThreshold in both the partitioned and the
 * per-vertex path (rank.cpp:95-96,124-137). */
static double contrib_flat(const orc_graph* gT, const orc_graph* gF,
                           uint32_t v, const double* prev) { /* rank.cpp:45-54 */
  double c = 0.0;
  for (uint64_t i = gT->off[v]; i < gT->off[v + 1]; ++i) {
    const uint32_t u = gT->tgt[i];
    c += prev[u] / degree(gF, u);
  }
  return c;
}
static double contrib_chunked(const orc_graph* gT, const orc_graph* gF,
                              uint32_t v, const double* prev) { /* rank.cpp:59-75 */
  double c = 0.0;
  const uint64_t b = gT->off[v], len = gT->off[v + 1] - b;
  for (uint64_t base = 0; base < len; base += 256) {
    const uint64_t end = base + 256 < len ? base + 256 : len;
    double partial = 0.0;
    for (uint64_t i = base; i < end; ++i) {
      const uint32_t u = gT->tgt[b + i];
      partial += prev[u] / degree(gF, u);
    }
    c += partial;
  }
  return c;
}
void orc_update_ranks(const orc_graph* gT, const orc_graph* gF, uint8_t* va,
                      uint8_t* np, const double* previous, double* current,
                      const dynpr_config* cfg, int mode) {
  const uint32_t n = gT->n;
  const double alpha = cfg->damping_factor;
  const double teleport = (1.0 - alpha) / n; /* rank.cpp:85 */
  for (uint32_t v = 0; v < n; ++v) {
    if (va && !va[v]) { current[v] = previous[v]; continue; } /* rank.cpp:90-92 */
    const int low = degree(gT, v) <= cfg->low_degree_threshold;
    const double c = low ? contrib_flat(gT, gF, v, previous)
                         : contrib_chunked(gT, gF, v, previous);
    double r;
    if (mode == DYNPR_RANK_CLOSED_LOOP_PRUNE) { /* rank.cpp:98-103 */
      const double d = degree(gF, v);
      r = (teleport + alpha * (c - previous[v] / d)) / (1.0 - alpha / d);
    } else {
      r = teleport + alpha * c; /* rank.cpp:104 */
    }
    current[v] = r;
    if (va) { /* rank.cpp:108-115 */
      const double deltaR = fabs(r - previous[v]);
      const double denom = r > previous[v] ? r : previous[v];
      const double relative = denom > 0.0 ? deltaR / denom : 0.0;
      if (mode == DYNPR_RANK_CLOSED_LOOP_PRUNE && relative <= cfg->prune_tolerance)
        va[v] = 0;
      if (relative > cfg->frontier_tolerance) np[v] = 1;
    }
  }
}

/* linfNormDelta (rank.cpp:142-146 -> blockMax, parallel.hpp:63-74). */
double orc_linf(const double* a, const double* b, uint64_t n) {
  double result = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double t = fabs(a[i] - b[i]);
    if (t > result) result = t;
  }
  return result;
}
/* l1NormDelta (rank.cpp:148-152 -> blockSum, parallel.hpp:41-59: 4096-wide
 * block partials combined in block order). */
double orc_l1(const double* a, const double* b, uint64_t n) {
  double total = 0.0;
  for (uint64_t begin = 0; begin < n; begin += 4096) {
    const uint64_t end = begin + 4096 < n ? begin + 4096 : n;
    double s = 0.0;
    for (uint64_t i = begin; i < end; ++i) s += fabs(a[i] - b[i]);
    total += s;
  }
  return total;
}

/* initialAffected (frontier.cpp:33-53). */
int orc_initial_affected(uint32_t n, const uint32_t* ds, const uint32_t* dd,
                         uint64_t nd, const uint32_t* is, const uint32_t* id,
                         uint64_t ni, uint8_t* va, uint8_t* np) {
  for (uint64_t i = 0; i < nd; ++i)
    if (ds[i] >= n || dd[i] >= n)
      return set_err(1, "initialAffected deletions: vertex id out of range");
  for (uint64_t i = 0; i < ni; ++i)
    if (is[i] >= n || id[i] >= n)
      return set_err(1, "initialAffected insertions: vertex id out of range");
  memset(va, 0, n);
  memset(np, 0, n);
  for (uint64_t i = 0; i < nd; ++i) { np[ds[i]] = 1; va[dd[i]] = 1; }
  for (uint64_t i = 0; i < ni; ++i) np[is[i]] = 1;
  return 0;
}

/* expandAffected (frontier.cpp:55-84); dispatch order is irrelevant. */
void orc_expand_affected(const orc_graph* g, uint8_t* va, const uint8_t* np) {
  for (uint32_t u = 0; u < g->n; ++u)
    if (np[u])
      for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i) va[g->tgt[i]] = 1;
}

/* EngineConfig::validate (rank.cpp:11-20). */
int orc_validate_config(const dynpr_config* c) {
  if (!(c->damping_factor > 0.0 && c->damping_factor < 1.0))
    return set_err(1, "EngineConfig: dampingFactor must be in (0,1)");
  if (!(c->iteration_tolerance > 0.0))
    return set_err(1, "EngineConfig: iterationTolerance must be > 0");
  if (c->frontier_tolerance < 0.0 || c->prune_tolerance < 0.0)
    return set_err(1, "EngineConfig: tolerances must be >= 0");
  if (c->max_iterations <= 0)
    return set_err(1, "EngineConfig: maxIterations must be positive");
  return 0;
}
static int check_pair(const orc_graph* gT, const orc_graph* gF) {
  /* engine.cpp:15-23 */
  if (gT->n != gF->n || gT->m != gF->m)
    return set_err(1, "engine: graph pair is not mutually transposed (count mismatch)");
  if (gT->n == 0) return set_err(1, "engine: empty graph");
  return 0;
}

/* convergeLoop (engine.cpp:61-95).  va/np NULL => full sweeps (Static/ND). */
static void converge_loop(const orc_graph* gT, const orc_graph* gF,
                          double* prev, double* cur, uint8_t* va, uint8_t* np,
                          int expand, int mode, const dynpr_config* cfg,
                          double* ranks_out, dynpr_stats* st,
                          dynpr_observer obs, void* user) {
  const uint32_t n = gT->n;
  dynpr_stats r;
  memset(&r, 0, sizeof r);
  uint8_t* snap = (obs && va) ? (uint8_t*)malloc(n) : NULL;
  for (int iter = 0; iter < cfg->max_iterations; ++iter) {
    uint64_t processed = n;
    uint64_t edges = 0;
    if (va) { /* engine.cpp:72-76 */
      processed = 0;
      for (uint32_t v = 0; v < n; ++v) {
        processed += va[v];
        if (va[v]) edges += degree(gT, v);
      }
      memset(np, 0, n);
      if (snap) memcpy(snap, va, n);
    } else {
      edges = gT->m;
    }
    orc_update_ranks(gT, gF, va, np, prev, cur, cfg, mode);
    const double delta = orc_linf(cur, prev, n);
    double* t = cur; cur = prev; prev = t; /* swap, engine.cpp:80 */
    r.iterations = iter + 1;
    r.affected_vertex_iterations += processed;
    r.processed_edges += edges;
    r.final_delta = delta;
    if (obs) obs(r.iterations, prev, snap, n, user);
    if (!cfg->convergence_check_disabled && delta <= cfg->iteration_tolerance) {
      r.converged = 1;
      break;
    }
    if (expand) orc_expand_affected(gF, va, np); /* engine.cpp:91 */
  }
  memcpy(ranks_out, prev, (size_t)n * sizeof(double));
  free(snap);
  if (st) *st = r;
}

/* staticPageRank (engine.cpp:99-108). */
int orc_static(const orc_graph* gT, const orc_graph* gF, const dynpr_config* cfg,
               double* ranks, dynpr_stats* st, dynpr_observer obs, void* user) {
  if (orc_validate_config(cfg) || check_pair(gT, gF)) return 1;
  const uint32_t n = gT->n;
  double* a = (double*)malloc((size_t)n * sizeof(double));
  double* b = (double*)malloc((size_t)n * sizeof(double));
  const double r0 = 1.0 / n; /* rank.cpp:25-28 */
  for (uint32_t v = 0; v < n; ++v) a[v] = b[v] = r0;
  converge_loop(gT, gF, a, b, NULL, NULL, 0, DYNPR_RANK_PLAIN, cfg, ranks, st,
                obs, user);
  free(a); free(b);
  return 0;
}

/* naiveDynamic (engine.cpp:110-122). */
int orc_naive_dynamic(const orc_graph* gT, const orc_graph* gF,
                      const double* prevRanks, uint64_t nprev,
                      const dynpr_config* cfg, double* ranks, dynpr_stats* st,
                      dynpr_observer obs, void* user) {
  if (orc_validate_config(cfg) || check_pair(gT, gF)) return 1;
  if (nprev != gT->n) return set_err(1, "naiveDynamic: previousRanks length mismatch");
  const uint32_t n = gT->n;
  double* a = (double*)malloc((size_t)n * sizeof(double));
  double* b = (double*)malloc((size_t)n * sizeof(double));
  memcpy(a, prevRanks, (size_t)n * sizeof(double));
  memcpy(b, prevRanks, (size_t)n * sizeof(double));
  converge_loop(gT, gF, a, b, NULL, NULL, 0, DYNPR_RANK_PLAIN, cfg, ranks, st,
                obs, user);
  free(a); free(b);
  return 0;
}

static int frontier_loop(const orc_graph* gF, const orc_graph* gT, uint8_t* va,
                         uint8_t* np, const double* prevRanks,
                         const dynpr_config* cfg, int pruning, double* ranks,
                         dynpr_stats* st, dynpr_observer obs, void* user) {
  /* frontierLoop (engine.cpp:164-174) */
  const uint32_t n = gT->n;
  double* a = (double*)malloc((size_t)n * sizeof(double));
  double* b = (double*)malloc((size_t)n * sizeof(double));
  memcpy(a, prevRanks, (size_t)n * sizeof(double));
  memcpy(b, prevRanks, (size_t)n * sizeof(double));
  converge_loop(gT, gF, a, b, va, np, 1,
                pruning ? DYNPR_RANK_CLOSED_LOOP_PRUNE : DYNPR_RANK_PLAIN, cfg,
                ranks, st, obs, user);
  free(a); free(b);
  return 0;
}

/* dynamicFrontier (engine.cpp:192-203). */
int orc_dynamic_frontier(const orc_graph* gF, const orc_graph* gT,
                         const uint32_t* ds, const uint32_t* dd, uint64_t nd,
                         const uint32_t* is, const uint32_t* id, uint64_t ni,
                         const double* prevRanks, uint64_t nprev,
                         const dynpr_config* cfg, int pruning, double* ranks,
                         dynpr_stats* st, dynpr_observer obs, void* user) {
  /* checkFrontierInputs (engine.cpp:155-162) */
  if (orc_validate_config(cfg) || check_pair(gT, gF)) return 1;
  if (nprev != gT->n)
    return set_err(1, "dynamicFrontier: previousRanks length mismatch");
  const uint32_t n = gT->n;
  uint8_t* va = (uint8_t*)malloc(n);
  uint8_t* np = (uint8_t*)malloc(n);
  if (orc_initial_affected(n, ds, dd, nd, is, id, ni, va, np)) {
    free(va); free(np);
    return 1;
  }
  orc_expand_affected(gF, va, np);
  int rc = frontier_loop(gF, gT, va, np, prevRanks, cfg, pruning, ranks, st,
                         obs, user);
  free(va); free(np);
  return rc;
}

/* dynamicFrontierFromFlags (engine.cpp:178-190). */
int orc_dynamic_frontier_from_flags(const orc_graph* gF, const orc_graph* gT,
                                    const uint8_t* va0, const uint8_t* np0,
                                    uint64_t nflags, const double* prevRanks,
                                    uint64_t nprev, const dynpr_config* cfg,
                                    int pruning, double* ranks,
                                    dynpr_stats* st, dynpr_observer obs,
                                    void* user) {
  if (orc_validate_config(cfg) || check_pair(gT, gF)) return 1;
  if (nprev != gT->n)
    return set_err(1, "dynamicFrontier: previousRanks length mismatch");
  if (nflags != gT->n) return set_err(1, "dynamicFrontier: flags length mismatch");
  const uint32_t n = gT->n;
  uint8_t* va = (uint8_t*)malloc(n);
  uint8_t* np = (uint8_t*)malloc(n);
  memcpy(va, va0, n);
  memcpy(np, np0, n);
  int rc = frontier_loop(gF, gT, va, np, prevRanks, cfg, pruning, ranks, st,
                         obs, user);
  free(va); free(np);
  return rc;
}

/* markReachable (frontier.cpp:86-121): every vertex reachable from a seed
 * over g's out-slices.  Sequential BFS; only the visited set is observable
 * (frontier.cpp:96-98), so the visit order does not matter. */
int orc_mark_reachable(const orc_graph* g, const uint32_t* seeds, uint64_t ns,
                       uint8_t* va) {
  const uint32_t n = g->n;
  for (uint64_t i = 0; i < ns; ++i)
    if (seeds[i] >= n) return set_err(1, "markReachable: seed out of range");
  memset(va, 0, n);
  uint32_t* q = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint64_t head = 0, tail = 0;
  for (uint64_t i = 0; i < ns; ++i)
    if (!va[seeds[i]]) {
      va[seeds[i]] = 1;
      q[tail++] = seeds[i];
    }
  while (head < tail) {
    const uint32_t u = q[head++];
    for (uint64_t k = g->off[u]; k < g->off[u + 1]; ++k) {
      const uint32_t w = g->tgt[k];
      if (!va[w]) {
        va[w] = 1;
        q[tail++] = w;
      }
    }
  }
  free(q);
  return 0;
}

/* dynamicTraversal (engine.cpp:124-151): seeds = update sources + deletion
 * targets, affected = markReachable(gForward, seeds), plain formula, no
 * expansion. */
int orc_dynamic_traversal(const orc_graph* gF, const orc_graph* gT,
                          const uint32_t* ds, const uint32_t* dd, uint64_t nd,
                          const uint32_t* is, const uint32_t* id, uint64_t ni,
                          const double* prevRanks, uint64_t nprev,
                          const dynpr_config* cfg, double* ranks,
                          dynpr_stats* st, dynpr_observer obs, void* user) {
  (void)id;
  if (orc_validate_config(cfg) || check_pair(gT, gF)) return 1;
  if (nprev != gT->n)
    return set_err(1, "dynamicTraversal: previousRanks length mismatch");
  const uint32_t n = gT->n;
  const uint64_t ns = 2 * nd + ni;
  uint32_t* seeds = (uint32_t*)malloc((ns + 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < nd; ++i) {
    seeds[2 * i] = ds[i];
    seeds[2 * i + 1] = dd[i];
  }
  for (uint64_t i = 0; i < ni; ++i) seeds[2 * nd + i] = is[i];
  uint8_t* va = (uint8_t*)malloc((size_t)n + 1);
  uint8_t* np = (uint8_t*)calloc((size_t)n + 1, 1);
  int rc = orc_mark_reachable(gF, seeds, ns, va);
  free(seeds);
  if (rc) {
    free(va); free(np);
    return rc;
  }
  double* a = (double*)malloc((size_t)n * sizeof(double));
  double* b = (double*)malloc((size_t)n * sizeof(double));
  memcpy(a, prevRanks, (size_t)n * sizeof(double));
  memcpy(b, prevRanks, (size_t)n * sizeof(double));
  converge_loop(gT, gF, a, b, va, np, 0, DYNPR_RANK_PLAIN, cfg, ranks, st, obs,
                user);
  free(a); free(b); free(va); free(np);
  return 0;
}

/* computeReferenceRanks (harness.cpp:340-349): static, check disabled. */
int orc_compute_reference_ranks(const orc_graph* gT, const orc_graph* gF,
                                const dynpr_config* cfg, double* ranks) {
  dynpr_config c = *cfg;
  c.convergence_check_disabled = 1;
  return orc_static(gT, gF, &c, ranks, NULL, NULL, NULL);
}

/* ---- workload (workload.cpp:183-249) ----------------------------------- */
uint64_t orc_batch_size_from_fraction(double fraction, uint64_t total) {
  const double scaled = fraction * (double)total;
  const uint64_t rounded = (uint64_t)floor(scaled + 0.5);
  return rounded < 1 ? 1 : rounded;
}

/* open-addressing set of u64 keys (membership of `chosen`, workload.cpp:205) */
typedef struct { uint64_t* slot; uint64_t cap; } u64set;
static int set_insert(u64set* s, uint64_t key) {
  uint64_t k = key + 1; /* 0 marks empty */
  uint64_t h = (k * 0x9E3779B97F4A7C15ULL) & (s->cap - 1);
  while (s->slot[h]) {
    if (s->slot[h] == k) return 0;
    h = (h + 1) & (s->cap - 1);
  }
  s->slot[h] = k;
  return 1;
}

int orc_generate_random_batch(const orc_graph* g, uint64_t total,
                              double insFrac, uint64_t seed, uint32_t* is,
                              uint32_t* id, uint64_t* ni_out, uint32_t* ds,
                              uint32_t* dd, uint64_t* nd_out) {
  if (total < 1) return set_err(1, "generateRandomBatch: totalSize must be >= 1");
  if (insFrac < 0.0 || insFrac > 1.0)
    return set_err(1, "generateRandomBatch: insertFraction must be in [0,1]");
  const uint32_t n = g->n;
  const uint64_t insertCount = (uint64_t)ceil(insFrac * (double)total);
  const uint64_t deleteCount = total - insertCount;
  orc_rng rng = {seed};
  if (insertCount > 0 && n < 2)
    return set_err(5, "generateRandomBatch: need at least 2 vertices for insertions");
  u64set chosen;
  chosen.cap = 16;
  while (chosen.cap < 2 * insertCount + 2) chosen.cap <<= 1;
  chosen.slot = (uint64_t*)calloc(chosen.cap, sizeof(uint64_t));
  const uint64_t maxAttempts = 100 * (insertCount > 1 ? insertCount : 1);
  uint64_t attempts = 0, have = 0;
  while (have < insertCount) { /* workload.cpp:208-220 */
    if (++attempts > maxAttempts) {
      free(chosen.slot);
      return set_err(5, "generateRandomBatch: could not find enough non-existing edges");
    }
    const uint32_t u = (uint32_t)rng_bounded(&rng, n);
    const uint32_t v = (uint32_t)rng_bounded(&rng, n);
    if (u == v || has_edge(g, u, v)) continue;
    if (!set_insert(&chosen, ((uint64_t)u << 32) | v)) continue;
    is[have] = u;
    id[have] = v;
    ++have;
  }
  free(chosen.slot);
  *ni_out = insertCount;
  *nd_out = 0;
  if (deleteCount > 0) { /* workload.cpp:224-241, partial Fisher-Yates */
    uint64_t nc = 0;
    for (uint32_t u = 0; u < n; ++u)
      for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i)
        if (g->tgt[i] != u) ++nc;
    if (deleteCount > nc) {
      snprintf(g_err, sizeof g_err,
               "generateRandomBatch: requested %llu deletions but only %llu "
               "non-loop edges exist",
               (unsigned long long)deleteCount, (unsigned long long)nc);
      return 5;
    }
    uint64_t* cand = (uint64_t*)malloc(nc * sizeof(uint64_t));
    uint64_t w = 0;
    for (uint32_t u = 0; u < n; ++u)
      for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i)
        if (g->tgt[i] != u) cand[w++] = ((uint64_t)u << 32) | g->tgt[i];
    for (uint64_t i = 0; i < deleteCount; ++i) {
      const uint64_t j = i + rng_bounded(&rng, nc - i);
      const uint64_t t = cand[i]; cand[i] = cand[j]; cand[j] = t;
      ds[i] = (uint32_t)(cand[i] >> 32);
      dd[i] = (uint32_t)cand[i];
    }
    free(cand);
    *nd_out = deleteCount;
  }
  return 0;
}

/* randomGraph (tests/common/oracles.hpp:80-89): `pairs` uniform draws from
 * the shared rng state, buildCsr, addSelfLoops. */
orc_graph* orc_random_graph(uint64_t* state, uint32_t n, uint64_t pairs) {
  orc_rng rng = {*state};
  uint32_t* s = (uint32_t*)malloc((pairs ? pairs : 1) * sizeof(uint32_t));
  uint32_t* d = (uint32_t*)malloc((pairs ? pairs : 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < pairs; ++i) {
    s[i] = (uint32_t)rng_bounded(&rng, n);
    d[i] = (uint32_t)rng_bounded(&rng, n);
  }
  *state = rng.state;
  orc_graph* g0 = NULL;
  orc_build_csr(n, s, d, pairs, &g0);
  orc_graph* g = orc_add_self_loops(g0);
  orc_graph_free(g0);
  free(s); free(d);
  return g;
}

/* Graph500-style Kronecker edge list (no reference counterpart): the RMAT
 * draws of orc_rmat_edges with (a, b, c) = (0.57, 0.19, 0.19), every id
 * mapped through the seeded bijection of [0, 2^scale) the CUDA generator
 * uses (graph.cu Scramble: keys from a SplitMix64 stream of
 * deriveSeed(seed, 2^40), odd multipliers, xor-shifts by ceil(s/2), ceil(s/3)). */
static uint32_t orc_scramble(uint32_t x, uint64_t k1, uint64_t k2, uint64_t k3, uint64_t mask, uint32_t sh1,
                             uint32_t sh2) {
  uint64_t y = ((uint64_t)x * k1) & mask;
  y ^= y >> sh1;
  y = (y * k2 + k3) & mask;
  y ^= y >> sh2;
  return (uint32_t)y;
}
void orc_rmat_edges(uint32_t scale, uint64_t count, double a, double b, double c, uint64_t seed, uint32_t* src,
                    uint32_t* dst);
void orc_kronecker_edges(uint32_t scale, uint64_t count, uint64_t seed, uint32_t* src, uint32_t* dst) {
  orc_rmat_edges(scale, count, 0.57, 0.19, 0.19, seed, src, dst);
  orc_rng key = {orc_derive_seed(seed, 1ull << 40)};
  const uint64_t k1 = rng_next(&key) | 1ull, k2 = rng_next(&key) | 1ull, k3 = rng_next(&key);
  const uint64_t mask = (1ull << scale) - 1;
  const uint32_t sh1 = (scale + 1) / 2, sh2 = (scale + 2) / 3;
  for (uint64_t i = 0; i < count; ++i) {
    src[i] = orc_scramble(src[i], k1, k2, k3, mask, sh1, sh2);
    dst[i] = orc_scramble(dst[i], k1, k2, k3, mask, sh1, sh2);
  }
}

/* Synthetic RMAT edge list (no reference counterpart): edge i
 * draws `scale` quadrants from SplitMix64(deriveSeed(seed, i)) with
 * cumulative thresholds t1=a, t2=a+b, t3=a+b+c.  Same as the CUDA generator. */
void orc_rmat_edges(uint32_t scale, uint64_t count, double a, double b,
                    double c, uint64_t seed, uint32_t* src, uint32_t* dst) {
  const double t1 = a, t2 = a + b, t3 = a + b + c;
  for (uint64_t i = 0; i < count; ++i) {
    orc_rng rng = {orc_derive_seed(seed, i)};
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      const double r = rng_double(&rng);
      const uint32_t bu = r >= t2, bv = (r >= t1 && r < t2) || r >= t3;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    src[i] = u;
    dst[i] = v;
  }
}
