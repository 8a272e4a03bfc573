/*
 * ORACLE / TEST INFRASTRUCTURE ONLY (built into oracle/_build/libdynpr_oracle.so).
 *
 * Multithreaded (OpenMP) builders of the benchmark's synthetic input for the
 * CPU arms of bench.py -- the reference arm and the cpu_baseline leg -- so
 * that those arms never load the product library to obtain their graph.
 * They produce exactly the bytes of the sequential restatement in
 * dynpr_oracle.c (which tests/test_oracle.py pins to the reference):
 *
 *   orc_par_rmat_edges   == orc_rmat_edges (edge i from SplitMix64(deriveSeed(seed, i)))
 *   orc_par_build_csr    == buildCsr (graph.cpp:56-68) [+ addSelfLoops
 *                           (graph.cpp:85-111) when add_loops]: rows sorted
 *                           ascending and deduplicated, so the result does not
 *                           depend on the scatter order of the threads
 *   orc_par_transpose    == transpose (graph.cpp:70-83): a deduplicated CSR's
 *                           transpose is buildCsr of its reversed pairs
 *
 * The reference's own buildCsr sorts the whole pair list with one sequential
 * std::sort (graph.cpp:23): 52 s at RMAT-24.  These take a few
 * seconds on the GPU box's host cores.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <omp.h>

typedef struct { uint64_t state; } par_rng;
static uint64_t par_next(par_rng* r) { /* rng.hpp:14-19 */
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static double par_double(par_rng* r) { return (double)(par_next(r) >> 11) * 0x1.0p-53; } /* rng.hpp:37 */
static uint64_t par_derive(uint64_t seed, uint64_t stream) {                            /* rng.hpp:44-47 */
  par_rng r = {seed ^ (0xD1B54A32D192ED03ULL * (stream + 1))};
  return par_next(&r);
}

void orc_par_rmat_edges(uint32_t scale, uint64_t count, double a, double b, double c, uint64_t seed,
                        uint32_t* src, uint32_t* dst) {
  const double t1 = a, t2 = a + b, t3 = a + b + c;
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < count; ++i) {
    par_rng rng = {par_derive(seed, i)};
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      const double r = par_double(&rng);
      const uint32_t bu = r >= t2, bv = (r >= t1 && r < t2) || r >= t3;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    src[i] = u;
    dst[i] = v;
  }
}

static void sort_u32(uint32_t* a, uint64_t n, uint32_t* tmp) {
  if (n < 48) { /* insertion sort: most rows are short */
    for (uint64_t i = 1; i < n; ++i) {
      const uint32_t x = a[i];
      uint64_t j = i;
      while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; --j; }
      a[j] = x;
    }
    return;
  }
  /* LSD radix, 4 passes of 8 bits (hub rows) */
  uint32_t* s = a;
  uint32_t* d = tmp;
  for (int sh = 0; sh < 32; sh += 8) {
    uint64_t cnt[257];
    memset(cnt, 0, sizeof cnt);
    for (uint64_t i = 0; i < n; ++i) cnt[((s[i] >> sh) & 255u) + 1]++;
    for (int k = 0; k < 256; ++k) cnt[k + 1] += cnt[k];
    for (uint64_t i = 0; i < n; ++i) d[cnt[(s[i] >> sh) & 255u]++] = s[i];
    uint32_t* t = s; s = d; d = t;
  }
  /* four passes: the sorted data is back in `a` */
}

/* Rows of (src[i], dst[i]) pairs (+ one (v, v) per vertex with add_loops),
 * each sorted and deduplicated.  off: n+1 entries; tgt: capacity
 * count + (add_loops ? n : 0).  Returns m. */
uint64_t orc_par_build_csr(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t count, int add_loops,
                           uint64_t* off, uint32_t* tgt) {
  uint64_t* cur = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < count; ++i) {
#pragma omp atomic
    cur[src[i] + 1]++;
  }
  if (add_loops) {
#pragma omp parallel for schedule(static)
    for (uint64_t v = 0; v < n; ++v) cur[v + 1] += 1;
  }
  for (uint64_t v = 0; v < n; ++v) cur[v + 1] += cur[v];
  uint64_t* start = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  memcpy(start, cur, ((size_t)n + 1) * sizeof(uint64_t));
  uint32_t* raw = (uint32_t*)malloc((start[n] ? start[n] : 1) * sizeof(uint32_t));
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < count; ++i) {
    uint64_t p;
#pragma omp atomic capture
    p = cur[src[i]]++;
    raw[p] = dst[i];
  }
  if (add_loops) {
#pragma omp parallel for schedule(static)
    for (uint64_t v = 0; v < n; ++v) raw[cur[v]++] = (uint32_t)v;
  }
  /* sort + dedupe each row in place; its unique length goes to cur[v] */
#pragma omp parallel
  {
    uint64_t cap = 0;
    uint32_t* tmp = NULL;
#pragma omp for schedule(dynamic, 4096)
    for (uint64_t v = 0; v < n; ++v) {
      uint32_t* r = raw + start[v];
      const uint64_t len = start[v + 1] - start[v];
      if (len > cap) {
        free(tmp);
        cap = len;
        tmp = (uint32_t*)malloc(cap * sizeof(uint32_t));
      }
      sort_u32(r, len, tmp);
      uint64_t w = 0;
      for (uint64_t k = 0; k < len; ++k)
        if (w == 0 || r[w - 1] != r[k]) r[w++] = r[k];
      cur[v] = w;
    }
    free(tmp);
  }
  off[0] = 0;
  for (uint64_t v = 0; v < n; ++v) off[v + 1] = off[v] + cur[v];
#pragma omp parallel for schedule(dynamic, 4096)
  for (uint64_t v = 0; v < n; ++v) memcpy(tgt + off[v], raw + start[v], cur[v] * sizeof(uint32_t));
  const uint64_t m = off[n];
  free(raw);
  free(start);
  free(cur);
  return m;
}

/* transpose of a sorted, deduplicated CSR (graph.cpp:70-83). */
void orc_par_transpose(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint64_t* toff, uint32_t* ttgt) {
  const uint64_t m = off[n];
  uint32_t* rsrc = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
#pragma omp parallel for schedule(dynamic, 4096)
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t e = off[u]; e < off[u + 1]; ++e) rsrc[e] = (uint32_t)u;
  orc_par_build_csr(n, tgt, rsrc, m, 0, toff, ttgt);
  free(rsrc);
}

int orc_par_threads(void) { return omp_get_max_threads(); }
