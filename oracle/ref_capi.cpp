// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// C-ABI wrapper around the *unmodified* reference library `dynpr`
// (/root/reference/proj/src/*.cpp), compiled from the sources where they lie
// by oracle/Makefile into oracle/_ref/libdynpr_ref.so.  Only tests/,
// __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm load it.
// Every function forwards to the reference's own public API; the one
// exception is ref_frontier_trace, which replays convergeLoop
// (engine.cpp:61-95) from the public primitives so the per-iteration affected
// sets can be observed (the reference observer only sees ranks).
#include <cstdint>
#include <chrono>
#include <cstring>
#include <optional>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "dynpr/engine.hpp"
#include "dynpr/frontier.hpp"
#include "dynpr/graph.hpp"
#include "dynpr/harness.hpp"
#include "dynpr/parallel.hpp"
#include "dynpr/partition.hpp"
#include "dynpr/rank.hpp"
#include "dynpr/rng.hpp"
#include "dynpr/workload.hpp"
#include "dynpr_cuda.h"  // POD config/stats/observer types only
#include "oracles.hpp"

using namespace dynpr;

namespace {

thread_local std::string g_error;

int fail(const std::exception& e) {
  g_error = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const SizingError*>(&e)) return 5;
  if (dynamic_cast<const ParseError*>(&e)) return 6;
  if (dynamic_cast<const std::runtime_error*>(&e)) return 7;
  return 2;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

EngineConfig toCfg(const dynpr_config* c) {
  EngineConfig cfg;
  if (!c) return cfg;
  cfg.dampingFactor = c->damping_factor;
  cfg.iterationTolerance = c->iteration_tolerance;
  cfg.frontierTolerance = c->frontier_tolerance;
  cfg.pruneTolerance = c->prune_tolerance;
  cfg.maxIterations = c->max_iterations;
  cfg.lowDegreeThreshold = c->low_degree_threshold;
  cfg.partitionStrategy = static_cast<PartitionStrategy>(c->partition_strategy);
  cfg.convergenceCheckDisabled = c->convergence_check_disabled != 0;
  return cfg;
}

EdgeList toEdges(const uint32_t* s, const uint32_t* d, uint64_t n) {
  EdgeList e;
  e.reserve(n);
  for (uint64_t i = 0; i < n; ++i) e.emplace_back(s[i], d[i]);
  return e;
}

void fillStats(const RankResult& r, dynpr_stats* st, double ms) {
  if (!st) return;
  st->iterations = r.iterations;
  st->converged = r.converged ? 1 : 0;
  st->affected_vertex_iterations = r.affectedVertexIterations;
  st->final_delta = r.finalDelta;
  st->processed_edges = 0;
  st->device_ms = ms;
}

IterationObserver wrapObserver(dynpr_observer obs, void* user) {
  if (!obs) return {};
  return [obs, user](int it, std::span<const double> ranks) {
    obs(it, ranks.data(), nullptr, ranks.size(), user);
  };
}

CsrGraph* G(void* h) { return static_cast<CsrGraph*>(h); }
const CsrGraph* CG(const void* h) { return static_cast<const CsrGraph*>(h); }

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_error.c_str(); }
void ref_set_threads(int t) { setThreadCount(t); }
int ref_max_threads(void) { return maxThreads(); }

// ---- rng (rng.hpp) --------------------------------------------------------
void* ref_rng_new(uint64_t seed) { return new SplitMix64(seed); }
void ref_rng_free(void* r) { delete static_cast<SplitMix64*>(r); }
uint64_t ref_rng_next(void* r) { return static_cast<SplitMix64*>(r)->next(); }
uint64_t ref_rng_bounded(void* r, uint64_t b) {
  return static_cast<SplitMix64*>(r)->bounded(b);
}
double ref_rng_next_double(void* r) {
  return static_cast<SplitMix64*>(r)->nextDouble();
}
uint64_t ref_derive_seed(uint64_t seed, uint64_t stream) {
  return deriveSeed(seed, stream);
}

// ---- graphs ----------------------------------------------------------------
int ref_graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt,
                       uint64_t m, void** out) {
  return guard([&] {
    std::vector<uint64_t> o(off, off + static_cast<size_t>(n) + 1);
    std::vector<Vertex> t(tgt, tgt + m);
    *out = new CsrGraph(n, std::move(o), std::move(t));
  });
}
int ref_build_csr(uint32_t n, const uint32_t* s, const uint32_t* d,
                  uint64_t count, void** out) {
  return guard([&] { *out = new CsrGraph(buildCsr(toEdges(s, d, count), n)); });
}
int ref_add_self_loops(const void* g, void** out) {
  return guard([&] { *out = new CsrGraph(addSelfLoops(*CG(g))); });
}
int ref_transpose(const void* g, void** out) {
  return guard([&] { *out = new CsrGraph(transpose(*CG(g))); });
}
int ref_apply_batch(const void* g, const uint32_t* ds, const uint32_t* dd,
                    uint64_t nd, const uint32_t* is, const uint32_t* id,
                    uint64_t ni, void** out, uint64_t* missing,
                    uint64_t* duplicate) {
  return guard([&] {
    BatchUpdate b;
    b.deletions = toEdges(ds, dd, nd);
    b.insertions = toEdges(is, id, ni);
    BatchApplyStats st;
    *out = new CsrGraph(applyBatch(*CG(g), b, &st));
    if (missing) *missing = st.missingDeletions;
    if (duplicate) *duplicate = st.duplicateInsertions;
  });
}
void ref_graph_info(const void* g, uint32_t* n, uint64_t* m) {
  *n = CG(g)->vertexCount();
  *m = CG(g)->edgeCount();
}
void ref_graph_download(const void* g, uint64_t* off, uint32_t* tgt) {
  const auto& o = CG(g)->offsets();
  const auto& t = CG(g)->targets();
  std::memcpy(off, o.data(), o.size() * sizeof(uint64_t));
  if (!t.empty()) std::memcpy(tgt, t.data(), t.size() * sizeof(uint32_t));
}
int ref_has_edge(const void* g, uint32_t s, uint32_t t) {
  return CG(g)->hasEdge(s, t) ? 1 : 0;
}
void ref_graph_free(void* g) { delete G(g); }

// oracles.hpp:80-89 randomGraph (consumes draws from the shared rng handle).
int ref_random_graph(void* rng, uint32_t n, uint64_t pairs, void** out) {
  return guard([&] {
    *out = new CsrGraph(
        oracles::randomGraph(*static_cast<SplitMix64*>(rng), n, pairs));
  });
}
// oracles.hpp:40-76 densePageRank.
int ref_dense_pagerank(const void* g, double alpha, double tol, int maxIter,
                       double* out, int* iters) {
  return guard([&] {
    auto r = oracles::densePageRank(oracles::edgesOf(*CG(g)),
                                    CG(g)->vertexCount(), alpha, tol, maxIter,
                                    iters);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// ---- primitives ---------------------------------------------------------
int ref_partition(const void* g, uint32_t thr, uint32_t* order,
                  uint32_t* low) {
  return guard([&] {
    DegreePartition p = partitionByDegree(*CG(g), thr);
    if (!p.order.empty())
      std::memcpy(order, p.order.data(), p.order.size() * sizeof(uint32_t));
    *low = p.lowCount;
  });
}

// updateRanks with optional flags; `use_partition` selects the in-degree
// partition of gT (PartitionTranspose/Both) vs per-vertex dispatch.
int ref_update_ranks(const void* gT, const void* gF, uint8_t* va, uint8_t* np,
                     const double* prev, double* cur, const dynpr_config* c,
                     int mode, int use_partition) {
  return guard([&] {
    const EngineConfig cfg = toCfg(c);
    const Vertex n = CG(gT)->vertexCount();
    RankState st;
    st.previous.assign(prev, prev + n);
    st.current.assign(cur, cur + n);
    std::optional<DegreePartition> part;
    if (use_partition) part = partitionByDegree(*CG(gT), cfg.lowDegreeThreshold);
    AffectedFlags flags(va ? n : 0);
    if (va) {
      flags.vertexAffected.assign(va, va + n);
      flags.neighborsPending.assign(np, np + n);
    }
    updateRanks(va ? &flags : nullptr, st, *CG(gT), *CG(gF),
                part ? &*part : nullptr, cfg,
                mode ? RankMode::ClosedLoopPrune : RankMode::Plain);
    std::memcpy(cur, st.current.data(), n * sizeof(double));
    if (va) {
      std::memcpy(va, flags.vertexAffected.data(), n);
      std::memcpy(np, flags.neighborsPending.data(), n);
    }
  });
}
int ref_linf(const double* a, const double* b, uint64_t n, double* out) {
  return guard([&] {
    *out = linfNormDelta(std::span<const double>(a, n),
                         std::span<const double>(b, n));
  });
}
int ref_l1(const double* a, const double* b, uint64_t n, double* out) {
  return guard([&] {
    *out = l1NormDelta(std::span<const double>(a, n),
                       std::span<const double>(b, n));
  });
}
int ref_initial_affected(const void* g, const uint32_t* ds, const uint32_t* dd,
                         uint64_t nd, const uint32_t* is, const uint32_t* id,
                         uint64_t ni, uint8_t* va, uint8_t* np) {
  return guard([&] {
    AffectedFlags f =
        initialAffected(*CG(g), toEdges(ds, dd, nd), toEdges(is, id, ni));
    std::memcpy(va, f.vertexAffected.data(), f.vertexAffected.size());
    std::memcpy(np, f.neighborsPending.data(), f.neighborsPending.size());
  });
}
int ref_expand_affected(const void* g, uint8_t* va, const uint8_t* np,
                        int use_partition, uint32_t thr) {
  return guard([&] {
    const Vertex n = CG(g)->vertexCount();
    AffectedFlags f(n);
    f.vertexAffected.assign(va, va + n);
    f.neighborsPending.assign(np, np + n);
    std::optional<DegreePartition> part;
    if (use_partition) part = partitionByDegree(*CG(g), thr);
    expandAffected(f, *CG(g), part ? &*part : nullptr);
    std::memcpy(va, f.vertexAffected.data(), n);
  });
}

// ---- engines ---------------------------------------------------------------
int ref_static(const void* gT, const void* gF, const dynpr_config* c,
               double* ranks, dynpr_stats* st, dynpr_observer obs,
               void* user) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    RankResult r = staticPageRank(*CG(gT), *CG(gF), toCfg(c),
                                  wrapObserver(obs, user));
    double ms = std::chrono::duration<double, std::milli>(
                    std::chrono::steady_clock::now() - t0).count();
    std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
    fillStats(r, st, ms);
  });
}
int ref_naive_dynamic(const void* gT, const void* gF, const double* prev,
                      uint64_t nprev, const dynpr_config* c, double* ranks,
                      dynpr_stats* st, dynpr_observer obs, void* user) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    RankResult r = naiveDynamic(*CG(gT), *CG(gF),
                                std::span<const double>(prev, nprev), toCfg(c),
                                wrapObserver(obs, user));
    double ms = std::chrono::duration<double, std::milli>(
                    std::chrono::steady_clock::now() - t0).count();
    std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
    fillStats(r, st, ms);
  });
}
int ref_dynamic_frontier(const void* gF, const void* gT, const uint32_t* ds,
                         const uint32_t* dd, uint64_t nd, const uint32_t* is,
                         const uint32_t* id, uint64_t ni, const double* prev,
                         uint64_t nprev, const dynpr_config* c, int pruning,
                         double* ranks, dynpr_stats* st, dynpr_observer obs,
                         void* user) {
  return guard([&] {
    EdgeList dels = toEdges(ds, dd, nd), ins = toEdges(is, id, ni);
    auto t0 = std::chrono::steady_clock::now();
    RankResult r = dynamicFrontier(*CG(gF), *CG(gT), dels, ins,
                                   std::span<const double>(prev, nprev),
                                   toCfg(c), pruning != 0,
                                   wrapObserver(obs, user));
    double ms = std::chrono::duration<double, std::milli>(
                    std::chrono::steady_clock::now() - t0).count();
    std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
    fillStats(r, st, ms);
  });
}
int ref_dynamic_traversal(const void* gF, const void* gT, const uint32_t* ds,
                          const uint32_t* dd, uint64_t nd, const uint32_t* is,
                          const uint32_t* id, uint64_t ni, const double* prev,
                          uint64_t nprev, const dynpr_config* c, double* ranks,
                          dynpr_stats* st, dynpr_observer obs, void* user) {
  return guard([&] {
    EdgeList dels = toEdges(ds, dd, nd), ins = toEdges(is, id, ni);
    auto t0 = std::chrono::steady_clock::now();
    RankResult r = dynamicTraversal(*CG(gF), *CG(gT), dels, ins,
                                    std::span<const double>(prev, nprev),
                                    toCfg(c), wrapObserver(obs, user));
    double ms = std::chrono::duration<double, std::milli>(
                    std::chrono::steady_clock::now() - t0).count();
    std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
    fillStats(r, st, ms);
  });
}
int ref_mark_reachable(const void* g, const uint32_t* seeds, uint64_t ns,
                       uint8_t* va) {
  return guard([&] {
    AffectedFlags f = markReachable(*CG(g), std::span<const Vertex>(seeds, ns));
    std::memcpy(va, f.vertexAffected.data(), f.vertexAffected.size());
  });
}
int ref_dynamic_frontier_from_flags(const void* gF, const void* gT,
                                    const uint8_t* va, const uint8_t* np,
                                    uint64_t nflags, const double* prev,
                                    uint64_t nprev, const dynpr_config* c,
                                    int pruning, double* ranks,
                                    dynpr_stats* st, dynpr_observer obs,
                                    void* user) {
  return guard([&] {
    AffectedFlags f(static_cast<Vertex>(nflags));
    f.vertexAffected.assign(va, va + nflags);
    f.neighborsPending.assign(np, np + nflags);
    RankResult r = dynamicFrontierFromFlags(
        *CG(gF), *CG(gT), std::move(f), std::span<const double>(prev, nprev),
        toCfg(c), pruning != 0, wrapObserver(obs, user));
    std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
    fillStats(r, st, 0.0);
  });
}

// Replay of convergeLoop (engine.cpp:61-95) for dynamicFrontier
// (engine.cpp:192-203) built only from public calls, reporting the processed
// set of every sweep.  tests/ check that its ranks/iterations/work equal
// ref_dynamic_frontier bit for bit, which pins the replay to the library.
int ref_frontier_trace(const void* gFv, const void* gTv, const uint32_t* ds,
                       const uint32_t* dd, uint64_t nd, const uint32_t* is,
                       const uint32_t* id, uint64_t ni, const double* prev,
                       const dynpr_config* c, int pruning, double* ranks,
                       dynpr_stats* st, dynpr_observer obs, void* user) {
  return guard([&] {
    const CsrGraph& gF = *CG(gFv);
    const CsrGraph& gT = *CG(gTv);
    const EngineConfig cfg = toCfg(c);
    cfg.validate();
    const Vertex n = gT.vertexCount();
    std::optional<DegreePartition> rankPart, expandPart;
    if (cfg.partitionStrategy != PartitionStrategy::DontPartition)
      rankPart = partitionByDegree(gT, cfg.lowDegreeThreshold);
    if (cfg.partitionStrategy == PartitionStrategy::PartitionBoth)
      expandPart = partitionByDegree(gF, cfg.lowDegreeThreshold);
    AffectedFlags flags =
        initialAffected(gF, toEdges(ds, dd, nd), toEdges(is, id, ni));
    expandAffected(flags, gF, expandPart ? &*expandPart : nullptr);
    RankState state = initRanksFrom(std::span<const double>(prev, n));
    const RankMode mode = pruning ? RankMode::ClosedLoopPrune : RankMode::Plain;
    RankResult result;
    for (int iter = 0; iter < cfg.maxIterations; ++iter) {
      std::vector<uint8_t> processedSet = flags.vertexAffected;
      uint64_t processed = 0;
      for (uint8_t b : processedSet) processed += b;
      std::fill(flags.neighborsPending.begin(), flags.neighborsPending.end(),
                uint8_t{0});
      updateRanks(&flags, state, gT, gF, rankPart ? &*rankPart : nullptr, cfg,
                  mode);
      const double delta = linfNormDelta(state.current, state.previous);
      std::swap(state.current, state.previous);
      result.iterations = iter + 1;
      result.affectedVertexIterations += processed;
      result.finalDelta = delta;
      if (obs) obs(result.iterations, state.previous.data(),
                   processedSet.data(), n, user);
      if (!cfg.convergenceCheckDisabled && delta <= cfg.iterationTolerance) {
        result.converged = true;
        break;
      }
      expandAffected(flags, gF, expandPart ? &*expandPart : nullptr);
    }
    std::memcpy(ranks, state.previous.data(), n * sizeof(double));
    fillStats(result, st, 0.0);
  });
}

int ref_compute_reference_ranks(const void* gT, const void* gF,
                                const dynpr_config* c, double* ranks) {
  return guard([&] {
    auto r = computeReferenceRanks(*CG(gT), *CG(gF), toCfg(c));
    std::memcpy(ranks, r.data(), r.size() * sizeof(double));
  });
}

// ---- workload (workload.cpp:183-249) --------------------------------------
int ref_generate_random_batch(const void* g, uint64_t total, double insFrac,
                              uint64_t seed, uint32_t* is, uint32_t* id,
                              uint64_t* ni, uint32_t* ds, uint32_t* dd,
                              uint64_t* nd) {
  return guard([&] {
    BatchUpdate b = generateRandomBatch(*CG(g), total, insFrac, seed);
    *ni = b.insertions.size();
    *nd = b.deletions.size();
    for (size_t i = 0; i < b.insertions.size(); ++i) {
      is[i] = b.insertions[i].first;
      id[i] = b.insertions[i].second;
    }
    for (size_t i = 0; i < b.deletions.size(); ++i) {
      ds[i] = b.deletions[i].first;
      dd[i] = b.deletions[i].second;
    }
  });
}
uint64_t ref_batch_size_from_fraction(double f, uint64_t total) {
  return batchSizeFromFraction(f, total);
}
int ref_validate_config(const dynpr_config* c) {
  return guard([&] { toCfg(c).validate(); });
}

// ---- input formats + harness (workload.cpp:43-181, harness.cpp) ------------
// Loaders return a heap EdgeBuf the caller reads with ref_edges_* and frees.
struct EdgeBuf {
  std::vector<uint32_t> s, d;
  std::vector<int64_t> t;
  uint32_t n = 0;
};
int ref_load_matrix_market(const char* path, void** out) {
  return guard([&] {
    auto mm = loadMatrixMarket(path);
    auto* b = new EdgeBuf;
    b->n = mm.vertexCount;
    for (auto& e : mm.edges) {
      b->s.push_back(e.first);
      b->d.push_back(e.second);
    }
    *out = b;
  });
}
int ref_load_temporal(const char* path, void** out) {
  return guard([&] {
    auto t = loadTemporalEdgeList(path);
    auto* b = new EdgeBuf;
    b->n = t.vertexCount;
    for (auto& e : t.entries) {
      b->s.push_back(e.source);
      b->d.push_back(e.target);
      b->t.push_back(e.timestamp);
    }
    *out = b;
  });
}
// splitTemporal of a loaded stream: base edges into a new EdgeBuf, batches
// concatenated into another (batch_count * batch_size insertions).
int ref_split_temporal(const void* stream, double baseFraction, int batchCount,
                       uint64_t batchSize, void** base, void** batches) {
  return guard([&] {
    const auto* b = static_cast<const EdgeBuf*>(stream);
    TemporalEdgeList t;
    t.vertexCount = b->n;
    for (size_t i = 0; i < b->s.size(); ++i) t.entries.push_back({b->s[i], b->d[i], b->t[i]});
    auto sp = splitTemporal(t, baseFraction, batchCount, batchSize);
    auto* bb = new EdgeBuf;
    bb->n = b->n;
    for (auto& e : sp.baseEdges) {
      bb->s.push_back(e.first);
      bb->d.push_back(e.second);
    }
    auto* ba = new EdgeBuf;
    ba->n = b->n;
    for (auto& batch : sp.batches)
      for (auto& e : batch.insertions) {
        ba->s.push_back(e.first);
        ba->d.push_back(e.second);
      }
    *base = bb;
    *batches = ba;
  });
}
uint64_t ref_edges_count(const void* e) { return static_cast<const EdgeBuf*>(e)->s.size(); }
uint32_t ref_edges_vertex_count(const void* e) { return static_cast<const EdgeBuf*>(e)->n; }
void ref_edges_copy(const void* e, uint32_t* s, uint32_t* d, int64_t* t) {
  const auto* b = static_cast<const EdgeBuf*>(e);
  std::memcpy(s, b->s.data(), b->s.size() * 4);
  std::memcpy(d, b->d.data(), b->d.size() * 4);
  if (t && !b->t.empty()) std::memcpy(t, b->t.data(), b->t.size() * 8);
}
void ref_edges_free(void* e) { delete static_cast<EdgeBuf*>(e); }

// runExperiment + emitReport (harness.hpp:41-79) with the fields of
// dynpr_experiment_spec; the report is written to `out_path`.
int ref_run_experiment(const dynpr_experiment_spec* s, int format, const char* out_path) {
  return guard([&] {
    ExperimentSpec spec;
    spec.graphPath = s->graph_path ? s->graph_path : "";
    spec.graphName = s->graph_name ? s->graph_name : "";
    spec.mode = static_cast<ExperimentMode>(s->mode);
    for (int i = 0; i < s->n_batch_size_specs; ++i) spec.batchSizeSpecs.push_back(s->batch_size_specs[i]);
    for (int i = 0; i < s->n_approaches; ++i) spec.approaches.push_back(static_cast<Approach>(s->approaches[i]));
    spec.seed = s->seed;
    spec.repetitions = s->repetitions;
    spec.baseFraction = s->base_fraction;
    spec.batchCount = s->batch_count;
    spec.insertFraction = s->insert_fraction;
    spec.chainMode = static_cast<ChainMode>(s->chain_mode);
    spec.threads = s->threads;
    spec.recordTiming = s->record_timing != 0;
    spec.config = toCfg(&s->config);
    auto rows = runExperiment(spec);
    emitReport(rows, format ? ReportFormat::Json : ReportFormat::Csv, out_path);
  });
}

// summarizeRows + emitReport over caller rows (dynpr_experiment_row layout).
int ref_summarize_emit(const dynpr_experiment_row* in, uint64_t count, int summarize, int format,
                       const char* out_path) {
  return guard([&] {
    std::vector<ExperimentRow> rows;
    for (uint64_t i = 0; i < count; ++i) {
      ExperimentRow r;
      r.graphName = in[i].graph_name;
      r.approach = in[i].approach;
      r.batchSizeSpec = in[i].batch_size_spec;
      r.batchIndex = in[i].batch_index;
      r.runtimeMillis = in[i].runtime_millis;
      r.iterations = in[i].iterations;
      r.affectedVertexIterations = in[i].affected_vertex_iterations;
      r.l1ErrorVsReference = in[i].l1_error_vs_reference;
      r.converged = in[i].converged != 0;
      rows.push_back(r);
    }
    if (summarize) rows = summarizeRows(rows);
    emitReport(rows, format ? ReportFormat::Json : ReportFormat::Csv, out_path);
  });
}

}  // extern "C"
