// dynpr_b200.hpp -- C++ drop-in for the reference library's compute path.
//
// Header-only shim over the C-ABI of dynpr_cuda.h.  It restores the
// reference's engine signatures (engine.hpp:33-71, graph.hpp:66-80,
// partition.hpp:20, rank.hpp:66-76) for C++ callers of `dynpr`:
//
//     #include "dynpr/engine.hpp"   // the caller's existing reference types
//     #include "dynpr_b200.hpp"
//     dynpr::RankResult r = dynpr_b200::staticPageRank(gT, gF, cfg);
//
// The graph, config and result types are the caller's own (the reference's
// dynpr::CsrGraph / EngineConfig / RankResult / EdgeList), accepted through
// templates, so this header does not depend on the reference headers.
// Failures re-throw the reference's exception types with the reference's
// message text: std::invalid_argument for DYNPR_INVALID_ARGUMENT,
// std::runtime_error otherwise.  Every call is synchronous, like the
// reference.
//
// Graph transfers: the reference API passes host graphs by value, so each
// engine call uploads its pair unless the caller keeps device snapshots
// alive with DeviceGraph (upload once, solve many times -- the form the
// benchmark and the paper's timing use).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dynpr_cuda.h"

namespace dynpr_b200 {

// SizingError / ParseError (workload.hpp:12-21) as thrown by this shim when
// the caller does not supply the reference's own classes (see check<>).
struct SizingError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(dynpr_status st) {
  if (st == DYNPR_OK) return;
  const std::string msg = dynpr_last_error();
  if (st == DYNPR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == DYNPR_SIZING_ERROR) throw SizingError(msg);
  if (st == DYNPR_PARSE_ERROR) throw ParseError(msg);
  throw std::runtime_error(msg);
}

// One CUDA device + stream + workspace.  A process-wide default context on
// device 0 is used unless the caller passes its own.
class Context {
 public:
  explicit Context(int device = 0) { check(dynpr_context_create(device, &ctx_)); }
  ~Context() { dynpr_context_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  dynpr_context* get() const { return ctx_; }
  static Context& instance() {
    static Context c(0);
    return c;
  }

 private:
  dynpr_context* ctx_ = nullptr;
};

// Owning device snapshot of a CSR graph.
class DeviceGraph {
 public:
  DeviceGraph() = default;
  explicit DeviceGraph(dynpr_graph* g) : g_(g, &dynpr_graph_destroy_void) {}
  template <class Graph>
  static DeviceGraph upload(const Graph& g, Context& ctx = Context::instance()) {
    dynpr_graph* h = nullptr;
    check(dynpr_graph_from_csr(ctx.get(), g.vertexCount(), g.offsets().data(), g.targets().data(),
                               g.targets().size(), &h));
    return DeviceGraph(h);
  }
  dynpr_graph* get() const { return g_.get(); }
  uint32_t vertexCount() const {
    uint32_t n = 0;
    uint64_t m = 0;
    check(dynpr_graph_info(g_.get(), &n, &m));
    return n;
  }
  uint64_t edgeCount() const {
    uint32_t n = 0;
    uint64_t m = 0;
    check(dynpr_graph_info(g_.get(), &n, &m));
    return m;
  }
  // Host copy in the caller's CsrGraph type (validating constructor).
  template <class Graph>
  Graph download(Context& ctx = Context::instance()) const {
    std::vector<uint64_t> off(static_cast<size_t>(vertexCount()) + 1);
    std::vector<uint32_t> tgt(edgeCount());
    check(dynpr_graph_download(ctx.get(), g_.get(), off.data(), tgt.data()));
    return Graph(vertexCount(), std::move(off), std::move(tgt));
  }

 private:
  static void dynpr_graph_destroy_void(dynpr_graph* g) { dynpr_graph_destroy(g); }
  std::shared_ptr<dynpr_graph> g_;
};

template <class Cfg>
dynpr_config toConfig(const Cfg& c) {
  dynpr_config d;
  d.damping_factor = c.dampingFactor;
  d.iteration_tolerance = c.iterationTolerance;
  d.frontier_tolerance = c.frontierTolerance;
  d.prune_tolerance = c.pruneTolerance;
  d.max_iterations = c.maxIterations;
  d.low_degree_threshold = c.lowDegreeThreshold;
  d.partition_strategy = static_cast<int32_t>(c.partitionStrategy);
  d.convergence_check_disabled = c.convergenceCheckDisabled ? 1 : 0;
  return d;
}

namespace detail {

struct ObserverBox {
  std::function<void(int, std::span<const double>)> fn;
  static void trampoline(int it, const double* r, const uint8_t*, uint64_t n, void* user) {
    static_cast<ObserverBox*>(user)->fn(it, std::span<const double>(r, n));
  }
};

template <class Result>
Result makeResult(std::vector<double> ranks, const dynpr_stats& st) {
  Result r;
  r.ranks = std::move(ranks);
  r.iterations = st.iterations;
  r.affectedVertexIterations = st.affected_vertex_iterations;
  r.converged = st.converged != 0;
  r.finalDelta = st.final_delta;
  return r;
}

template <class EdgeList>
void split(const EdgeList& e, std::vector<uint32_t>& s, std::vector<uint32_t>& d) {
  s.resize(e.size());
  d.resize(e.size());
  for (size_t i = 0; i < e.size(); ++i) {
    s[i] = e[i].first;
    d[i] = e[i].second;
  }
}

}  // namespace detail

// ---- engines on device snapshots ------------------------------------------------
template <class Result, class Cfg, class Observer = std::function<void(int, std::span<const double>)>>
Result staticPageRank(const DeviceGraph& gT, const DeviceGraph& gF, const Cfg& cfg, const Observer& obs = {},
                      Context& ctx = Context::instance()) {
  const dynpr_config c = toConfig(cfg);
  std::vector<double> ranks(gT.vertexCount());
  dynpr_stats st{};
  detail::ObserverBox box{std::function<void(int, std::span<const double>)>(obs)};
  check(dynpr_static_pagerank(ctx.get(), gT.get(), gF.get(), &c, ranks.data(), &st,
                              box.fn ? &detail::ObserverBox::trampoline : nullptr, &box));
  return detail::makeResult<Result>(std::move(ranks), st);
}

template <class Result, class EdgeList, class Cfg,
          class Observer = std::function<void(int, std::span<const double>)>>
Result dynamicFrontier(const DeviceGraph& gF, const DeviceGraph& gT, const EdgeList& deletions,
                       const EdgeList& insertions, std::span<const double> previousRanks, const Cfg& cfg,
                       bool pruning, const Observer& obs = {}, Context& ctx = Context::instance()) {
  const dynpr_config c = toConfig(cfg);
  std::vector<uint32_t> ds, dd, is, id;
  detail::split(deletions, ds, dd);
  detail::split(insertions, is, id);
  std::vector<double> ranks(gT.vertexCount());
  dynpr_stats st{};
  detail::ObserverBox box{std::function<void(int, std::span<const double>)>(obs)};
  check(dynpr_dynamic_frontier(ctx.get(), gF.get(), gT.get(), ds.data(), dd.data(), ds.size(), is.data(),
                               id.data(), is.size(), previousRanks.data(), previousRanks.size(), &c,
                               pruning ? 1 : 0, ranks.data(), &st,
                               box.fn ? &detail::ObserverBox::trampoline : nullptr, &box));
  return detail::makeResult<Result>(std::move(ranks), st);
}

// ---- the reference signatures (host graphs, uploaded per call) -------------------
// staticPageRank(gTranspose, gForward, cfg, observer) -- engine.hpp:33-35
template <class Result, class Graph, class Cfg,
          class Observer = std::function<void(int, std::span<const double>)>>
Result staticPageRank(const Graph& gT, const Graph& gF, const Cfg& cfg, const Observer& obs = {}) {
  // one call: gF's targets (unused by Static) upload and validate while the
  // solve runs (dynpr_static_pagerank_csr)
  Context& ctx = Context::instance();
  const dynpr_config c = toConfig(cfg);
  if (gT.vertexCount() != gF.vertexCount() || gT.targets().size() != gF.targets().size())
    return staticPageRank<Result>(DeviceGraph::upload(gT), DeviceGraph::upload(gF), cfg, obs);
  std::vector<double> ranks(gT.vertexCount());
  dynpr_stats st{};
  detail::ObserverBox box{std::function<void(int, std::span<const double>)>(obs)};
  check(dynpr_static_pagerank_csr(ctx.get(), gT.vertexCount(), gT.offsets().data(), gT.targets().data(),
                                  gF.offsets().data(), gF.targets().data(), gT.targets().size(), &c, ranks.data(),
                                  &st, box.fn ? &detail::ObserverBox::trampoline : nullptr, &box));
  return detail::makeResult<Result>(std::move(ranks), st);
}

// dynamicFrontier(gForward, gTranspose, dels, ins, prev, cfg, pruning) -- engine.hpp:58-62
template <class Result, class Graph, class EdgeList, class Cfg,
          class Observer = std::function<void(int, std::span<const double>)>>
Result dynamicFrontier(const Graph& gF, const Graph& gT, const EdgeList& deletions, const EdgeList& insertions,
                       std::span<const double> previousRanks, const Cfg& cfg, bool pruning,
                       const Observer& obs = {}) {
  return dynamicFrontier<Result>(DeviceGraph::upload(gF), DeviceGraph::upload(gT), deletions, insertions,
                                 previousRanks, cfg, pruning, obs);
}

// ---- graph construction on the device (graph.hpp:66-80) ---------------------------
template <class EdgeList>
DeviceGraph buildCsr(const EdgeList& edges, uint32_t vertexCount, Context& ctx = Context::instance()) {
  std::vector<uint32_t> s, d;
  detail::split(edges, s, d);
  dynpr_graph* h = nullptr;
  check(dynpr_graph_build(ctx.get(), vertexCount, s.data(), d.data(), s.size(), &h));
  return DeviceGraph(h);
}
inline DeviceGraph addSelfLoops(const DeviceGraph& g, Context& ctx = Context::instance()) {
  dynpr_graph* h = nullptr;
  check(dynpr_graph_add_self_loops(ctx.get(), g.get(), &h));
  return DeviceGraph(h);
}
inline DeviceGraph transpose(const DeviceGraph& g, Context& ctx = Context::instance()) {
  dynpr_graph* h = nullptr;
  check(dynpr_graph_transpose(ctx.get(), g.get(), &h));
  return DeviceGraph(h);
}
// applyBatch(g, batch, stats) -- graph.hpp:79-80 (Stats: missingDeletions /
// duplicateInsertions, accumulated like BatchApplyStats).
template <class Batch, class Stats = std::nullptr_t>
DeviceGraph applyBatch(const DeviceGraph& g, const Batch& batch, Stats* stats = nullptr,
                       Context& ctx = Context::instance()) {
  std::vector<uint32_t> ds, dd, is, id;
  detail::split(batch.deletions, ds, dd);
  detail::split(batch.insertions, is, id);
  uint64_t missing = 0, dup = 0;
  dynpr_graph* h = nullptr;
  check(dynpr_graph_apply_batch(ctx.get(), g.get(), ds.data(), dd.data(), ds.size(), is.data(), id.data(),
                                is.size(), &h, &missing, &dup));
  if constexpr (!std::is_same_v<Stats, std::nullptr_t>) {
    if (stats) {
      stats->missingDeletions += missing;
      stats->duplicateInsertions += dup;
    }
  }
  return DeviceGraph(h);
}

// partitionByDegree(g, threshold) -- partition.hpp:20
template <class Partition>
Partition partitionByDegree(const DeviceGraph& g, uint32_t threshold, Context& ctx = Context::instance()) {
  Partition p;
  p.order.resize(g.vertexCount());
  uint32_t low = 0;
  check(dynpr_partition_by_degree(ctx.get(), g.get(), threshold, p.order.data(), &low));
  p.lowCount = low;
  return p;
}

// linfNormDelta(a, b) -- rank.hpp:71
inline double linfNormDelta(std::span<const double> a, std::span<const double> b,
                            Context& ctx = Context::instance()) {
  if (a.size() != b.size()) throw std::invalid_argument("linfNormDelta: length mismatch");
  double out = 0.0;
  check(dynpr_linf_norm_delta(ctx.get(), a.data(), b.data(), a.size(), &out));
  return out;
}


// ---- input formats + harness (workload.hpp:43-64, harness.hpp:12-79) -------

// loadMatrixMarket -- workload.hpp:45-48.  MMGraph = {EdgeList edges;
// Vertex vertexCount;} (the reference's MatrixMarketGraph).
template <class MMGraph>
MMGraph loadMatrixMarket(const std::string& path) {
  dynpr_edge_list* e = nullptr;
  check(dynpr_load_matrix_market(path.c_str(), &e));
  std::unique_ptr<dynpr_edge_list, dynpr_status (*)(dynpr_edge_list*)> guard(e, &dynpr_edge_list_destroy);
  uint32_t n = 0;
  uint64_t cnt = 0;
  int ts = 0;
  check(dynpr_edge_list_info(e, &n, &cnt, &ts));
  std::vector<uint32_t> s(cnt), d(cnt);
  check(dynpr_edge_list_copy(e, 0, cnt, s.data(), d.data(), nullptr));
  MMGraph out;
  out.vertexCount = n;
  out.edges.reserve(cnt);
  for (uint64_t i = 0; i < cnt; ++i) out.edges.emplace_back(s[i], d[i]);
  return out;
}

// computeReferenceRanks -- harness.hpp:57-61 (500 sweeps on the device).
template <class Graph, class Cfg>
std::vector<double> computeReferenceRanks(const Graph& gT, const Graph& gF, const Cfg& cfg,
                                          Context& ctx = Context::instance()) {
  const DeviceGraph dT = DeviceGraph::upload(gT, ctx), dF = DeviceGraph::upload(gF, ctx);
  const dynpr_config c = toConfig(cfg);
  std::vector<double> r(gT.vertexCount());
  check(dynpr_compute_reference_ranks(ctx.get(), dT.get(), dF.get(), &c, r.data()));
  return r;
}

// runExperiment -- harness.hpp:63-65, on the device engines.  Spec / Row are
// the reference's ExperimentSpec / ExperimentRow (field for field); the
// enums convert through their underlying values, which match
// DYNPR_APPROACH_* / DYNPR_MODE_* / DYNPR_CHAIN_*.
template <class Row, class Spec>
std::vector<Row> runExperiment(const Spec& spec, Context& ctx = Context::instance()) {
  dynpr_experiment_spec c;
  dynpr_experiment_spec_default(&c);
  std::vector<const char*> sizes;
  for (const auto& x : spec.batchSizeSpecs) sizes.push_back(x.c_str());
  std::vector<int32_t> approaches;
  for (auto a : spec.approaches) approaches.push_back(static_cast<int32_t>(a));
  c.graph_path = spec.graphPath.c_str();
  c.graph_name = spec.graphName.c_str();
  c.mode = static_cast<int32_t>(spec.mode);
  c.batch_size_specs = sizes.data();
  c.n_batch_size_specs = static_cast<int32_t>(sizes.size());
  c.approaches = approaches.data();
  c.n_approaches = static_cast<int32_t>(approaches.size());
  c.seed = spec.seed;
  c.repetitions = spec.repetitions;
  c.base_fraction = spec.baseFraction;
  c.batch_count = spec.batchCount;
  c.insert_fraction = spec.insertFraction;
  c.chain_mode = static_cast<int32_t>(spec.chainMode);
  c.threads = spec.threads;
  c.record_timing = spec.recordTiming ? 1 : 0;
  c.config = toConfig(spec.config);
  dynpr_report* rep = nullptr;
  check(dynpr_run_experiment(ctx.get(), &c, &rep));
  std::unique_ptr<dynpr_report, dynpr_status (*)(dynpr_report*)> guard(rep, &dynpr_report_destroy);
  uint64_t cnt = 0;
  check(dynpr_report_size(rep, &cnt));
  std::vector<Row> rows(cnt);
  for (uint64_t i = 0; i < cnt; ++i) {
    dynpr_experiment_row r;
    check(dynpr_report_row(rep, i, &r));
    rows[i].graphName = r.graph_name;
    rows[i].approach = r.approach;
    rows[i].batchSizeSpec = r.batch_size_spec;
    rows[i].batchIndex = r.batch_index;
    rows[i].runtimeMillis = r.runtime_millis;
    rows[i].iterations = r.iterations;
    rows[i].affectedVertexIterations = r.affected_vertex_iterations;
    rows[i].l1ErrorVsReference = r.l1_error_vs_reference;
    rows[i].converged = r.converged != 0;
  }
  return rows;
}

// emitReport -- harness.hpp:77-79 (format: 0 CSV, 1 JSON).
template <class Row>
void emitReport(const std::vector<Row>& rows, int format, const std::string& path) {
  dynpr_report* rep = nullptr;
  check(dynpr_report_create(&rep));
  std::unique_ptr<dynpr_report, dynpr_status (*)(dynpr_report*)> guard(rep, &dynpr_report_destroy);
  for (const auto& r : rows) {
    dynpr_experiment_row c{r.graphName.c_str(), r.approach.c_str(), r.batchSizeSpec.c_str(), r.batchIndex,
                           r.runtimeMillis, r.iterations, r.affectedVertexIterations, r.l1ErrorVsReference,
                           r.converged ? 1 : 0};
    check(dynpr_report_append(rep, &c));
  }
  check(dynpr_report_emit(rep, format, path.c_str()));
}

}  // namespace dynpr_b200
