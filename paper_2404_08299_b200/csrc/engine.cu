// Engines and the extern "C" boundary of libdynpr_cuda.so.
//
//   staticPageRank            engine.cpp:99-108   -> dynpr_static_pagerank
//   naiveDynamic              engine.cpp:110-122  -> dynpr_naive_dynamic
//   dynamicFrontier           engine.cpp:192-203  -> dynpr_dynamic_frontier
//   dynamicFrontierFromFlags  engine.cpp:178-190  -> dynpr_dynamic_frontier_from_flags
//   convergeLoop              engine.cpp:61-95    -> solve() below
//   updateRanks / linfNormDelta / l1NormDelta     rank.cpp:79-152
//   initialAffected / expandAffected              frontier.cpp:33-84
//   partitionByDegree                             partition.cpp:7-61
//   EngineConfig::validate                        rank.cpp:11-20
//
// The host loop mirrors convergeLoop's order exactly (count -> clear pending
// -> update -> L-inf -> swap -> record -> observer -> convergence test ->
// expand); the count, the pending clear and the L-inf are fused into the
// sweep kernels, and the only per-iteration host traffic is one 32-byte
// readback (delta, processed, edges, pending-list sizes).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <string>
#include <mutex>
#include <vector>

#include "layout.cuh"
#include "comm.cuh"
#include "sweep.cuh"

namespace dynpr_b200 {

// Test hook: a 1-rank NCCL / LocalTeam context takes the team path (range
// plan, collectives, speculative host loop) instead of the single-GPU one,
// so the real transport code runs on a one-GPU box.
bool team_forced() {
  const char* e = std::getenv("DYNPR_FORCE_TEAM");
  return e && e[0] && e[0] != '0';
}
bool is_team(const dynpr_context* ctx) { return ctx->comm && (ctx->comm->world > 1 || team_forced()); }

thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

bool any_bad_ids(dynpr_context* ctx, const uint32_t* d_s, const uint32_t* d_d, uint64_t cnt, uint32_t n);

// Range check of a batch list: on the host when the caller's arrays are host
// memory (no device round trip), else on the device (staged arrays).
bool batch_ids_bad(dynpr_context* ctx, const uint32_t* user_s, const uint32_t* user_d, const uint32_t* dev_s,
                   const uint32_t* dev_d, uint64_t cnt, uint32_t n) {
  if (!cnt) return false;
  if (user_s && user_d && !is_device_ptr(user_s) && !is_device_ptr(user_d)) {
    for (uint64_t i = 0; i < cnt; ++i)
      if (user_s[i] >= n || user_d[i] >= n) return true;
    return false;
  }
  return any_bad_ids(ctx, dev_s, dev_d, cnt, n);
}

namespace {

void validate_config(const dynpr_config* c) {  // rank.cpp:11-20
  if (!c) invalid("null config");
  if (!(c->damping_factor > 0.0 && c->damping_factor < 1.0))
    invalid("EngineConfig: dampingFactor must be in (0,1)");
  if (!(c->iteration_tolerance > 0.0)) invalid("EngineConfig: iterationTolerance must be > 0");
  if (c->frontier_tolerance < 0.0 || c->prune_tolerance < 0.0)
    invalid("EngineConfig: tolerances must be >= 0");
  if (c->max_iterations <= 0) invalid("EngineConfig: maxIterations must be positive");
}

void check_pair(const dynpr_graph* gT, const dynpr_graph* gF) {  // engine.cpp:15-23
  if (!gT || !gF) invalid("null graph");
  if (gT->n != gF->n || gT->m != gF->m)
    invalid("engine: graph pair is not mutually transposed (count mismatch)");
  if (gT->n == 0) invalid("engine: empty graph");
}

double bits_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

SweepRed read_red(dynpr_context* ctx, const SweepRed* d) {
  DYNPR_CK(cudaMemcpyAsync(ctx->pinned, d, sizeof(SweepRed), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  SweepRed h;
  std::memcpy(&h, ctx->pinned, sizeof h);
  return h;
}

// A team shares one replicated graph: every rank must hold the same pair,
// or the ranges it sweeps belong to different graphs.  The content
// fingerprint of the pair (both CSRs) is computed once per layout; every
// team solve all-reduces it (max and sum agree only if all ranks match).
void ensure_fingerprint(dynpr_context* ctx, Layout* L, const dynpr_graph* gT, const dynpr_graph* gF) {
  if (L->fingerprint) return;
  SweepRed* red = ctx->red.as<SweepRed>(2);
  DYNPR_CK(cudaMemsetAsync(red, 0, sizeof(SweepRed), ctx->stream));
  auto* acc = reinterpret_cast<unsigned long long*>(&red->delta_bits);
  launch_fingerprint(ctx, reinterpret_cast<const uint32_t*>(gT->off), 2 * ((uint64_t)gT->n + 1), 1ull << 40, acc);
  launch_fingerprint(ctx, gT->tgt, gT->m, 2ull << 40, acc);
  launch_fingerprint(ctx, reinterpret_cast<const uint32_t*>(gF->off), 2 * ((uint64_t)gF->n + 1), 3ull << 40, acc);
  launch_fingerprint(ctx, gF->tgt, gF->m, 4ull << 40, acc);
  const uint64_t fp = read_red(ctx, red).delta_bits;
  L->fingerprint = fp ? fp : 1;
}

void team_check_graph(dynpr_context* ctx, Comm* comm, Layout* L, const dynpr_graph* gT, const dynpr_graph* gF,
                      SweepRed* red) {
  ensure_fingerprint(ctx, L, gT, gF);
  SweepRed rec{};
  rec.delta_bits = L->fingerprint;
  rec.processed = L->fingerprint;
  std::memcpy(ctx->pinned, &rec, sizeof rec);
  DYNPR_CK(cudaMemcpyAsync(red, ctx->pinned, sizeof rec, cudaMemcpyHostToDevice, ctx->stream));
  comm->allreduce_red(red, ctx->stream);
  const SweepRed t = read_red(ctx, red);
  if (t.processed != t.delta_bits * (uint64_t)comm->world)
    throw Error(DYNPR_INVALID_ARGUMENT, "team: the ranks hold different graphs (a team sweeps one replicated graph)");
}

struct SolveSpec {
  const dynpr_graph* gT = nullptr;
  const dynpr_graph* gF = nullptr;
  const dynpr_config* cfg = nullptr;
  const double* prev = nullptr;  // device, or null for the uniform start
  bool flagged = false;          // DF / DF-P frontier loop
  bool closed = false;           // ClosedLoopPrune formula (DF-P)
  // frontier seeds: batch (device arrays) or explicit flags (device)
  const uint32_t* ds = nullptr;
  const uint32_t* dd = nullptr;
  uint64_t nd = 0;
  const uint32_t* is = nullptr;
  uint64_t ni = 0;
  const uint8_t* flags_in = nullptr;
  // dynamicTraversal (engine.cpp:124-151): the affected set is everything
  // reachable from the seeds, fixed for the whole solve (no expansion)
  bool traversal = false;
  const uint32_t* seeds = nullptr;
  uint64_t nseeds = 0;
};

bool host_loop_forced() {
  const char* e = std::getenv("DYNPR_HOST_LOOP");
  return e && e[0] && e[0] != '0';
}

// convergeLoop (engine.cpp:61-95) run entirely on the device: one CUDA graph
// whose WHILE node repeats a body of body_sweeps() iterations (even sweeps
// R0->R1, odd sweeps R1->R0, so the ping-pong buffers are baked in), each
//   sweep -> k_loop_end -> [collect | push expand]
// where k_loop_end does the count / delta / convergence / max-iterations
// bookkeeping of engine.cpp:79-91 on the device, zeroes the record, picks
// the expansion direction, and sets the loop condition.  Kernels of an
// iteration after convergence return immediately (done flag), so the rest
// of the last body is free.  The host waits once, at the end.
//
// The kernels read their SweepArgs from constant-bank slots written per solve,
// so an instantiated graph depends only on the sweep plan (kernel choice and
// grids) and is cached on the context: a solve costs one ~1 KB upload and a
// graph launch, not a capture + instantiate (~0.2 ms).
struct LoopGraph {
  SweepPlan plan;
  int frontier;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t launches_per_body = 0;  // (without the push expansions' IF bodies)
  uint64_t launches_per_push = 0;
  uint64_t launches_per_empty_check = 0;
};
struct LoopGraphCache {
  std::vector<LoopGraph> items;
  ~LoopGraphCache() {
    for (auto& x : items) {
      if (x.exec) cudaGraphExecDestroy(x.exec);
      if (x.g) cudaGraphDestroy(x.g);
    }
  }
};
constexpr size_t kLoopCacheMax = 16;
// Sweeps per WHILE body: the body's re-evaluation costs ~17 us, paid once
// per body -- 4 for the latency-mode (fused) sweeps of small graphs
// (RMAT-18 Static 3.03 -> 2.94 ms, RMAT-20 4.25 -> 4.18), 2 for the split
// sweeps (4 made RMAT-24 Static 56.0 -> 59.8 ms).
int body_sweeps(const SweepPlan& p) { return p.split ? 2 : 4; }

// expandAffected direction (both loops): pull when push_cost x the pending
// vertices' out-edges exceed the in-edges of the vertices the sweep left
// unaffected (what a pull scans).  A pushed edge is a dependent id load plus
// a flag read-modify-write, a pulled one a gather the in-sweep pull merges
// into the sweep it precedes: push_cost 4 (profiles/r02/push_cost_ab.txt:
// RMAT-20 1e-7 0.75 -> 0.50 ms, 1e-5 1.00 -> 0.83, uniform n=2^20 1e-4 /
// 1e-3 0.85 -> 0.63 / 0.94 -> 0.74, RMAT-24 unchanged).  DYNPR_PUSH_COST
// overrides (A/B).
int push_cost_factor() {
  const char* e = std::getenv("DYNPR_PUSH_COST");
  const long v = e ? std::strtol(e, nullptr, 10) : 4L;
  return v > 0 ? (int)v : 1;
}

bool pull_fused_enabled() {
  const char* pf = std::getenv("DYNPR_PULL_FUSED");
  return !(pf && pf[0] == '0');
}

// Device-loop solves of one GPU in this process go one at a time (the
// constant-bank argument slots are per device); captures too.
std::mutex& loop_slot_lock(int device) {
  static std::mutex locks[64];
  return locks[device & 63];
}

LoopGraph& loop_graph(dynpr_context* ctx, const SweepPlan& plan, int frontier, LoopCtl* dc, SweepRed* red) {
  auto* cache = static_cast<LoopGraphCache*>(ctx->loop_graphs);
  if (!cache) ctx->loop_graphs = cache = new LoopGraphCache();
  for (auto& x : cache->items)
    if (x.frontier == frontier && std::memcmp(&x.plan, &plan, sizeof plan) == 0) return x;
  if (cache->items.size() >= kLoopCacheMax) {
    LoopGraph& old = cache->items.front();
    cudaGraphExecDestroy(old.exec);
    cudaGraphDestroy(old.g);
    cache->items.erase(cache->items.begin());
  }
  cudaStream_t st = ctx->stream;
  LoopGraph lg;
  lg.plan = plan;
  lg.frontier = frontier;
  const uint64_t launches0 = ctx->launches;
  uint32_t* tick = sweep_tick(ctx);
  DYNPR_CK(cudaGraphCreate(&lg.g, 0));
  cudaGraphConditionalHandle cond;
  DYNPR_CK(cudaGraphConditionalHandleCreate(&cond, lg.g, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = cond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  DYNPR_CK(cudaGraphAddNode(&node, lg.g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  // A frontier loop's push expansion sits in an IF node that k_loop_end
  // arms only when a push follows: pull iterations (and the last one) launch
  // no expansion kernels at all (before: three gated-off 16-CTA/SM grids
  // per iteration, ~13 us of an RMAT-20 sweep's ~62).
  const int nb = body_sweeps(plan);
  // The DF-P end-game check (launch_empty_check) in its own IF node: split
  // plans only -- an empty sweep there costs ~0.2-0.3 ms (RMAT-24), while on
  // the latency-mode plans a second IF node per iteration cost more than the
  // empty sweeps it saves (profiles/r02/empty_check_ab.txt).
  const bool end_check = frontier && plan.split && plan.closed;
  std::vector<cudaGraphConditionalHandle> hpush(frontier ? nb : 0), hempty(end_check ? nb : 0);
  for (auto& x : hpush) DYNPR_CK(cudaGraphConditionalHandleCreate(&x, body, 0u, cudaGraphCondAssignDefault));
  for (auto& x : hempty) DYNPR_CK(cudaGraphConditionalHandleCreate(&x, body, 0u, cudaGraphCondAssignDefault));
  if (frontier && !ctx->capture_aux)
    DYNPR_CK(cudaStreamCreateWithFlags(&ctx->capture_aux, cudaStreamNonBlocking));
  uint64_t push_launches = 0, empty_launches = 0;
  std::vector<cudaGraphNode_t> if_nodes;  // (cudaGraphNodeGetType fails on them: skipped below)
  // an IF node after the captured work so far; its body captured from `fill`
  // on the capture-only stream; returns the kernels launched in it
  auto add_if = [&](cudaGraphConditionalHandle hc, const std::function<void(cudaStream_t)>& fill) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    DYNPR_CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams ip{};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hc;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t ifn;
    DYNPR_CK(cudaGraphAddNode(&ifn, cg, deps, nd, &ip));
    if_nodes.push_back(ifn);
    DYNPR_CK(cudaStreamUpdateCaptureDependencies(st, &ifn, 1, cudaStreamSetCaptureDependencies));
    const uint64_t l0 = ctx->launches;
    DYNPR_CK(cudaStreamBeginCaptureToGraph(ctx->capture_aux, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    fill(ctx->capture_aux);
    cudaGraph_t ib = nullptr;
    DYNPR_CK(cudaStreamEndCapture(ctx->capture_aux, &ib));
    const uint64_t used = ctx->launches - l0;
    ctx->launches = l0;
    return used;
  };
  DYNPR_CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  try {
    // body_sweeps() per body (an even number: the ping-pong parity of every
    // position is fixed)
    for (int k = 0; k < nb; ++k) {
      const int half = k & 1;
      launch_sweep_ind(ctx, plan, half, tick);  // the record is zero: before the launch, then k_loop_end
      launch_loop_end(ctx, dc, red, cond, k == nb - 1, frontier ? hpush[k] : 0, frontier,
                      end_check ? hempty[k] : 0, end_check);
      if (frontier) {
        push_launches = add_if(hpush[k], [&](cudaStream_t s) { launch_expand_ind(ctx, half, dc, s); });
        if (end_check)
          empty_launches = add_if(hempty[k], [&](cudaStream_t s) {
            launch_empty_check(ctx, dc, half, s, cond, k == nb - 1);
          });
        if (!plan.pull_fused) launch_pull_ind(ctx, plan, half);  // (else: inside the next sweep)
      }
    }
  } catch (...) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(st, &junk);
    if (ctx->capture_aux) cudaStreamEndCapture(ctx->capture_aux, &junk);
    cudaGetLastError();
    throw;  // (the half-built graph is leaked: destroying it crashes in the driver)
  }
  cudaGraph_t captured = nullptr;
  DYNPR_CK(cudaStreamEndCapture(st, &captured));
  {  // the multi-chunk sweep branch first: highest node priority
    size_t cnt = 0;
    DYNPR_CK(cudaGraphGetNodes(body, nullptr, &cnt));
    std::vector<cudaGraphNode_t> nodes(cnt);
    DYNPR_CK(cudaGraphGetNodes(body, nodes.data(), &cnt));
    int lo = 0, hi = 0;
    DYNPR_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (cudaGraphNode_t nd : nodes) {
      if (std::find(if_nodes.begin(), if_nodes.end(), nd) != if_nodes.end()) continue;
      cudaGraphNodeType t;
      DYNPR_CK(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      DYNPR_CK(cudaGraphKernelNodeGetParams(nd, &kp));
      if (!is_priority_sweep_kernel(kp.func)) continue;
      cudaLaunchAttributeValue v{};
      v.priority = hi;
      DYNPR_CK(cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributePriority, &v));
    }
  }
  DYNPR_CK(cudaGraphInstantiate(&lg.exec, lg.g, 0));
  lg.launches_per_body = ctx->launches - launches0;
  lg.launches_per_push = push_launches;
  lg.launches_per_empty_check = empty_launches;
  ctx->launches = launches0;
  cache->items.push_back(lg);
  return cache->items.back();
}

// Returns true when the last iteration was accounted without its sweep
// (k_loop_end: nothing left affected); the result is then R[(iterations - 1) & 1].
bool run_device_loop(dynpr_context* ctx, const SolveSpec& sp, const SweepArgs& a_in, double* const R[2],
                     double* const CB[2], const Layout* L, SweepRed* red, dynpr_stats& res) {
  const dynpr_config& c = *sp.cfg;
  cudaStream_t st = ctx->stream;
  LoopCtl h{};
  h.max_iter = c.max_iterations;
  h.check = c.convergence_check_disabled ? 0 : 1;
  h.frontier = sp.flagged && !sp.traversal;
  h.flagged = sp.flagged;
  h.tol = c.iteration_tolerance;
  h.m = sp.gT->m;
  h.n = sp.gT->n;
  LoopCtl* dc = ctx->loopctl.as<LoopCtl>(1);
  // the constant-bank argument slots are per device: one device-loop solve
  // at a time per GPU in this process
  std::lock_guard<std::mutex> guard(loop_slot_lock(ctx->device));
  prepare_sweep_launch(ctx);  // allocations / attributes must not happen inside a capture

  SweepArgs half[2] = {a_in, a_in};
  for (int k = 0; k < 2; ++k) {
    half[k].rank_prev = R[k];
    half[k].rank_cur = R[k ^ 1];
    half[k].contrib_prev = CB[k];
    half[k].contrib_cur = CB[k ^ 1];
    half[k].npeers = 0;
    half[k].done = &dc->done;
    half[k].expand = &dc->expand;
    half[k].begF = L->begF;
    half[k].tgtF = L->tgtF;
    half[k].tick_sm = sweep_tick(ctx);
  }
  // In-sweep pull (SweepArgs::pull_fused): a pull-mode expansion is folded
  // into the next sweep's gathers, pending flags ride in the contributions'
  // sign bits (no pull pass, no pending byte array).
  // DYNPR_PULL_FUSED=0 keeps the separate pull kernels (A/B).
  const bool want_pf = h.frontier && pull_fused_enabled();
  for (int k = 0; k < 2; ++k) half[k].pull_fused = want_pf ? 1 : 0;
  const SweepPlan plan = plan_sweep(ctx, half[0], sp.flagged, sp.closed);
  const char* ll = std::getenv("DYNPR_LAZY_LISTS");
  const bool lazy = plan.pull_fused && !(ll && ll[0] == '0');
  for (int k = 0; k < 2; ++k) {
    half[k].pull_fused = plan.pull_fused;
    half[k].lazy_lists = lazy ? 1 : 0;
    if (plan.pull_fused) half[k].np = nullptr;
  }
  h.lazy_lists = lazy ? 1 : 0;
  h.push_cost = push_cost_factor();
  LoopGraph& lg = loop_graph(ctx, plan, h.frontier, dc, red);

  // per-solve state: loop control + both halves' arguments, one upload
  static_assert(sizeof(LoopCtl) <= 1024 && 2 * sizeof(SweepArgs) <= 2048, "pinned staging layout");
  char* stage = static_cast<char*>(ctx->pinned);
  std::memcpy(stage + 1024, &h, sizeof h);
  std::memcpy(stage + 2048, half, sizeof half);
  DYNPR_CK(cudaMemcpyAsync(dc, stage + 1024, sizeof h, cudaMemcpyHostToDevice, st));
  DYNPR_CK(cudaMemsetAsync(red, 0, sizeof(SweepRed), st));
  upload_loop_args(ctx, reinterpret_cast<const SweepArgs*>(stage + 2048));
  DYNPR_CK(cudaGraphLaunch(lg.exec, st));
  DYNPR_CK(cudaMemcpyAsync(stage + 1024, dc, sizeof h, cudaMemcpyDeviceToHost, st));
  sync(ctx);
  std::memcpy(&h, stage + 1024, sizeof h);
  // launches: the captured body (two iterations) ran once per two sweeps
  ctx->launches += lg.launches_per_body * (uint64_t)((h.iterations + body_sweeps(plan) - 1) / body_sweeps(plan)) +
                   lg.launches_per_push * h.pushes + lg.launches_per_empty_check * h.empty_checks;
  res.iterations = h.iterations;
  res.converged = h.converged;
  res.affected_vertex_iterations = h.affected;
  res.processed_edges = h.edges;
  res.final_delta = h.final_delta;
  return h.skipped != 0;
}

// Snapshot preparation also readies the solves that follow (single GPU,
// device loop): the engine workspace at this graph's size and the
// instantiated loop graphs of Static and of the frontier engines (DF-P,
// DF) for this layout's sweep plan, so a first solve pays neither
// allocations nor a graph capture + instantiation (RMAT-20: the first DF-P
// of a process took ~20 ms of device time, the next 0.6).  Both are cached
// on the context and reused by every snapshot of the same shape.
void prewarm_solves(dynpr_context* ctx, const Layout* L, uint64_t m, bool frontier) {
  const uint32_t n = L->n;
  for (int k = 0; k < 2; ++k) {
    ctx->rank[k].as<double>(n);
    ctx->contrib[k].as<double>(n);
  }
  double* partials = ctx->partials.as<double>(L->n_mseg + 1);
  SweepRed* red = ctx->red.as<SweepRed>(2);
  LoopCtl* dc = ctx->loopctl.as<LoopCtl>(1);
  if (frontier) {
    ctx->flags_va.as<uint8_t>((uint64_t)n + 4);
    ctx->pend_flags.as<uint8_t>(n);
    ctx->flags_written.as<uint8_t>(n);
    ctx->pend_low.as<uint32_t>((uint64_t)n + 1);
    ctx->pend_high.as<uint2>((uint64_t)n + m / kExpandChunk + 1);
  }
  std::lock_guard<std::mutex> guard(loop_slot_lock(ctx->device));
  prepare_sweep_launch(ctx);
  const bool want_pf = pull_fused_enabled();
  const int kinds[3][2] = {{0, 0}, {1, 1}, {1, 0}};  // (flagged, closed): Static / ND, DF-P, DF
  for (int i = 0; i < (frontier ? 3 : 1); ++i) {
    SweepArgs a = layout_args(L, partials);
    a.pull_fused = kinds[i][0] && want_pf ? 1 : 0;
    const SweepPlan plan = plan_sweep(ctx, a, kinds[i][0] != 0, kinds[i][1] != 0);
    loop_graph(ctx, plan, kinds[i][0], dc, red);
  }
}

// convergeLoop (engine.cu:61-95) on the device, in the layout's new-id
// space; inputs are permuted in and the result permuted back out.
void solve_impl(dynpr_context* ctx, const SolveSpec& sp, double* ranks_out, dynpr_stats* stats,
                dynpr_observer obs, void* user) {
  const dynpr_graph* gT = sp.gT;
  const dynpr_graph* gF = sp.gF;
  const dynpr_config& c = *sp.cfg;
  const uint32_t n = gT->n;
  cudaStream_t st = ctx->stream;
  // The engine layout is part of the device graph format (built at ingest
  // or by dynpr_graph_prepare); an uncached build is timed with the solve.
  DYNPR_CK(cudaEventRecord(ctx->ev_a, st));
  // a team expands by pull over its own in-lists: only the traversal engine
  // (markReachable) reads the relabelled forward CSR there
  const Layout* L = [&] {
    NvtxRange r("dynpr layout");
    return get_layout(ctx, gT, gF, c.low_degree_threshold, is_team(ctx) ? sp.traversal : sp.flagged);
  }();
  // workspace (allocation is excluded from the timed region)
  double* R[2] = {ctx->rank[0].as<double>(n), ctx->rank[1].as<double>(n)};
  // Multi-GPU with attached peer buffers: contributions live in the
  // peer-mapped buffers and each sweep stores its new values straight into
  // every rank's copy (fused exchange); otherwise they are all-gathered.
  Comm* comm = ctx->comm;
  const bool dist = comm && (comm->world > 1 || team_forced());
  const bool fused = dist && (int)ctx->peer_cb[0].size() == comm->world && ctx->peer_capacity >= n;
  double* CB[2] = {fused ? ctx->peer_cb[0][comm->rank] : ctx->contrib[0].as<double>(n),
                   fused ? ctx->peer_cb[1][comm->rank] : ctx->contrib[1].as<double>(n)};
  // Device-driven loop (CUDA graph WHILE node, no host round trip per
  // iteration) unless the caller needs the host in the loop: an observer,
  // a multi-GPU team (host-orchestrated collectives), per-sweep profiling.
  const bool device_loop = !obs && !dist && !ctx->profiling && !host_loop_forced();
  double* partials = ctx->partials.as<double>(L->n_mseg + 1);
  SweepRed* red = ctx->red.as<SweepRed>(2);
  uint8_t* va = nullptr;
  uint8_t* np = nullptr;
  uint8_t* written = nullptr;
  uint32_t* pl = nullptr;
  uint2* ph = nullptr;
  if (sp.flagged) {
    va = ctx->flags_va.as<uint8_t>((uint64_t)n + 4);  // +4: word-wide claims (markReachable)
    np = ctx->pend_flags.as<uint8_t>(n);
    written = ctx->flags_written.as<uint8_t>(n);
    pl = ctx->pend_low.as<uint32_t>((uint64_t)n + 1);
    // every high out-degree vertex contributes ceil(outdeg/1024) items
    ph = ctx->pend_high.as<uint2>((uint64_t)n + gT->m / kExpandChunk + 1);
  }
  std::vector<double> h_ranks;
  std::vector<uint8_t> h_flags;
  double* obs_ranks = nullptr;
  uint8_t* obs_flags = nullptr;
  if (obs) {
    h_ranks.resize(n);
    obs_ranks = ctx->stage_c.as<double>(n);
    if (sp.flagged) {
      h_flags.resize(n);
      obs_flags = ctx->flags_np.as<uint8_t>(2ull * n);
    }
  }
  // initRanksUniform / initRanksFrom (rank.cpp:22-37) + contributions
  // (the second buffers only where a sweep may leave vertices unwritten:
  // frontier engines; a plain sweep writes every owned vertex)
  launch_init_ranks(ctx, L, sp.prev, 1.0 / (double)n, R[0], sp.flagged ? R[1] : nullptr, CB[0],
                    sp.flagged ? CB[1] : nullptr);
  if (sp.flagged) {
    DYNPR_CK(cudaMemsetAsync(written, 0, n, st));
    if (sp.flags_in) {
      launch_gather_perm_u8(ctx, L, sp.flags_in, va);
    } else if (sp.traversal) {
      // markReachable over the relabelled forward CSR (frontier.cpp:86-121)
      DYNPR_CK(cudaMemsetAsync(va, 0, n, st));
      mark_reachable(ctx, Rows{L->begF, L->outdeg, L->tgtF}, n, L->m, L->inv, sp.seeds, sp.nseeds, va);
    } else {
      // initialAffected + the one expandAffected before the loop
      // (engine.cpp:199-200)
      DYNPR_CK(cudaMemsetAsync(va, 0, n, st));
      DYNPR_CK(cudaMemsetAsync(np, 0, n, st));
      DYNPR_CK(cudaMemsetAsync(red + 1, 0, sizeof(SweepRed), st));
      launch_init_affected(ctx, L->inv, sp.ds, sp.dd, sp.nd, sp.is, sp.ni, va, np);
      if (!dist) {  // (a team expands by pull into its own rows, below)
        launch_collect_pending(ctx, L->outdeg, nullptr, n, np, c.low_degree_threshold, pl, ph, red + 1);
        if (device_loop) {  // list sizes stay on the device
          launch_expand_dev(ctx, Rows{L->begF, L->outdeg, L->tgtF}, va, pl, ph, &red[1].pend_low, nullptr);
        } else {
          const SweepRed r0 = read_red(ctx, red + 1);
          launch_expand(ctx, Rows{L->begF, L->outdeg, L->tgtF}, va, pl, r0.pend_low, ph, r0.pend_high);
        }
      }
    }
  }

  SweepArgs a = layout_args(L, partials);
  a.alpha = c.damping_factor;
  a.teleport = (1.0 - c.damping_factor) / (double)n;  // rank.cpp:85
  a.tf = c.frontier_tolerance;
  a.tp = c.prune_tolerance;
  a.va = va;
  a.np = sp.traversal ? nullptr : np;  // pending flags (new ids) for pull expansion
  a.written = written;
  a.pend_low = sp.traversal ? nullptr : pl;
  a.pend_high = sp.traversal ? nullptr : ph;
  a.red = red;

  // Multi-GPU: this rank sweeps only its edge-balanced vertex
  // range; contributions (and DF pending flags) are all-gathered after
  // every sweep and the reduction record all-reduced, so every rank takes
  // the same convergence / expansion decisions.
  std::vector<uint64_t> off_c, off_f;  // allgatherv byte offsets: f64 / u8 per vertex
  FlagBitmapPlan fplan;
  uint32_t* fbits = nullptr;
  uint32_t* fbounds = nullptr;
  if (dist) {
    const std::vector<RankRange> plan = plan_ranges(ctx, const_cast<Layout*>(L), comm->world);
    const RankRange& me = plan[comm->rank];
    a.v_lo = me.v_lo;
    a.v_hi = me.v_hi;
    a.ss_lo = me.ss_lo;
    a.ss_hi = me.ss_hi;
    a.ms_lo = me.ms_lo;
    a.ms_hi = me.ms_hi;
    off_c.resize(comm->world + 1);
    off_f.resize(comm->world + 1);
    for (int r = 0; r < comm->world; ++r) {
      off_c[r] = 8ull * plan[r].v_lo;
      off_f[r] = plan[r].v_lo;
    }
    off_c[comm->world] = 8ull * n;
    off_f[comm->world] = n;
    if (sp.flagged && !sp.traversal) {
      std::vector<uint32_t> lo(comm->world);
      for (int r = 0; r < comm->world; ++r) lo[r] = plan[r].v_lo;
      fplan = make_flag_bitmap_plan(lo, n);
      fbits = ctx->flag_bits.as<uint32_t>(fplan.words + 1);
      fbounds = ctx->flag_bounds.as<uint32_t>(fplan.host_bounds.size());
      DYNPR_CK(cudaMemcpyAsync(fbounds, fplan.host_bounds.data(), 4 * fplan.host_bounds.size(),
                               cudaMemcpyHostToDevice, st));
    }
  }
  // DF/DF-P pending flags: packed to bits, all-gathered, unpacked into the
  // other ranks' ranges (n/8 bytes per sweep on the wire)
  auto exchange_flags = [&] {
    const int me = comm->rank;
    launch_pack_flags(ctx, np, fplan.host_bounds[me], fplan.host_bounds[me + 1],
                      fbits + fplan.host_bounds[comm->world + 1 + me]);
    comm->allgatherv(fbits, fplan.byte_off.data(), st);
    launch_unpack_flags(ctx, fbits, fbounds, comm->world, me, n, np);
  };
  if (dist) team_check_graph(ctx, comm, const_cast<Layout*>(L), gT, gF, red);
  if (dist && sp.flagged && !sp.traversal && !sp.flags_in) {
    // initial expandAffected (engine.cpp:199-200) as a pull: every rank holds
    // the batch's pending flags (replicated), and marks its own rows
    SweepArgs a0 = a;
    a0.red = red + 1;  // zeroed above: the pull work queue starts at 0
    launch_pull_expand(ctx, a0);
  }

  if (fused) {
    // Team barrier: no rank may store into a peer's buffers before that
    // peer has initialised them (an all-reduce of a zeroed record is
    // stream-ordered after this rank's init on every rank).
    DYNPR_CK(cudaMemsetAsync(red, 0, sizeof(SweepRed), st));
    comm->allreduce_red(red, st);
  }

  // The in-sweep pull in the host-driven loop too (single GPU and teams;
  // not with an observer, which is shown the affected set before each sweep
  // -- an in-sweep pull completes it only during the sweep): the pending
  // flags ride in the contributions' sign bits, which a team's contribution
  // exchange already carries, so a team exchanges no pending-flag bitmap and
  // runs no separate pull pass.  The decision for the next sweep is a device
  // int the sweeps read (LoopCtl::expand).
  const bool host_pf = !device_loop && sp.flagged && !sp.traversal && !obs && pull_fused_enabled();
  int* expand_dev = nullptr;
  if (host_pf) {
    expand_dev = &ctx->loopctl.as<LoopCtl>(1)->expand;
    launch_set_expand(ctx, expand_dev, kExpandNone);
    a.pull_fused = 1;
    a.expand = expand_dev;
    a.np = nullptr;  // (the batch's flags served the expansion before the loop)
    if (dist) {
      a.pend_low = nullptr;  // a team never pushes
      a.pend_high = nullptr;
    } else {
      a.lazy_lists = 1;
    }
  }

  dynpr_stats res{};
  int cur = 0;  // R[cur] holds the latest iterate ("previous")
  if (device_loop) {
    NvtxRange r("dynpr device loop");
    const bool skipped = run_device_loop(ctx, sp, a, R, CB, L, red, res);
    cur = (res.iterations - (skipped ? 1 : 0)) & 1;
  }
  // Multi-GPU team, no observer / profiling: the host-driven loop runs one
  // iteration ahead -- iteration k+1 (sweep, collectives, pull expansion) is
  // enqueued before iteration k's record is read back, so no host round trip
  // sits between two sweeps.  Safe because nothing enqueued depends on a host
  // decision: teams always expand by pull, and an iteration enqueued after
  // convergence only overwrites the buffers of the iterate before last (the
  // result R[iterations & 1] is untouched; flags are not results).  The
  // stream-ordered record all-reduce stays the team barrier of the fused
  // exchange.  Every rank enqueues the same sequence of collectives.
  const bool speculative = !device_loop && dist && !obs && !ctx->profiling;
  if (speculative) {
    for (int k = 0; k < 2; ++k)
      if (!ctx->ev_rec[k]) DYNPR_CK(cudaEventCreateWithFlags(&ctx->ev_rec[k], cudaEventDisableTiming));
    auto* slot = reinterpret_cast<SweepRed*>(static_cast<char*>(ctx->pinned) + 512);  // 2 records
    auto enqueue = [&](int k) {
      SweepRed* rk = red + (k & 1);
      const int cu = k & 1;
      DYNPR_CK(cudaMemsetAsync(rk, 0, sizeof(SweepRed), st));
      SweepArgs ak = a;
      ak.red = rk;
      ak.rank_prev = R[cu];
      ak.rank_cur = R[cu ^ 1];
      ak.contrib_prev = CB[cu];
      ak.contrib_cur = CB[cu ^ 1];
      ak.npeers = 0;
      if (fused)
        for (int q = 0; q < comm->world; ++q)
          if (q != comm->rank) ak.peer_cur[ak.npeers++] = ctx->peer_cb[cu ^ 1][q];
      launch_sweep(ctx, ak, sp.flagged, sp.closed);
      comm->allreduce_red(rk, st);
      if (!fused) comm->allgatherv(CB[cu ^ 1], off_c.data(), st);
      if (sp.flagged && !sp.traversal && !host_pf) exchange_flags();
      DYNPR_CK(cudaMemcpyAsync(slot + (k & 1), rk, sizeof(SweepRed), cudaMemcpyDeviceToHost, st));
      DYNPR_CK(cudaEventRecord(ctx->ev_rec[k & 1], st));
      if (sp.flagged && !sp.traversal) {
        if (host_pf) {
          if (k == 0) launch_set_expand(ctx, expand_dev, kExpandPull);  // every later sweep pulls
        } else {
          launch_pull_expand(ctx, ak);
        }
      }
    };
    enqueue(0);
    for (int iter = 0; iter < c.max_iterations; ++iter) {
      if (iter + 1 < c.max_iterations) enqueue(iter + 1);
      DYNPR_CK(cudaEventSynchronize(ctx->ev_rec[iter & 1]));
      SweepRed r;
      std::memcpy(&r, slot + (iter & 1), sizeof r);
      const double delta = bits_to_double(r.delta_bits);
      res.iterations = iter + 1;
      res.affected_vertex_iterations += sp.flagged ? r.processed : (uint64_t)n;
      res.processed_edges += r.edges;
      res.final_delta = delta;
      if (!c.convergence_check_disabled && delta <= c.iteration_tolerance) {
        res.converged = 1;
        break;
      }
    }
    cur = res.iterations & 1;
  }
  bool prev_pull = false;  // the last expansion was a pull (host_pf: the next sweep appends no lists)
  for (int iter = 0; !device_loop && !speculative && iter < c.max_iterations; ++iter) {
    DYNPR_CK(cudaMemsetAsync(red, 0, sizeof(SweepRed), st));
    if (obs && sp.flagged) {
      uint8_t* snap = obs_flags + n;  // owned entries are current on each rank
      DYNPR_CK(cudaMemcpyAsync(snap, va, n, cudaMemcpyDeviceToDevice, st));
      if (dist) comm->allgatherv(snap, off_f.data(), st);
      launch_scatter_inv_u8(ctx, L, snap, obs_flags);
      DYNPR_CK(cudaMemcpyAsync(h_flags.data(), obs_flags, n, cudaMemcpyDeviceToHost, st));
    }
    a.rank_prev = R[cur];
    a.rank_cur = R[cur ^ 1];
    a.contrib_prev = CB[cur];
    a.contrib_cur = CB[cur ^ 1];
    a.npeers = 0;
    if (fused) {
      for (int r = 0; r < comm->world; ++r)
        if (r != comm->rank) a.peer_cur[a.npeers++] = ctx->peer_cb[cur ^ 1][r];
    }
    if (ctx->profiling) DYNPR_CK(cudaEventRecord(ctx->ev_s0, st));
    launch_sweep(ctx, a, sp.flagged, sp.closed);
    if (ctx->profiling) DYNPR_CK(cudaEventRecord(ctx->ev_s1, st));
    if (dist) {
      comm->allreduce_red(red, st);  // also the team barrier of the fused exchange
      if (!fused) comm->allgatherv(CB[cur ^ 1], off_c.data(), st);
      if (sp.flagged && !sp.traversal && !host_pf) exchange_flags();
      if (obs) comm->allgatherv(R[cur ^ 1], off_c.data(), st);
    }
    const SweepRed r = read_red(ctx, red);
    if (ctx->profiling) {
      float ms = 0.f;
      DYNPR_CK(cudaEventElapsedTime(&ms, ctx->ev_s0, ctx->ev_s1));
      ctx->sweep_ms += ms;
      ctx->sweeps += 1;
      // algorithmic bytes of the sweep: 4 B per gathered in-edge
      // id + 28 B per processed vertex (8 offset, 4 out-degree, 8 R_prev,
      // 8 R_new) [+ 1 B flag read per vertex in frontier mode]
      ctx->sweep_bytes += 4ull * r.edges + 28ull * r.processed + 8ull + (sp.flagged ? (uint64_t)n : 0ull);
    }
    const double delta = bits_to_double(r.delta_bits);
    cur ^= 1;  // swap (engine.cpp:80)
    res.iterations = iter + 1;
    res.affected_vertex_iterations += sp.flagged ? r.processed : (uint64_t)n;
    res.processed_edges += r.edges;
    res.final_delta = delta;
    if (obs) {
      launch_scatter_inv_f64(ctx, L, R[cur], obs_ranks);
      DYNPR_CK(cudaMemcpyAsync(h_ranks.data(), obs_ranks, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
      sync(ctx);
      obs(res.iterations, h_ranks.data(), sp.flagged ? h_flags.data() : nullptr, n, user);
    }
    if (!c.convergence_check_disabled && delta <= c.iteration_tolerance) {
      res.converged = 1;
      break;
    }
    if (sp.flagged && !sp.traversal) {  // expandAffected (engine.cpp:91), direction-optimising
      // push touches the pending vertices' out-edges; pull scans at most
      // the in-edges of the vertices that were not processed this sweep
      const uint64_t pull_bound = gT->m > r.edges ? gT->m - r.edges : 0;
      // multi-GPU: pending flags are replicated, each rank pulls into its
      // own rows (no remote writes)
      const bool pull = dist || r.pend_edges * (uint64_t)push_cost_factor() > pull_bound;
      if (host_pf) {  // a pull happens inside the next sweep
        if (pull) {
          launch_set_expand(ctx, expand_dev, kExpandPull);
        } else {
          SweepRed lists = r;
          if (prev_pull) {  // a pull sweep appended no lists: collect them from the sign bits
            launch_collect_signs(ctx, a, red + 1);
            lists = read_red(ctx, red + 1);
          }
          launch_expand(ctx, Rows{L->begF, L->outdeg, L->tgtF}, va, pl, lists.pend_low, ph, lists.pend_high);
          launch_set_expand(ctx, expand_dev, kExpandPush);
        }
        prev_pull = pull;
      } else if (pull) {
        launch_pull_expand(ctx, a);
      } else {
        launch_expand(ctx, Rows{L->begF, L->outdeg, L->tgtF}, va, pl, r.pend_low, ph, r.pend_high);
      }
      if (pull) ctx->pull_expansions += 1;
    }
  }
  // result back to old ids (R[cur ^ 1] is free and receives the permuted copy
  // when the caller's buffer is on the host)
  const bool host_out = !is_device_ptr(ranks_out);
  double* out_dev = host_out ? R[cur ^ 1] : ranks_out;
  if (dist) comm->allgatherv(R[cur], off_c.data(), st);  // every rank returns the full vector
  launch_scatter_inv_f64(ctx, L, R[cur], out_dev);
  DYNPR_CK(cudaEventRecord(ctx->ev_b, st));
  if (host_out) DYNPR_CK(cudaMemcpyAsync(ranks_out, out_dev, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  sync(ctx);
  float ms = 0.f;
  DYNPR_CK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
  res.device_ms = ms;
  if (stats) *stats = res;
}

// A team rank that fails mid-solve releases the others (host-side barriers
// of the team throw instead of waiting for it), then rethrows.
void solve(dynpr_context* ctx, const SolveSpec& sp, double* ranks_out, dynpr_stats* stats, dynpr_observer obs,
           void* user) {
  try {
    solve_impl(ctx, sp, ranks_out, stats, obs, user);
  } catch (...) {
    if (is_team(ctx)) ctx->comm->abort();
    throw;
  }
}

}  // namespace
}  // namespace dynpr_b200

using namespace dynpr_b200;

void dynpr_b200::context_teardown(dynpr_context* ctx) {
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->side) cudaStreamSynchronize(ctx->side);
  delete ctx->comm;
  ctx->comm = nullptr;
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
  if (ctx->ev_s0) cudaEventDestroy(ctx->ev_s0);
  if (ctx->ev_s1) cudaEventDestroy(ctx->ev_s1);
  delete static_cast<LoopGraphCache*>(ctx->loop_graphs);
  ctx->loop_graphs = nullptr;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->capture_aux) cudaStreamDestroy(ctx->capture_aux);
  if (ctx->aux) {
    cudaStreamSynchronize(ctx->aux);
    cudaStreamDestroy(ctx->aux);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_side) cudaEventDestroy(ctx->ev_side);
  for (auto& e : ctx->ev_rec)
    if (e) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

extern "C" {

const char* dynpr_last_error(void) { return g_last_error.c_str(); }
const char* dynpr_version(void) { return "dynpr_b200 0.1 (sm_100a)"; }

void dynpr_config_default(dynpr_config* c) {
  if (!c) return;
  c->damping_factor = 0.85;
  c->iteration_tolerance = 1e-10;
  c->frontier_tolerance = 1e-6;
  c->prune_tolerance = 1e-6;
  c->max_iterations = 500;
  c->low_degree_threshold = 32;
  c->partition_strategy = DYNPR_PARTITION_BOTH;
  c->convergence_check_disabled = 0;
}

dynpr_status dynpr_config_validate(const dynpr_config* c) {
  return api_guard([&] { validate_config(c); });
}

dynpr_status dynpr_context_create(int device, dynpr_context** out) {
  return api_guard([&] {
    if (!out) invalid("null argument");
    int count = 0;
    DYNPR_CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) invalid("dynpr_context_create: no such CUDA device");
    DYNPR_CK(cudaSetDevice(device));
    auto* ctx = new dynpr_context();
    ctx->device = device;
    try {
      DYNPR_CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
      DYNPR_CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      // keep freed snapshot memory reserved in the stream-ordered pool
      cudaMemPool_t pool;
      DYNPR_CK(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = ~0ull;
      DYNPR_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      DYNPR_CK(cudaEventCreate(&ctx->ev_a));
      DYNPR_CK(cudaEventCreate(&ctx->ev_b));
      DYNPR_CK(cudaEventCreate(&ctx->ev_s0));
      DYNPR_CK(cudaEventCreate(&ctx->ev_s1));
      DYNPR_CK(cudaMallocHost(&ctx->pinned, 8192));  // [4096, 8192): ingest status slots (graph.cu)
    } catch (...) {
      dynpr_context_destroy(ctx);
      throw;
    }
    *out = ctx;
  });
}

// ---- multi-GPU contexts ------------------------------------------------------------
struct dynpr_team {
  std::shared_ptr<dynpr_b200::LocalTeam> team;
};

dynpr_status dynpr_nccl_get_unique_id(uint8_t* id128) {
  if (!id128) {
    set_last_error("null argument");
    return DYNPR_INVALID_ARGUMENT;
  }
  return nccl_unique_id(id128);
}

dynpr_status dynpr_context_create_nccl(int device, int rank, int world, const uint8_t* id128,
                                       dynpr_context** out) {
  dynpr_status st = dynpr_context_create(device, out);
  if (st != DYNPR_OK) return st;
  st = api_guard([&] {
    if (world < 1 || rank < 0 || rank >= world || !id128) invalid("dynpr_context_create_nccl: bad rank/world");
    (*out)->comm = make_nccl_comm(rank, world, id128).release();
  });
  if (st != DYNPR_OK) {
    dynpr_context_destroy(*out);
    *out = nullptr;
  }
  return st;
}

dynpr_status dynpr_team_create(int world, dynpr_team** out) {
  return api_guard([&] {
    if (!out || world < 1) invalid("dynpr_team_create: bad world size");
    *out = new dynpr_team{make_local_team(world)};
  });
}

dynpr_status dynpr_team_destroy(dynpr_team* t) {
  return api_guard([&] { delete t; });
}

dynpr_status dynpr_context_create_team(int device, dynpr_team* team, int rank, dynpr_context** out) {
  dynpr_status st = dynpr_context_create(device, out);
  if (st != DYNPR_OK) return st;
  st = api_guard([&] {
    if (!team || rank < 0 || rank >= local_team_world(*team->team)) invalid("dynpr_context_create_team: bad rank");
    (*out)->comm = make_local_comm(team->team, rank, device).release();
  });
  if (st != DYNPR_OK) {
    dynpr_context_destroy(*out);
    *out = nullptr;
  }
  return st;
}

dynpr_status dynpr_context_create_hostcomm(int device, int rank, int world, const dynpr_comm_ops* ops, void* user,
                                           dynpr_context** out) {
  if (!out) {
    set_last_error("null argument");
    return DYNPR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world || !ops || !ops->allreduce_u64 || !ops->allgatherv || !ops->barrier) {
    set_last_error("dynpr_context_create_hostcomm: bad rank/world or missing transport callback");
    return DYNPR_INVALID_ARGUMENT;
  }
  dynpr_status st = dynpr_context_create(device, out);
  if (st != DYNPR_OK) return st;
  st = api_guard([&] { (*out)->comm = make_host_comm(rank, world, *ops, user).release(); });
  if (st != DYNPR_OK) {
    dynpr_context_destroy(*out);
    *out = nullptr;
  }
  return st;
}

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");

dynpr_status dynpr_ipc_alloc(dynpr_context* ctx, uint64_t bytes, void** dptr, uint8_t* handle64) {
  return api_guard([&] {
    if (!ctx || !dptr || !handle64 || !bytes) invalid("dynpr_ipc_alloc: null argument or zero size");
    DYNPR_CK(cudaSetDevice(ctx->device));
    void* p = nullptr;
    DYNPR_CK(cudaMalloc(&p, bytes));  // IPC needs a plain cudaMalloc allocation (not the stream pool)
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      DYNPR_CK(e);
    }
    std::memcpy(handle64, &h, 64);
    *dptr = p;
  });
}

dynpr_status dynpr_ipc_open(dynpr_context* ctx, const uint8_t* handle64, void** dptr) {
  return api_guard([&] {
    if (!ctx || !dptr || !handle64) invalid("dynpr_ipc_open: null argument");
    DYNPR_CK(cudaSetDevice(ctx->device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    DYNPR_CK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

dynpr_status dynpr_ipc_close(dynpr_context* ctx, void* dptr) {
  return api_guard([&] {
    if (!ctx || !dptr) invalid("dynpr_ipc_close: null argument");
    DYNPR_CK(cudaSetDevice(ctx->device));
    DYNPR_CK(cudaIpcCloseMemHandle(dptr));
  });
}

dynpr_status dynpr_ipc_free(dynpr_context* ctx, void* dptr) {
  return api_guard([&] {
    if (!ctx || !dptr) invalid("dynpr_ipc_free: null argument");
    DYNPR_CK(cudaSetDevice(ctx->device));
    DYNPR_CK(cudaFree(dptr));
  });
}

dynpr_status dynpr_context_attach_peers(dynpr_context* ctx, int world, const uint64_t* ptrs0, const uint64_t* ptrs1,
                                        uint64_t capacity) {
  return api_guard([&] {
    if (!ctx) invalid("null context");
    ctx->peer_cb[0].clear();
    ctx->peer_cb[1].clear();
    ctx->peer_capacity = 0;
    if (world == 0) return;  // detach
    const int team = ctx->comm ? ctx->comm->world : 1;
    if (world != team || !ptrs0 || !ptrs1) invalid("dynpr_context_attach_peers: world does not match the team");
    if (world - 1 > kMaxPeers) invalid("dynpr_context_attach_peers: team larger than kMaxPeers + 1");
    for (int r = 0; r < world; ++r) {
      if (!ptrs0[r] || !ptrs1[r]) invalid("dynpr_context_attach_peers: null buffer");
      ctx->peer_cb[0].push_back(reinterpret_cast<double*>(ptrs0[r]));
      ctx->peer_cb[1].push_back(reinterpret_cast<double*>(ptrs1[r]));
    }
    ctx->peer_capacity = capacity;
  });
}

dynpr_status dynpr_context_rank(const dynpr_context* ctx, int* rank, int* world) {
  return api_guard([&] {
    if (!ctx) invalid("null context");
    if (rank) *rank = ctx->comm ? ctx->comm->rank : 0;
    if (world) *world = ctx->comm ? ctx->comm->world : 1;
  });
}

dynpr_status dynpr_context_destroy(dynpr_context* ctx) {
  return api_guard([&] {
    if (!ctx) return;
    ctx->closing.store(true);
    // graphs still alive: the last one's destroy tears the context down
    if (ctx->live_graphs.load() == 0 && !ctx->torn_down.exchange(true)) context_teardown(ctx);
  });
}


uint64_t dynpr_context_launches(const dynpr_context* ctx) { return ctx ? ctx->launches : 0; }

dynpr_status dynpr_context_set_profiling(dynpr_context* ctx, int enable) {
  return api_guard([&] {
    if (!ctx) invalid("null context");
    ctx->profiling = enable != 0;
    ctx->sweep_ms = 0.0;
    ctx->sweeps = 0;
    ctx->sweep_bytes = 0;
  });
}

dynpr_status dynpr_context_sweep_times(dynpr_context* ctx, double* total_ms, uint64_t* sweeps, uint64_t* bytes) {
  return api_guard([&] {
    if (!ctx) invalid("null context");
    if (total_ms) *total_ms = ctx->sweep_ms;
    if (sweeps) *sweeps = ctx->sweeps;
    if (bytes) *bytes = ctx->sweep_bytes;
  });
}

// ---- primitives ---------------------------------------------------------------
dynpr_status dynpr_partition_by_degree(dynpr_context* ctx, const dynpr_graph* g, uint32_t threshold,
                                       uint32_t* order, uint32_t* low_count) {
  NvtxRange nvtx__("dynpr_partition_by_degree");
  return api_guard([&] {
    if (!ctx || !g || !low_count) invalid("null argument");
    bind_device(ctx);
    StageOut<uint32_t> o(ctx, ctx->stage_a, order, g->n);
    Schedule s = build_partition(ctx, g, threshold, g->n ? o.dev : nullptr);
    o.commit();
    *low_count = s.n_low;
  });
}

dynpr_status dynpr_graph_prepare(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF,
                                 uint32_t threshold, int with_forward, double* build_ms) {
  NvtxRange nvtx__("dynpr_graph_prepare");
  return api_guard([&] {
    if (!ctx) invalid("null context");
    check_pair(gT, gF);
    bind_device(ctx);
    // team engines expand by pull: the forward CSR is left to the traversal
    // engine, which builds it on first use
    const Layout* L = get_layout(ctx, gT, gF, threshold, with_forward != 0 && !is_team(ctx));
    if (build_ms) *build_ms = L->build_ms;
    // a team's per-snapshot work (edge-balanced range plan, graph
    // fingerprint) belongs to the snapshot build, not to the first solve
    if (is_team(ctx)) {
      plan_ranges(ctx, const_cast<Layout*>(L), ctx->comm->world);
      ensure_fingerprint(ctx, const_cast<Layout*>(L), gT, gF);
    } else if (!host_loop_forced()) {
      prewarm_solves(ctx, L, gT->m, with_forward != 0);
    }
  });
}

dynpr_status dynpr_graph_layout_info(const dynpr_graph* gT, uint64_t* sell_words, uint32_t* v_lo, uint32_t* v_hi,
                                     int* has_forward, int* generation) {
  return api_guard([&] {
    if (!gT) invalid("null graph");
    const Layout* L = gT->layout.get();
    if (!L) invalid("dynpr_graph_layout_info: the graph has no engine layout yet (dynpr_graph_prepare)");
    if (sell_words) *sell_words = L->sell_words;
    if (v_lo) *v_lo = L->owned ? L->own.v_lo : 0u;
    if (v_hi) *v_hi = L->owned ? L->own.v_hi : L->n;
    if (has_forward) *has_forward = L->has_forward ? 1 : 0;
    if (generation) *generation = L->generation;
  });
}

dynpr_status dynpr_update_ranks(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF,
                                uint8_t* vertex_affected, uint8_t* neighbors_pending, const double* previous,
                                double* current, const dynpr_config* cfg, int mode) {
  NvtxRange nvtx__("dynpr_update_ranks");
  return api_guard([&] {
    if (!ctx || !gT || !gF || !cfg) invalid("null argument");
    if ((vertex_affected == nullptr) != (neighbors_pending == nullptr))
      invalid("updateRanks: pass both flag arrays or neither");
    bind_device(ctx);
    const uint32_t n = gT->n;
    if (n == 0) return;
    if (gF->n != n) invalid("engine: graph pair is not mutually transposed (count mismatch)");
    const Layout* L = get_layout(ctx, gT, gF, cfg->low_degree_threshold, false);
    if (L->owned)
      invalid("updateRanks: a team context holds only its rank's rows; call it on a single-GPU context");
    const double* prev = stage_in(ctx, ctx->stage_b, previous, n);
    double* R0 = ctx->rank[0].as<double>(n);
    double* R1 = ctx->rank[1].as<double>(n);
    double* C0 = ctx->contrib[0].as<double>(n);
    launch_init_ranks(ctx, L, prev, 0.0, R0, nullptr, C0, nullptr);
    const bool flagged = vertex_affected != nullptr;
    uint8_t* va = nullptr;
    uint8_t* np = nullptr;
    uint8_t* flag_old = nullptr;
    if (flagged) {
      va = ctx->flags_va.as<uint8_t>(n);
      np = ctx->flags_written.as<uint8_t>(n);
      flag_old = ctx->flags_np.as<uint8_t>(2ull * n);
      DYNPR_CK(cudaMemcpyAsync(flag_old, vertex_affected, n, cudaMemcpyDefault, ctx->stream));
      DYNPR_CK(cudaMemcpyAsync(flag_old + n, neighbors_pending, n, cudaMemcpyDefault, ctx->stream));
      launch_gather_perm_u8(ctx, L, flag_old, va);
      launch_gather_perm_u8(ctx, L, flag_old + n, np);
    }
    SweepRed* red = ctx->red.as<SweepRed>(2);
    DYNPR_CK(cudaMemsetAsync(red, 0, sizeof(SweepRed), ctx->stream));
    SweepArgs a = layout_args(L, ctx->partials.as<double>(L->n_mseg + 1));
    a.alpha = cfg->damping_factor;
    a.teleport = (1.0 - cfg->damping_factor) / (double)n;
    a.tf = cfg->frontier_tolerance;
    a.tp = cfg->prune_tolerance;
    a.rank_prev = R0;
    a.rank_cur = R1;
    a.contrib_prev = C0;
    a.contrib_cur = nullptr;
    a.va = va;
    a.np = np;
    a.written = nullptr;
    a.red = red;
    a.np_accumulate = 1;
    a.copy_all = 1;
    launch_sweep(ctx, a, flagged, mode == DYNPR_RANK_CLOSED_LOOP_PRUNE);
    StageOut<double> out(ctx, ctx->stage_c, current, n);
    launch_scatter_inv_f64(ctx, L, R1, out.dev);
    if (flagged) {
      launch_scatter_inv_u8(ctx, L, va, flag_old);
      launch_scatter_inv_u8(ctx, L, np, flag_old + n);
      DYNPR_CK(cudaMemcpyAsync(vertex_affected, flag_old, n, cudaMemcpyDefault, ctx->stream));
      DYNPR_CK(cudaMemcpyAsync(neighbors_pending, flag_old + n, n, cudaMemcpyDefault, ctx->stream));
    }
    out.commit();
  });
}

dynpr_status dynpr_linf_norm_delta(dynpr_context* ctx, const double* a, const double* b, uint64_t n, double* out) {
  return api_guard([&] {
    if (!ctx || !out) invalid("null argument");
    bind_device(ctx);
    const double* da = stage_in(ctx, ctx->stage_a, a, n);
    const double* db = stage_in(ctx, ctx->stage_b, b, n);
    auto* bits = ctx->scratch64a.as<unsigned long long>(1);
    launch_linf(ctx, da, db, n, bits);
    DYNPR_CK(cudaMemcpyAsync(ctx->pinned, bits, 8, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    unsigned long long h;
    std::memcpy(&h, ctx->pinned, 8);
    *out = bits_to_double(h);
  });
}

dynpr_status dynpr_l1_norm_delta(dynpr_context* ctx, const double* a, const double* b, uint64_t n, double* out) {
  return api_guard([&] {
    if (!ctx || !out) invalid("null argument");
    bind_device(ctx);
    const double* da = stage_in(ctx, ctx->stage_a, a, n);
    const double* db = stage_in(ctx, ctx->stage_b, b, n);
    double* part = ctx->stage_c.as<double>((n + 4095) / 4096 + 2);
    double* res = part + (n + 4095) / 4096 + 1;
    launch_l1(ctx, da, db, n, part, res);
    DYNPR_CK(cudaMemcpyAsync(ctx->pinned, res, 8, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    std::memcpy(out, ctx->pinned, 8);
  });
}

dynpr_status dynpr_initial_affected(dynpr_context* ctx, const dynpr_graph* g, const uint32_t* del_src,
                                    const uint32_t* del_dst, uint64_t n_del, const uint32_t* ins_src,
                                    const uint32_t* ins_dst, uint64_t n_ins, uint8_t* vertex_affected,
                                    uint8_t* neighbors_pending) {
  return api_guard([&] {
    if (!ctx || !g) invalid("null argument");
    bind_device(ctx);
    const uint32_t n = g->n;
    const uint32_t* ds = stage_in(ctx, ctx->batch[0], del_src, n_del);
    const uint32_t* dd = stage_in(ctx, ctx->batch[1], del_dst, n_del);
    const uint32_t* is = stage_in(ctx, ctx->batch[2], ins_src, n_ins);
    const uint32_t* id = stage_in(ctx, ctx->batch[3], ins_dst, n_ins);
    if (any_bad_ids(ctx, ds, dd, n_del, n)) invalid("initialAffected deletions: vertex id out of range");
    if (any_bad_ids(ctx, is, id, n_ins, n)) invalid("initialAffected insertions: vertex id out of range");
    StageOut<uint8_t> va(ctx, ctx->flags_va, vertex_affected, n);
    StageOut<uint8_t> np(ctx, ctx->flags_np, neighbors_pending, n);
    if (n) {
      DYNPR_CK(cudaMemsetAsync(va.dev, 0, n, ctx->stream));
      DYNPR_CK(cudaMemsetAsync(np.dev, 0, n, ctx->stream));
    }
    launch_init_affected(ctx, nullptr, ds, dd, n_del, is, n_ins, va.dev, np.dev);
    va.commit();
    np.commit();
  });
}

dynpr_status dynpr_expand_affected(dynpr_context* ctx, const dynpr_graph* g, uint8_t* vertex_affected,
                                   const uint8_t* neighbors_pending, uint32_t threshold) {
  NvtxRange nvtx__("dynpr_expand_affected");
  return api_guard([&] {
    if (!ctx || !g) invalid("null argument");
    bind_device(ctx);
    const uint32_t n = g->n;
    if (!n) return;
    const uint8_t* np = stage_in(ctx, ctx->flags_np, neighbors_pending, n);
    StageOut<uint8_t> va(ctx, ctx->flags_va, vertex_affected, n);
    if (va.host)
      DYNPR_CK(cudaMemcpyAsync(va.dev, vertex_affected, n, cudaMemcpyHostToDevice, ctx->stream));
    uint32_t* pl = ctx->pend_low.as<uint32_t>((uint64_t)n + 1);
    uint2* ph = ctx->pend_high.as<uint2>((uint64_t)n + g->m / kExpandChunk + 1);
    SweepRed* red = ctx->red.as<SweepRed>(2);
    DYNPR_CK(cudaMemsetAsync(red, 0, sizeof(SweepRed), ctx->stream));
    launch_collect_pending(ctx, nullptr, g->off, n, np, threshold, pl, ph, red);
    const SweepRed r = read_red(ctx, red);
    launch_expand(ctx, Rows{g->off, nullptr, g->tgt}, va.dev, pl, r.pend_low, ph, r.pend_high);
    va.commit();
  });
}

// ---- engines -------------------------------------------------------------------
dynpr_status dynpr_static_pagerank(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF,
                                   const dynpr_config* cfg, double* ranks_out, dynpr_stats* stats,
                                   dynpr_observer observer, void* observer_user) {
  NvtxRange nvtx__("dynpr_static_pagerank");
  return api_guard([&] {
    if (!ctx) invalid("null context");
    validate_config(cfg);
    check_pair(gT, gF);
    if (!ranks_out) invalid("null output array");
    bind_device(ctx);
    SolveSpec sp;
    sp.gT = gT;
    sp.gF = gF;
    sp.cfg = cfg;
    solve(ctx, sp, ranks_out, stats, observer, observer_user);
  });
}

// staticPageRank(gT, gF, cfg) on host CSR arrays (the reference's by-value
// call with freshly constructed graphs): gT is uploaded and validated first;
// gF's offsets follow, and its targets -- which Static never reads -- are
// uploaded and validated on the side stream while the solve runs.  Errors
// keep the reference's order: graph construction (gT, then gF), then the
// engine's own checks.
dynpr_status dynpr_static_pagerank_csr(dynpr_context* ctx, uint32_t n, const uint64_t* offT, const uint32_t* tgtT,
                                       const uint64_t* offF, const uint32_t* tgtF, uint64_t m,
                                       const dynpr_config* cfg, double* ranks_out, dynpr_stats* stats,
                                       dynpr_observer observer, void* observer_user) {
  NvtxRange nvtx__("dynpr_static_pagerank_csr");
  dynpr_graph* gT = nullptr;
  const dynpr_status st = dynpr_graph_from_csr(ctx, n, offT, tgtT, m, &gT);
  if (st != DYNPR_OK) return st;
  struct Own {
    dynpr_graph* g;
    ~Own() { dynpr_graph_destroy(g); }
  } own{gT};
  return api_guard([&] {
    bind_device(ctx);
    if (!ctx->ev_side) DYNPR_CK(cudaEventCreateWithFlags(&ctx->ev_side, cudaEventDisableTiming));
    DeferredCsr gF;
    upload_csr_deferred(ctx, n, offF, tgtF, m, ctx->ev_side, gF);
    try {
      validate_config(cfg);
      check_pair(gT, gF.g);
      if (!ranks_out) invalid("null output array");
    } catch (...) {
      gF.finish();  // an invalid gF would have failed at construction, first
      throw;
    }
    // A team fingerprints both CSRs of the pair (team_check_graph) on the
    // main stream: gF's targets must have landed (and be valid) first, so a
    // team joins the side upload before the solve instead of after it.
    if (is_team(ctx)) gF.finish();
    SolveSpec sp;
    sp.gT = gT;
    sp.gF = gF.g;
    sp.cfg = cfg;
    solve(ctx, sp, ranks_out, stats, observer, observer_user);
    gF.finish();
  });
}

dynpr_status dynpr_naive_dynamic(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF,
                                 const double* previous, uint64_t n_previous, const dynpr_config* cfg,
                                 double* ranks_out, dynpr_stats* stats, dynpr_observer observer,
                                 void* observer_user) {
  NvtxRange nvtx__("dynpr_naive_dynamic");
  return api_guard([&] {
    if (!ctx) invalid("null context");
    validate_config(cfg);
    check_pair(gT, gF);
    if (n_previous != gT->n) invalid("naiveDynamic: previousRanks length mismatch");
    if (!ranks_out) invalid("null output array");
    bind_device(ctx);
    SolveSpec sp;
    sp.gT = gT;
    sp.gF = gF;
    sp.cfg = cfg;
    sp.prev = stage_in(ctx, ctx->stage_b, previous, n_previous);
    solve(ctx, sp, ranks_out, stats, observer, observer_user);
  });
}

dynpr_status dynpr_dynamic_frontier(dynpr_context* ctx, const dynpr_graph* gF, const dynpr_graph* gT,
                                    const uint32_t* del_src, const uint32_t* del_dst, uint64_t n_del,
                                    const uint32_t* ins_src, const uint32_t* ins_dst, uint64_t n_ins,
                                    const double* previous, uint64_t n_previous, const dynpr_config* cfg,
                                    int pruning, double* ranks_out, dynpr_stats* stats, dynpr_observer observer,
                                    void* observer_user) {
  NvtxRange nvtx__("dynpr_dynamic_frontier");
  return api_guard([&] {
    if (!ctx) invalid("null context");
    // checkFrontierInputs (engine.cpp:155-162)
    validate_config(cfg);
    check_pair(gT, gF);
    if (n_previous != gT->n) invalid("dynamicFrontier: previousRanks length mismatch");
    if (!ranks_out) invalid("null output array");
    bind_device(ctx);
    SolveSpec sp;
    sp.gT = gT;
    sp.gF = gF;
    sp.cfg = cfg;
    sp.prev = stage_in(ctx, ctx->stage_b, previous, n_previous);
    sp.ds = stage_in(ctx, ctx->batch[0], del_src, n_del);
    sp.dd = stage_in(ctx, ctx->batch[1], del_dst, n_del);
    sp.is = stage_in(ctx, ctx->batch[2], ins_src, n_ins);
    const uint32_t* id = stage_in(ctx, ctx->batch[3], ins_dst, n_ins);
    sp.nd = n_del;
    sp.ni = n_ins;
    // initialAffected range checks (frontier.cpp:36-37)
    if (batch_ids_bad(ctx, del_src, del_dst, sp.ds, sp.dd, n_del, gT->n))
      invalid("initialAffected deletions: vertex id out of range");
    if (batch_ids_bad(ctx, ins_src, ins_dst, sp.is, id, n_ins, gT->n))
      invalid("initialAffected insertions: vertex id out of range");
    sp.flagged = true;
    sp.closed = pruning != 0;
    solve(ctx, sp, ranks_out, stats, observer, observer_user);
  });
}

dynpr_status dynpr_dynamic_traversal(dynpr_context* ctx, const dynpr_graph* gF, const dynpr_graph* gT,
                                     const uint32_t* del_src, const uint32_t* del_dst, uint64_t n_del,
                                     const uint32_t* ins_src, const uint32_t* ins_dst, uint64_t n_ins,
                                     const double* previous, uint64_t n_previous, const dynpr_config* cfg,
                                     double* ranks_out, dynpr_stats* stats, dynpr_observer observer,
                                     void* observer_user) {
  NvtxRange nvtx__("dynpr_dynamic_traversal");
  return api_guard([&] {
    if (!ctx) invalid("null context");
    validate_config(cfg);
    check_pair(gT, gF);
    if (n_previous != gT->n) invalid("dynamicTraversal: previousRanks length mismatch");
    if (!ranks_out) invalid("null output array");
    bind_device(ctx);
    // seeds: sources of all updates + targets of deletions (engine.cpp:138-145)
    const uint64_t ns = 2 * n_del + n_ins;
    uint32_t* seeds = ctx->stage_d.as<uint32_t>(ns + 1);
    auto put = [&](const uint32_t* p, uint64_t cnt, uint64_t at) {
      if (cnt) DYNPR_CK(cudaMemcpyAsync(seeds + at, p, cnt * 4, cudaMemcpyDefault, ctx->stream));
    };
    if (n_del && (!del_src || !del_dst)) invalid("null array argument");
    if (n_ins && !ins_src) invalid("null array argument");
    put(del_src, n_del, 0);
    put(del_dst, n_del, n_del);
    put(ins_src, n_ins, 2 * n_del);
    if (any_bad_ids(ctx, seeds, seeds, ns, gT->n)) invalid("markReachable: seed out of range");
    (void)ins_dst;
    SolveSpec sp;
    sp.gT = gT;
    sp.gF = gF;
    sp.cfg = cfg;
    sp.prev = stage_in(ctx, ctx->stage_b, previous, n_previous);
    sp.flagged = true;
    sp.closed = false;
    sp.traversal = true;
    sp.seeds = seeds;
    sp.nseeds = ns;
    solve(ctx, sp, ranks_out, stats, observer, observer_user);
  });
}

dynpr_status dynpr_mark_reachable(dynpr_context* ctx, const dynpr_graph* g, const uint32_t* seeds, uint64_t n_seeds,
                                  uint8_t* vertex_affected) {
  NvtxRange nvtx__("dynpr_mark_reachable");
  return api_guard([&] {
    if (!ctx || !g) invalid("null argument");
    bind_device(ctx);
    const uint32_t n = g->n;
    const uint32_t* s = stage_in(ctx, ctx->stage_d, seeds, n_seeds);
    if (any_bad_ids(ctx, s, s, n_seeds, n)) invalid("markReachable: seed out of range");
    uint8_t* flags = ctx->flags_va.as<uint8_t>((uint64_t)n + 4);
    DYNPR_CK(cudaMemsetAsync(flags, 0, (size_t)n + 4, ctx->stream));
    mark_reachable(ctx, Rows{g->off, nullptr, g->tgt}, n, g->m, nullptr, s, n_seeds, flags);
    if (n) DYNPR_CK(cudaMemcpyAsync(vertex_affected, flags, n, cudaMemcpyDefault, ctx->stream));
    sync(ctx);
  });
}

dynpr_status dynpr_dynamic_frontier_from_flags(dynpr_context* ctx, const dynpr_graph* gF, const dynpr_graph* gT,
                                               const uint8_t* vertex_affected, const uint8_t* neighbors_pending,
                                               uint64_t n_flags, const double* previous, uint64_t n_previous,
                                               const dynpr_config* cfg, int pruning, double* ranks_out,
                                               dynpr_stats* stats, dynpr_observer observer, void* observer_user) {
  NvtxRange nvtx__("dynpr_dynamic_frontier_from_flags");
  return api_guard([&] {
    if (!ctx) invalid("null context");
    validate_config(cfg);
    check_pair(gT, gF);
    if (n_previous != gT->n) invalid("dynamicFrontier: previousRanks length mismatch");
    if (n_flags != gT->n) invalid("dynamicFrontier: flags length mismatch");
    if (!ranks_out) invalid("null output array");
    (void)neighbors_pending;  // cleared by the first sweep before any expansion (engine.cpp:74-76)
    bind_device(ctx);
    SolveSpec sp;
    sp.gT = gT;
    sp.gF = gF;
    sp.cfg = cfg;
    sp.prev = stage_in(ctx, ctx->stage_b, previous, n_previous);
    sp.flags_in = stage_in(ctx, ctx->stage_a, vertex_affected, n_flags);
    sp.flagged = true;
    sp.closed = pruning != 0;
    solve(ctx, sp, ranks_out, stats, observer, observer_user);
  });
}

}  // extern "C"
