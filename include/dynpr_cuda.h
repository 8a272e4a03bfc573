/*
 * dynpr_cuda.h -- C-ABI of the B200-native Static / DF-P PageRank engine.
 *
 * This is the drop-in boundary for the compute path of the reference C++
 * library `dynpr` (/root/reference/proj).  The reference exposes a plain
 * C++20 API in namespace `dynpr` and has no FFI of its own; every entry point
 * below replaces one reference function (cited file:line) and keeps its
 * argument meaning, its validation order and its exception message text
 * (returned through dynpr_last_error()).  A C++ shim that restores the exact
 * `dynpr::` signatures on top of this ABI is include/dynpr_b200.hpp; the
 * Python mirror of the reference's pybind11 module is
 * paper_2404_08299_b200/__init__.py.  INTEGRATION.md shows both bindings.
 *
 * Conventions
 *  - Every function returns a dynpr_status; on failure the thread-local
 *    dynpr_last_error() holds the message (the reference's exception text for
 *    validation errors, e.g. "engine: empty graph").
 *  - Plain pointers + sizes only.  Array arguments may be host memory
 *    (pageable or pinned) or device memory of the context's GPU; the library
 *    detects which with cudaPointerGetAttributes and copies as needed.
 *  - Graph handles are immutable device CSR arrays ("snapshots"), exactly like
 *    the reference's value-typed CsrGraph (graph.hpp:17-49).  Operations that
 *    produce a new snapshot (add_self_loops, transpose, apply_batch) return a
 *    new handle and never mutate their input.
 *  - All calls are synchronous on return.  One context per host thread at a
 *    time (reference SPEC: each engine call is single-caller).
 *  - Types follow graph.hpp:9,47-48: vertex ids uint32, CSR offsets uint64,
 *    ranks fp64, affected flags uint8 (frontier.hpp:16-17).
 */
#ifndef DYNPR_CUDA_H
#define DYNPR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dynpr_status {
  DYNPR_OK = 0,
  DYNPR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  DYNPR_CUDA_ERROR = 2,
  DYNPR_NCCL_ERROR = 3,
  DYNPR_OUT_OF_MEMORY = 4,
  DYNPR_SIZING_ERROR = 5,     /* dynpr::SizingError (workload.hpp:17-19) */
  DYNPR_PARSE_ERROR = 6,      /* dynpr::ParseError (workload.hpp:12-15) */
  DYNPR_RUNTIME_ERROR = 7     /* std::runtime_error (e.g. "cannot open <path>") */
} dynpr_status;

/* rank.hpp:14-18 PartitionStrategy */
enum {
  DYNPR_DONT_PARTITION = 0,
  DYNPR_PARTITION_TRANSPOSE = 1,
  DYNPR_PARTITION_BOTH = 2
};

/* rank.hpp:23 RankMode */
enum { DYNPR_RANK_PLAIN = 0, DYNPR_RANK_CLOSED_LOOP_PRUNE = 1 };

/* rank.hpp:25-39 EngineConfig, field for field. */
typedef struct dynpr_config {
  double damping_factor;         /* alpha, default 0.85 */
  double iteration_tolerance;    /* L-inf convergence threshold, 1e-10 */
  double frontier_tolerance;     /* tau_f, 1e-6 */
  double prune_tolerance;        /* tau_p, 1e-6 */
  int32_t max_iterations;        /* 500 */
  uint32_t low_degree_threshold; /* D_P, 32 */
  int32_t partition_strategy;    /* DYNPR_PARTITION_BOTH */
  int32_t convergence_check_disabled; /* 0 */
} dynpr_config;

/* engine.hpp:16-22 RankResult telemetry (ranks are returned separately). */
typedef struct dynpr_stats {
  int32_t iterations;
  int32_t converged;
  uint64_t affected_vertex_iterations;
  double final_delta;
  uint64_t processed_edges; /* sum of in-degree over processed vertices */
  double device_ms;         /* CUDA-event time of the engine call */
} dynpr_stats;

/*
 * Per-iteration observer (engine.hpp:24-27 IterationObserver).  `ranks` is a
 * host copy of the latest iterate; `processed` is a host copy of the
 * vertexAffected flags at the start of that sweep (the processed set), or
 * NULL for the full-sweep engines.  Only honoured when non-NULL: it forces a
 * device-to-host copy per iteration.
 */
typedef void (*dynpr_observer)(int iteration, const double* ranks,
                               const uint8_t* processed, uint64_t n,
                               void* user);

typedef struct dynpr_context dynpr_context;
typedef struct dynpr_graph dynpr_graph;

/* ---- errors, config ----------------------------------------------------- */
const char* dynpr_last_error(void);
const char* dynpr_version(void);
void dynpr_config_default(dynpr_config* cfg);
/* EngineConfig::validate (rank.cpp:11-20), same messages. */
dynpr_status dynpr_config_validate(const dynpr_config* cfg);

/* ---- context ------------------------------------------------------------ */
dynpr_status dynpr_context_create(int device, dynpr_context** out);
/* Graphs live in their context's device memory pool: destroying a context
 * whose graphs are still alive defers the teardown until the last of them
 * is destroyed (any order of the two calls is safe; using a graph after its
 * context's destroy is not supported). */
dynpr_status dynpr_context_destroy(dynpr_context* ctx);
/* Kernel-launch counter (every kernel this library launched). */
uint64_t dynpr_context_launches(const dynpr_context* ctx);
/*
 * Profiling: when enabled the engines bracket every rank-update sweep with
 * CUDA events on their stream; dynpr_context_sweep_times returns the summed
 * sweep time (ms) and the number of sweeps since the last reset.
 */
dynpr_status dynpr_context_set_profiling(dynpr_context* ctx, int enable);
dynpr_status dynpr_context_sweep_times(dynpr_context* ctx, double* total_ms,
                                       uint64_t* sweeps, uint64_t* bytes);

/* ---- multi-GPU (the reference is single-node CPU only) -------- */
/* One process per GPU: rank 0 obtains a 128-byte NCCL unique id, shares it
 * (e.g. torch.distributed broadcast), every rank creates its context.  The
 * engines are then called SPMD with identical (replicated) graphs and
 * inputs: each rank sweeps its edge-balanced vertex range, contributions and
 * pending flags are all-gathered over NVLink after every sweep, and every
 * rank returns the full result.  NCCL is loaded at run time (dlopen). */
dynpr_status dynpr_nccl_get_unique_id(uint8_t* id128);
dynpr_status dynpr_context_create_nccl(int device, int rank, int world,
                                       const uint8_t* id128,
                                       dynpr_context** out);
/* The same partitioned engine with `world` virtual ranks on host threads of
 * one process (any devices, typically one): the test harness of the
 * multi-GPU path on a single GPU. */
typedef struct dynpr_team dynpr_team;
dynpr_status dynpr_team_create(int world, dynpr_team** out);
dynpr_status dynpr_team_destroy(dynpr_team* team);
dynpr_status dynpr_context_create_team(int device, dynpr_team* team, int rank,
                                       dynpr_context** out);
dynpr_status dynpr_context_rank(const dynpr_context* ctx, int* rank,
                                int* world);
/* The same partitioned engine over a caller-supplied host transport (any
 * process-group library: torch.distributed gloo, MPI, ...).  The engine
 * stages every collective through pinned host memory and calls these on the
 * solving thread, identically ordered on every rank; a nonzero return fails
 * the solve with DYNPR_RUNTIME_ERROR.  Ranks may share a GPU (NCCL refuses
 * that), which is how the cross-process path is tested on one GPU. */
typedef struct dynpr_comm_ops {
  /* in place on host data[count]: element-wise over the ranks, op 0 = sum
   * (mod 2^64), op 1 = max (unsigned) */
  int (*allreduce_u64)(uint64_t* data, uint64_t count, int op, void* user);
  /* in place on host buf: rank r contributes bytes [offsets[r],
   * offsets[r+1]) and receives all offsets[world] bytes */
  int (*allgatherv)(void* buf, const uint64_t* offsets, int world,
                    void* user);
  int (*barrier)(void* user);
} dynpr_comm_ops;
dynpr_status dynpr_context_create_hostcomm(int device, int rank, int world,
                                           const dynpr_comm_ops* ops,
                                           void* user, dynpr_context** out);
/* Device buffers shareable across processes (CUDA IPC) for the fused
 * exchange: dynpr_ipc_alloc returns a device buffer and its 64-byte handle;
 * another process maps it with dynpr_ipc_open (same or peer GPU) and unmaps
 * with dynpr_ipc_close; the owner releases it with dynpr_ipc_free. */
dynpr_status dynpr_ipc_alloc(dynpr_context* ctx, uint64_t bytes, void** dptr,
                             uint8_t* handle64);
dynpr_status dynpr_ipc_open(dynpr_context* ctx, const uint8_t* handle64,
                            void** dptr);
dynpr_status dynpr_ipc_close(dynpr_context* ctx, void* dptr);
dynpr_status dynpr_ipc_free(dynpr_context* ctx, void* dptr);
/* Fused exchange: ptrs0[r] / ptrs1[r] are rank r's two contribution buffers
 * (`capacity` doubles each) mapped into this process -- CUDA IPC / torch
 * symmetric memory across processes, plain device pointers for a LocalTeam.
 * With them attached, every sweep's epilogue stores each new contribution
 * straight into all ranks' copies over NVLink (the transfer overlaps the
 * sweep), replacing the per-sweep all-gather; the sweep-record all-reduce
 * remains as the team barrier.  world = 0 detaches. */
dynpr_status dynpr_context_attach_peers(dynpr_context* ctx, int world,
                                        const uint64_t* ptrs0,
                                        const uint64_t* ptrs1,
                                        uint64_t capacity);

/* ---- graphs (graph.hpp:17-80) ------------------------------------------- */
/* CsrGraph(vertexCount, offsets, targets) incl. validation (graph.cpp:30-49).
 * offsets has n+1 entries, targets offsets[n] entries. */
dynpr_status dynpr_graph_from_csr(dynpr_context* ctx, uint32_t n,
                                  const uint64_t* offsets,
                                  const uint32_t* targets, uint64_t m,
                                  dynpr_graph** out);
/* buildCsr (graph.cpp:56-68): sort + dedupe, throws on ids >= n. */
dynpr_status dynpr_graph_build(dynpr_context* ctx, uint32_t n,
                               const uint32_t* src, const uint32_t* dst,
                               uint64_t count, dynpr_graph** out);
/* addSelfLoops (graph.cpp:85-111). */
dynpr_status dynpr_graph_add_self_loops(dynpr_context* ctx,
                                        const dynpr_graph* g,
                                        dynpr_graph** out);
/* transpose (graph.cpp:70-83): slices in ascending source order. */
dynpr_status dynpr_graph_transpose(dynpr_context* ctx, const dynpr_graph* g,
                                   dynpr_graph** out);
/* applyBatch (graph.cpp:113-203): (E \ dels) U ins, loops re-ensured.
 * missing / duplicate may be NULL; otherwise they are ADDED to (like
 * BatchApplyStats accumulation, graph.cpp:198-201). */
dynpr_status dynpr_graph_apply_batch(dynpr_context* ctx, const dynpr_graph* g,
                                     const uint32_t* del_src,
                                     const uint32_t* del_dst, uint64_t n_del,
                                     const uint32_t* ins_src,
                                     const uint32_t* ins_dst, uint64_t n_ins,
                                     dynpr_graph** out, uint64_t* missing,
                                     uint64_t* duplicate);
/* Batch ingest for a (forward, transpose) pair: applies the batch to gF and
 * the reversed batch to gT, so out_gT == transpose(out_gF) byte for byte
 * without a full re-transpose (replaces harness.cpp:203-204). */
dynpr_status dynpr_graph_apply_batch_pair(
    dynpr_context* ctx, const dynpr_graph* gF, const dynpr_graph* gT,
    const uint32_t* del_src, const uint32_t* del_dst, uint64_t n_del,
    const uint32_t* ins_src, const uint32_t* ins_dst, uint64_t n_ins,
    dynpr_graph** out_gF, dynpr_graph** out_gT, uint64_t* missing,
    uint64_t* duplicate);
dynpr_status dynpr_graph_info(const dynpr_graph* g, uint32_t* n, uint64_t* m);
/* Copies offsets (n+1) and targets (m) out (host or device pointers). */
dynpr_status dynpr_graph_download(dynpr_context* ctx, const dynpr_graph* g,
                                  uint64_t* offsets, uint32_t* targets);
dynpr_status dynpr_graph_has_edge(dynpr_context* ctx, const dynpr_graph* g,
                                  uint32_t source, uint32_t target, int* out);
dynpr_status dynpr_graph_destroy(dynpr_graph* g);
/* Synthetic RMAT/Kronecker generator (no reference counterpart):
 * edge i draws `scale` quadrant choices from SplitMix64(deriveSeed(seed,i))
 * (rng.hpp:10-47) with probabilities (a, b, c, 1-a-b-c); count =
 * edge_factor << scale pairs, then buildCsr + addSelfLoops. */
dynpr_status dynpr_graph_rmat(dynpr_context* ctx, uint32_t scale,
                              uint32_t edge_factor, double a, double b,
                              double c, uint64_t seed, dynpr_graph** out);
/* Kronecker graph in the Graph500 style: the RMAT draws above with the
 * Graph500 initiator (a, b, c) = (0.57, 0.19, 0.19), then every vertex id
 * mapped through a seeded bijection of [0, 2^scale) (odd multiplications,
 * an added constant and xor-shifts modulo 2^scale) so the hubs are spread
 * over the id space; buildCsr + addSelfLoops. */
dynpr_status dynpr_graph_kronecker(dynpr_context* ctx, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                                   dynpr_graph** out);

/* Builds (or reuses) the engine layout of the pair (gT, gF) for degree
 * threshold `threshold`: vertices relabelled by in-degree, SELL-32 segment
 * slices of the in-CSR, and with `with_forward` the relabelled out-CSR for
 * frontier expansion.  It is cached on gT (snapshots are immutable), so the
 * engines reuse it; an engine call on a pair without it builds it inside the
 * call.  `build_ms` (nullable) receives the device time of the build. */
dynpr_status dynpr_graph_prepare(dynpr_context* ctx, const dynpr_graph* gT,
                                 const dynpr_graph* gF, uint32_t threshold,
                                 int with_forward, double* build_ms);
/* The cached engine layout of gT (after dynpr_graph_prepare or a solve):
 * SELL words held by this context (a team rank holds only its own rows:
 * about 1/world of the single-GPU figure), the owned vertex range
 * [v_lo, v_hi) in the layout's relabelled order (everything on one GPU),
 * whether the relabelled forward CSR is built, and its generation: 0 for a
 * layout built from scratch, k for one derived incrementally k batches after
 * (dynpr_graph_apply_batch_pair of a prepared pair seeds the derivation).
 * DYNPR_INVALID_ARGUMENT if gT has no layout yet.  Outputs may be null. */
dynpr_status dynpr_graph_layout_info(const dynpr_graph* gT,
                                     uint64_t* sell_words, uint32_t* v_lo,
                                     uint32_t* v_hi, int* has_forward,
                                     int* generation);

/* ---- workload (workload.hpp:189-197, rng.hpp:44-47) --------------------- */
/* batchSizeFromFraction (workload.cpp:245-249): round half up, floor 1. */
uint64_t dynpr_batch_size_from_fraction(double fraction, uint64_t total);
/* deriveSeed (rng.hpp:44-47). */
uint64_t dynpr_derive_seed(uint64_t seed, uint64_t stream);
/* generateRandomBatch (workload.cpp:183-243), same draws and order: the
 * insertions (ceil(insert_fraction * total) uniform non-existing,
 * non-self, distinct pairs) then the deletions (uniform without
 * replacement from the non-loop edges, partial Fisher-Yates).  Host-side
 * (the RNG stream is sequential); outputs are host arrays of capacity
 * total_size.  Errors: SizingError / invalid_argument texts of the
 * reference. */
dynpr_status dynpr_generate_random_batch(dynpr_context* ctx,
                                         const dynpr_graph* g,
                                         uint64_t total_size,
                                         double insert_fraction, uint64_t seed,
                                         uint32_t* ins_src, uint32_t* ins_dst,
                                         uint64_t* n_ins, uint32_t* del_src,
                                         uint32_t* del_dst, uint64_t* n_del);

/* ---- primitives (partition.hpp:20, rank.hpp:66-76, frontier.hpp:28-36) -- */
/* partitionByDegree: order[n] (low group then high group, ascending ids). */
dynpr_status dynpr_partition_by_degree(dynpr_context* ctx,
                                       const dynpr_graph* g,
                                       uint32_t threshold, uint32_t* order,
                                       uint32_t* low_count);
/* updateRanks (rank.cpp:79-140).  vertex_affected / neighbors_pending are
 * either both NULL (full sweep, no flags) or both n-byte arrays that are
 * read and updated in place.  previous is read, current written. */
dynpr_status dynpr_update_ranks(dynpr_context* ctx, const dynpr_graph* gT,
                                const dynpr_graph* gF,
                                uint8_t* vertex_affected,
                                uint8_t* neighbors_pending,
                                const double* previous, double* current,
                                const dynpr_config* cfg, int mode);
/* linfNormDelta / l1NormDelta (rank.cpp:142-152). */
dynpr_status dynpr_linf_norm_delta(dynpr_context* ctx, const double* a,
                                   const double* b, uint64_t n, double* out);
dynpr_status dynpr_l1_norm_delta(dynpr_context* ctx, const double* a,
                                 const double* b, uint64_t n, double* out);
/* initialAffected (frontier.cpp:33-53): writes both n-byte flag arrays. */
dynpr_status dynpr_initial_affected(dynpr_context* ctx, const dynpr_graph* g,
                                    const uint32_t* del_src,
                                    const uint32_t* del_dst, uint64_t n_del,
                                    const uint32_t* ins_src,
                                    const uint32_t* ins_dst, uint64_t n_ins,
                                    uint8_t* vertex_affected,
                                    uint8_t* neighbors_pending);
/* expandAffected (frontier.cpp:55-84): vertex_affected |= out(pending). */
dynpr_status dynpr_expand_affected(dynpr_context* ctx, const dynpr_graph* g,
                                   uint8_t* vertex_affected,
                                   const uint8_t* neighbors_pending,
                                   uint32_t threshold);

/* ---- engines (engine.hpp:33-71) ---------------------------------------- */
/* staticPageRank(gTranspose, gForward, cfg) -- engine.cpp:99-108. */
dynpr_status dynpr_static_pagerank(dynpr_context* ctx, const dynpr_graph* gT,
                                   const dynpr_graph* gF,
                                   const dynpr_config* cfg, double* ranks_out,
                                   dynpr_stats* stats, dynpr_observer observer,
                                   void* observer_user);
/* staticPageRank on host (or device) CSR arrays -- the reference's call with
 * freshly constructed CsrGraph values (graph.cpp:30-49 + engine.cpp:99-108):
 * gT is uploaded and validated, then gF's offsets; gF's targets, which Static
 * does not read, are uploaded and validated on a side stream while the solve
 * runs.  Same errors as constructing the two graphs then calling
 * dynpr_static_pagerank. */
dynpr_status dynpr_static_pagerank_csr(dynpr_context* ctx, uint32_t n,
                                       const uint64_t* offsets_t,
                                       const uint32_t* targets_t,
                                       const uint64_t* offsets_f,
                                       const uint32_t* targets_f, uint64_t m,
                                       const dynpr_config* cfg,
                                       double* ranks_out, dynpr_stats* stats,
                                       dynpr_observer observer,
                                       void* observer_user);
/* naiveDynamic(gTranspose, gForward, previousRanks, cfg) -- engine.cpp:110. */
dynpr_status dynpr_naive_dynamic(dynpr_context* ctx, const dynpr_graph* gT,
                                 const dynpr_graph* gF, const double* previous,
                                 uint64_t n_previous, const dynpr_config* cfg,
                                 double* ranks_out, dynpr_stats* stats,
                                 dynpr_observer observer, void* observer_user);
/* dynamicFrontier(gForward, gTranspose, dels, ins, prev, cfg, pruning) --
 * engine.cpp:192-203.  DF-P when pruning != 0. */
dynpr_status dynpr_dynamic_frontier(
    dynpr_context* ctx, const dynpr_graph* gF, const dynpr_graph* gT,
    const uint32_t* del_src, const uint32_t* del_dst, uint64_t n_del,
    const uint32_t* ins_src, const uint32_t* ins_dst, uint64_t n_ins,
    const double* previous, uint64_t n_previous, const dynpr_config* cfg,
    int pruning, double* ranks_out, dynpr_stats* stats,
    dynpr_observer observer, void* observer_user);
/* dynamicTraversal(gForward, gTranspose, dels, ins, prev, cfg) --
 * engine.cpp:124-151: the affected set is everything reachable (device BFS,
 * markReachable frontier.cpp:86-121) from the update sources and the
 * deletion targets, fixed for the solve; plain rank formula, no expansion. */
dynpr_status dynpr_dynamic_traversal(
    dynpr_context* ctx, const dynpr_graph* gF, const dynpr_graph* gT,
    const uint32_t* del_src, const uint32_t* del_dst, uint64_t n_del,
    const uint32_t* ins_src, const uint32_t* ins_dst, uint64_t n_ins,
    const double* previous, uint64_t n_previous, const dynpr_config* cfg,
    double* ranks_out, dynpr_stats* stats, dynpr_observer observer,
    void* observer_user);
/* markReachable(g, seeds) -- frontier.cpp:86-121: vertex_affected[v] = 1 for
 * every v reachable from a seed (n bytes out; neighborsPending stays 0). */
dynpr_status dynpr_mark_reachable(dynpr_context* ctx, const dynpr_graph* g,
                                  const uint32_t* seeds, uint64_t n_seeds,
                                  uint8_t* vertex_affected);
/* dynamicFrontierFromFlags -- engine.cpp:178-190. */
dynpr_status dynpr_dynamic_frontier_from_flags(
    dynpr_context* ctx, const dynpr_graph* gF, const dynpr_graph* gT,
    const uint8_t* vertex_affected, const uint8_t* neighbors_pending,
    uint64_t n_flags, const double* previous, uint64_t n_previous,
    const dynpr_config* cfg, int pruning, double* ranks_out,
    dynpr_stats* stats, dynpr_observer observer, void* observer_user);

/* ---- input formats (workload.hpp:22-64, workload.cpp:43-181) ------------ */
/* A host edge list: MatrixMarket pairs, or a compacted, timestamp-sorted
 * temporal stream (TemporalEdgeList).  Parsed from a memory map of the file;
 * the messages of ParseError ("<path>:<line>: <what>") and of the
 * "cannot open <path>" runtime_error are the reference's. */
typedef struct dynpr_edge_list dynpr_edge_list;
/* loadMatrixMarket (workload.cpp:43-107): general or symmetric coordinate
 * files, 1-based ids, symmetric off-diagonal entries expanded to both
 * directions, weights ignored; vertex_count = max(rows, cols). */
dynpr_status dynpr_load_matrix_market(const char* path, dynpr_edge_list** out);
/* loadTemporalEdgeList (workload.cpp:109-136): `src dst timestamp` lines,
 * `#` comments, ids compacted to first-appearance order, entries stably
 * sorted by timestamp, duplicates kept. */
dynpr_status dynpr_load_temporal_edge_list(const char* path,
                                           dynpr_edge_list** out);
/* splitTemporal (workload.cpp:138-181): `base` = the first
 * floor(base_fraction * count) entries, sorted and deduplicated; batch b is
 * entries [base_count + b*batch_size, base_count + (b+1)*batch_size) of the
 * stream, as insertions.  SizingError text of the reference when short. */
dynpr_status dynpr_split_temporal(const dynpr_edge_list* stream,
                                  double base_fraction, int32_t batch_count,
                                  uint64_t batch_size, dynpr_edge_list** base,
                                  uint64_t* base_count);
dynpr_status dynpr_edge_list_info(const dynpr_edge_list* e,
                                  uint32_t* vertex_count, uint64_t* count,
                                  int* has_timestamps);
/* Copies entries [first, first+count) out; ts may be NULL. */
dynpr_status dynpr_edge_list_copy(const dynpr_edge_list* e, uint64_t first,
                                  uint64_t count, uint32_t* src, uint32_t* dst,
                                  int64_t* ts);
dynpr_status dynpr_edge_list_destroy(dynpr_edge_list* e);
/* A caller-built edge list (e.g. the reference's TemporalEdgeList entries,
 * workload.hpp:26-36): `count` pairs, timestamps optional (ts NULL = not a
 * temporal stream).  Ids are not checked (the reference's lists are plain
 * values). */
dynpr_status dynpr_edge_list_create(uint32_t vertex_count, const uint32_t* src,
                                    const uint32_t* dst, const int64_t* ts,
                                    uint64_t count, dynpr_edge_list** out);

/* ---- experiment harness (harness.hpp:12-79, harness.cpp:68-399) --------- */
/* computeReferenceRanks (harness.cpp:340-349): Static with the convergence
 * check disabled, exactly cfg->max_iterations sweeps, on the device. */
dynpr_status dynpr_compute_reference_ranks(dynpr_context* ctx,
                                           const dynpr_graph* gT,
                                           const dynpr_graph* gF,
                                           const dynpr_config* cfg,
                                           double* ranks_out);

/* harness.hpp:12 Approach, harness.hpp:16 ExperimentMode, harness.hpp:20-23
 * ChainMode, harness.hpp:55 ReportFormat. */
enum {
  DYNPR_APPROACH_STATIC = 0,
  DYNPR_APPROACH_ND = 1,
  DYNPR_APPROACH_DT = 2,
  DYNPR_APPROACH_DF = 3,
  DYNPR_APPROACH_DFP = 4
};
enum { DYNPR_MODE_STATIC = 0, DYNPR_MODE_TEMPORAL = 1, DYNPR_MODE_RANDOM = 2 };
enum { DYNPR_CHAIN_PER_APPROACH = 0, DYNPR_CHAIN_SHARED_REFERENCE = 1 };
enum { DYNPR_REPORT_CSV = 0, DYNPR_REPORT_JSON = 1 };

/* ExperimentSpec (harness.hpp:41-53), field for field. */
typedef struct dynpr_experiment_spec {
  const char* graph_path;
  const char* graph_name;            /* NULL or "" = file stem */
  int32_t mode;                      /* DYNPR_MODE_* */
  const char* const* batch_size_specs; /* fraction strings, e.g. "1e-3" */
  int32_t n_batch_size_specs;
  const int32_t* approaches;         /* DYNPR_APPROACH_* */
  int32_t n_approaches;
  uint64_t seed;                     /* 1 */
  int32_t repetitions;               /* 1 */
  double base_fraction;              /* 0.9 (temporal) */
  int32_t batch_count;               /* 100 (temporal) */
  double insert_fraction;            /* 0.8 */
  int32_t chain_mode;                /* DYNPR_CHAIN_PER_APPROACH */
  int32_t threads;                   /* accepted, ignored: one GPU context */
  int32_t record_timing;             /* 1; 0 writes deterministic zeros */
  dynpr_config config;
} dynpr_experiment_spec;
void dynpr_experiment_spec_default(dynpr_experiment_spec* spec);

/* ExperimentRow (harness.hpp:29-39).  The strings belong to the report. */
typedef struct dynpr_experiment_row {
  const char* graph_name;
  const char* approach; /* "static" | "nd" | "dt" | "df" | "dfp" */
  const char* batch_size_spec;
  int64_t batch_index;  /* -1 = summary row */
  double runtime_millis;
  int64_t iterations;
  uint64_t affected_vertex_iterations;
  double l1_error_vs_reference; /* NaN when absent */
  int32_t converged;
} dynpr_experiment_row;

typedef struct dynpr_report dynpr_report;
/* runExperiment (harness.cpp:351-381): per-batch rows then one summary row
 * per (approach, batch size).  Graphs are built, batches ingested and the
 * 500-sweep reference ranks computed on the device; runtime_millis is the
 * host wall clock of the engine call alone (harness.cpp:133-135). */
dynpr_status dynpr_run_experiment(dynpr_context* ctx,
                                  const dynpr_experiment_spec* spec,
                                  dynpr_report** out);
dynpr_status dynpr_report_create(dynpr_report** out);
dynpr_status dynpr_report_append(dynpr_report* r, const dynpr_experiment_row* row);
dynpr_status dynpr_report_size(const dynpr_report* r, uint64_t* rows);
dynpr_status dynpr_report_row(const dynpr_report* r, uint64_t i,
                              dynpr_experiment_row* out);
/* summarizeRows (harness.cpp:68-113): geometric means of runtime and error,
 * rounded arithmetic means of the counters, AND of converged. */
dynpr_status dynpr_report_summarize(const dynpr_report* r, dynpr_report** out);
/* emitReport (harness.cpp:287-396): CSV (fixed header) or JSON array, %.17g
 * floats, NaN -> empty field / null; path "-" = stdout. */
dynpr_status dynpr_report_emit(const dynpr_report* r, int32_t format,
                               const char* path);
dynpr_status dynpr_report_destroy(dynpr_report* r);

/* ---- debug ---------------------------------------------------------------- */
/* With DYNPR_TRACE set in the environment the fused sweep records, per warp,
 * {smid, start ns, end ns, heavy items | light items << 32, first heavy item,
 * end of heavy phase ns} of the latest sweep; copies up to `cap` words. */
dynpr_status dynpr_debug_sweep_trace(uint64_t* out, uint64_t cap, uint64_t* count);
/* Per-iteration trace of the last device-loop solve: 4 words per iteration
 * {globaltimer ns at the end of the sweep, gathered edges, processed
 * vertices, pending out-edges | expansion direction << 62 (1 push, 2 pull)}.
 * Diagnostics only (profiles/dfp_iter_probe.py). */
dynpr_status dynpr_debug_loop_trace(uint64_t* out, uint64_t cap, uint64_t* count);
/* Unit-test entry for the hand-written device primitives (csrc/prims.cuh)
 * on host arrays: op 0 radix sort of u64 keys (bits = key width), 1 radix
 * sort of (u32 key, u32 value) pairs, 2 exclusive scan of u64 (total in
 * *out_count), 3 indices of the nonzero bytes, 4 unique of sorted u64
 * (count in *out_count). */
dynpr_status dynpr_debug_prims(dynpr_context* ctx, int op, const void* in, const void* in2, uint64_t count,
                               int bits, void* out, void* out2, uint64_t* out_count);

#ifdef __cplusplus
}
#endif

#endif /* DYNPR_CUDA_H */
