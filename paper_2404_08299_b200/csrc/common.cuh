// Shared host/device plumbing of libdynpr_cuda.so: error model, context,
// grow-only device workspace, host<->device argument staging.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "dynpr_cuda.h"

namespace dynpr_b200 {

// NVTX range for the span of a scope (tracing): every C-ABI entry
// point and the solve / ingest / layout phases inside it, so an nsys or ncu
// NVTX view attributes kernels to the API call that launched them.
// (nvtx3 is header-only: without an attached tool a range costs a branch.)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- error model -----------------------------------------------------------
// Internal code throws; every extern "C" entry point converts to a status and
// stores the message for dynpr_last_error().
struct Error : std::runtime_error {
  dynpr_status code;
  Error(dynpr_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void invalid(const std::string& m) {
  throw Error(DYNPR_INVALID_ARGUMENT, m);
}

void set_last_error(const std::string& m);

#define DYNPR_CK(call)                                                        \
  do {                                                                        \
    cudaError_t e__ = (call);                                                 \
    if (e__ != cudaSuccess) {                                                 \
      throw ::dynpr_b200::Error(                                              \
          e__ == cudaErrorMemoryAllocation ? DYNPR_OUT_OF_MEMORY              \
                                           : DYNPR_CUDA_ERROR,                \
          std::string(#call) + ": " + cudaGetErrorString(e__));               \
    }                                                                         \
  } while (0)

template <class F>
dynpr_status api_guard(F&& f) {
  try {
    f();
    return DYNPR_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return DYNPR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return DYNPR_CUDA_ERROR;
  }
}

// ---- device buffers ----------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void* ensure(size_t bytes) {
    if (bytes <= cap && p) return p;
    if (p) DYNPR_CK(cudaFree(p));
    p = nullptr;
    cap = 0;
    // 25% headroom: snapshots of a batch stream grow by a few edges at a
    // time, and a re-allocation (cudaFree synchronises the device) must not
    // land inside an engine call's timed region on every batch
    size_t want = bytes < 256 ? 256 : bytes + bytes / 4;
    DYNPR_CK(cudaMalloc(&p, want));
    cap = want;
    return p;
  }
  template <class T>
  T* as(size_t count) {
    return static_cast<T*>(ensure(count * sizeof(T)));
  }
};

// Per-solve reduction slot (device), read back once per sweep.
struct SweepRed {
  unsigned long long delta_bits;  // max |r - prev| as IEEE bits (>= 0)
  unsigned long long processed;   // vertices processed (affected count)
  unsigned long long edges;       // in-edges gathered
  unsigned long long pend_edges;  // out-edges of the pending vertices
  unsigned int pend_low;          // pending vertices with out-degree <= T
  unsigned int pend_high;         // 1024-edge expansion items of the others
  unsigned int ticket_heavy;      // fused sweep work queues (dynamic scheduling)
  unsigned int ticket_light;
  unsigned int ticket_pull;       // pull expansion work queue
  unsigned int pad_;
};

// Out-edges per expansion work item of a high out-degree vertex.
constexpr uint32_t kExpandChunk = 1024;

class Comm;
}  // namespace dynpr_b200

struct dynpr_context {
  int device = 0;
  dynpr_b200::Comm* comm = nullptr;  // owned; null = single GPU
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  // profiling of rank sweeps
  bool profiling = false;
  double sweep_ms = 0.0;
  uint64_t sweeps = 0;
  uint64_t sweep_bytes = 0;
  uint64_t pull_expansions = 0;
  // fused multi-GPU exchange: every rank's two contribution buffers, mapped
  // into this process (dynpr_context_attach_peers); empty = all-gather path
  std::vector<double*> peer_cb[2];
  uint64_t peer_capacity = 0;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;
  // pinned host scratch for small readbacks
  void* pinned = nullptr;
  cudaStream_t side = nullptr;  // deferred uploads / validation (created on first use)
  cudaEvent_t ev_side = nullptr;
  cudaEvent_t ev_rec[2] = {nullptr, nullptr};  // speculative team loop: per-record readiness
  // split sweep: the multi-chunk kernel runs on `aux`, concurrently with the
  // single-vertex kernel (fork / join events)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // captures the IF bodies of the device-loop graph (never launched on)
  cudaStream_t capture_aux = nullptr;
  // instantiated device-loop graphs (engine.cu LoopGraphCache), keyed by
  // sweep plan; owned
  void* loop_graphs = nullptr;
  // workspace (grow-only; the engines never allocate inside the timed loop)
  dynpr_b200::DevBuf rank[2], contrib[2], flags_va, flags_np, flags_written,
      pend_low, pend_high, pend_flags, partials, perm_stage,
      tile_counts, red, stage_a, stage_b, stage_c, stage_d, stage_e, stage_f,
      prims_tmp, sort_hist, ingest_state[2], tick, loopctl, layout_tmp, plan_prefix, side_err, bfs_a, bfs_b, run_list, run_pieces, scratch64a, scratch64b, scratch32a, scratch32b, scratch8a, batch[4],
      flag_bits, flag_bounds;  // team pending-flag bitmap exchange
  // lifetime: graphs are allocated from this context's stream-ordered pool.
  // dynpr_context_destroy with graphs still alive (e.g. a garbage-collected
  // binding finalising both in arbitrary order) defers the teardown to the
  // last graph's destroy.
  std::atomic<uint64_t> live_graphs{0};
  std::atomic<bool> closing{false};
  std::atomic<bool> torn_down{false};
};

namespace dynpr_b200 {
struct Layout;
struct LayoutSeed;
}

struct dynpr_graph {
  uint64_t id = 0;          // unique per snapshot (layout cache key)
  std::shared_ptr<dynpr_b200::Layout> layout;  // cached engine layout (transpose side)
  // set by apply_batch_pair on the new transpose: the parent snapshot's
  // layout + the rows the batch touched, from which the new layout is
  // derived incrementally (layout.cu) instead of rebuilt
  std::shared_ptr<dynpr_b200::LayoutSeed> seed;
  dynpr_context* ctx = nullptr;
  uint32_t n = 0;
  uint64_t m = 0;
  uint64_t* off = nullptr;  // n+1, device
  uint32_t* tgt = nullptr;  // m, device
  bool all_loops = false;   // every vertex known to carry its self-loop
};

namespace dynpr_b200 {

constexpr int kWarp = 32;

inline unsigned grid_for(uint64_t items, unsigned per_block,
                         unsigned cap = 1u << 30) {
  uint64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

inline void count_launch(dynpr_context* ctx, uint64_t k = 1) {
  ctx->launches += k;
}
inline void check_launch() { DYNPR_CK(cudaGetLastError()); }

// ---- host/device argument staging ---------------------------------------------
bool is_device_ptr(const void* p);

// Makes `count` elements of a caller array available on the device.
template <class T>
const T* stage_in(dynpr_context* ctx, DevBuf& buf, const T* p, uint64_t count) {
  if (count == 0) return static_cast<const T*>(buf.ensure(sizeof(T)));
  if (p == nullptr) invalid("null array argument");
  if (is_device_ptr(p)) return p;
  T* d = buf.as<T>(count);
  DYNPR_CK(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice,
                           ctx->stream));
  return d;
}

// Output staging: returns a device pointer to write; commit() copies back.
template <class T>
struct StageOut {
  dynpr_context* ctx;
  T* user;
  T* dev;
  uint64_t count;
  bool host;
  StageOut(dynpr_context* c, DevBuf& buf, T* p, uint64_t n)
      : ctx(c), user(p), count(n) {
    if (n && p == nullptr) invalid("null output array");
    host = n && !is_device_ptr(p);
    dev = host ? buf.as<T>(n) : p;
  }
  void commit() {
    if (host && count)
      DYNPR_CK(cudaMemcpyAsync(user, dev, count * sizeof(T),
                               cudaMemcpyDeviceToHost, ctx->stream));
    DYNPR_CK(cudaStreamSynchronize(ctx->stream));
  }
};

inline void sync(dynpr_context* ctx) {
  DYNPR_CK(cudaStreamSynchronize(ctx->stream));
}

inline void bind_device(dynpr_context* ctx) { DYNPR_CK(cudaSetDevice(ctx->device)); }

// Long-lived arrays (graph snapshots, engine layouts) come from the device's
// stream-ordered memory pool (release threshold = unlimited, set at context
// creation), so snapshot churn during batch ingest reuses memory instead of
// paying cudaMalloc/cudaFree.
inline void* pool_alloc(dynpr_context* ctx, size_t bytes) {
  void* p = nullptr;
  // Large arrays are over-allocated by ~3% and rounded to 2 MiB: the next
  // snapshot of a batch stream is a few edges larger, and without slack its
  // arrays could not reuse the blocks the previous snapshot returned to the
  // pool (new physical memory is mapped on such a miss: tens of ms per GB).
  if (bytes >= (size_t(1) << 21)) {
    const size_t slack = bytes + bytes / 32;
    bytes = (slack + (size_t(1) << 21) - 1) & ~((size_t(1) << 21) - 1);
  }
  static const bool dbg = std::getenv("DYNPR_ALLOC_DEBUG") != nullptr;
  const auto t0 = dbg ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
  cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, ctx->stream);
  if (dbg) {
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    if (us > 1000.0) std::fprintf(stderr, "pool_alloc %zu bytes: %.1f us\n", bytes, us);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(DYNPR_OUT_OF_MEMORY, "device allocation of " + std::to_string(bytes) + " bytes failed");
  }
  return p;
}
template <class T>
T* pool_alloc_n(dynpr_context* ctx, uint64_t count) {
  return static_cast<T*>(pool_alloc(ctx, count * sizeof(T)));
}
inline void pool_free(dynpr_context* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

// ---- device helpers ------------------------------------------------------------
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Binary search: first index in [lo, hi) with a[i] >= key.
template <class T, class I>
__device__ __forceinline__ I lower_bound_dev(const T* a, I lo, I hi, T key) {
  while (lo < hi) {
    I mid = lo + (hi - lo) / 2;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// First index in [0, len) with a[i] > x (a ascending).
__device__ __forceinline__ uint64_t upper_bound_u32(const uint32_t* a, uint64_t len, uint32_t x) {
  uint64_t lo = 0, hi = len;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Number of bits needed to represent x (0 -> 0).
inline int bits_for(uint64_t x) {
  int b = 0;
  while (x) { ++b; x >>= 1; }
  return b;
}

// ---- shared internals used across translation units ------------------------
// graph.cu
dynpr_graph* new_graph_struct(dynpr_context* ctx, uint32_t n);
dynpr_graph* make_graph(dynpr_context* ctx, uint32_t n, uint64_t m);
void destroy_graph(dynpr_graph* g);
// releases every resource of a context (engine.cu); called exactly once
void context_teardown(dynpr_context* ctx);

// A host CSR uploaded with its targets' transfer + validation deferred to
// the context's side stream (dynpr_static_pagerank_csr): the graph is usable
// for anything that reads only its offsets until finish() has joined.
struct DeferredCsr {
  dynpr_context* ctx = nullptr;
  dynpr_graph* g = nullptr;
  unsigned* rowstart = nullptr;
  unsigned long long* err = nullptr;
  unsigned long long* host = nullptr;
  bool pending = false;
  void finish();
  ~DeferredCsr();
};
cudaStream_t side_stream(dynpr_context* ctx);
void upload_csr_deferred(dynpr_context* ctx, uint32_t n, const uint64_t* offsets, const uint32_t* targets,
                         uint64_t m, cudaEvent_t after, DeferredCsr& d);
void graph_apply_batch_multi(dynpr_context* ctx, int count, const dynpr_graph* const* gs,
                             const uint32_t* const* ds, const uint32_t* const* dd, uint64_t nd,
                             const uint32_t* const* is, const uint32_t* const* id, uint64_t ni, bool validate,
                             const uint32_t* h_ds, const uint32_t* h_dd, const uint32_t* h_is,
                             const uint32_t* h_id, dynpr_graph** outs, uint64_t* missing_out,
                             uint64_t* duplicate_out, uint32_t** rows_out, uint64_t* nrows_out);
void graph_apply_batch_impl(dynpr_context* ctx, const dynpr_graph* g,
                            const uint32_t* d_ds, const uint32_t* d_dd,
                            uint64_t nd, const uint32_t* d_is,
                            const uint32_t* d_id, uint64_t ni, bool validate,
                            const uint32_t* h_ds, const uint32_t* h_dd,
                            const uint32_t* h_is, const uint32_t* h_id,
                            dynpr_graph** out, uint64_t* missing,
                            uint64_t* duplicate, uint32_t** rows_out = nullptr,
                            uint64_t* nrows_out = nullptr);

}  // namespace dynpr_b200
