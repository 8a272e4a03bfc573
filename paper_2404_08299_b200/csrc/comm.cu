// NcclComm (NCCL over NVLink, resolved with dlopen) and LocalComm (virtual
// ranks on host threads) -- see comm.cuh.
#include <dlfcn.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "comm.cuh"

namespace dynpr_b200 {

namespace {

// ---- minimal NCCL ABI (nccl.h, stable since 2.x) ----------------------------
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
  char internal[128];
};
typedef int ncclResult_t;  // 0 = ncclSuccess
enum { kNcclUint8 = 1, kNcclUint32 = 3, kNcclUint64 = 5 };
enum { kNcclSum = 0, kNcclMax = 2 };

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // an NCCL already loaded in the process (e.g. torch's) wins
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!a.lib) a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) return a;
    auto sym = [&](const char* s) { return dlsym(a.lib, s); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!api.lib || !api.CommInitRank || !api.Broadcast || !api.AllReduce)
    throw Error(DYNPR_NCCL_ERROR, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0)
    throw Error(DYNPR_NCCL_ERROR, std::string(what) + ": " +
                                      (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error"));
}

class NcclComm final : public Comm {
 public:
  NcclComm(int r, int w, const void* id128) {
    rank = r;
    world = w;
    ncclUniqueId id;
    std::memcpy(id.internal, id128, 128);
    nccl_check(nccl().CommInitRank(&comm_, w, id, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void allgatherv(void* buf, const uint64_t* off, cudaStream_t st) override {
    auto* b = static_cast<uint8_t*>(buf);
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int r = 0; r < world; ++r) {
      const uint64_t bytes = off[r + 1] - off[r];
      if (!bytes) continue;
      nccl_check(nccl().Broadcast(b + off[r], b + off[r], bytes, kNcclUint8, r, comm_, st), "ncclBroadcast");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }
  void allreduce_red(SweepRed* red, cudaStream_t st) override {
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    nccl_check(nccl().AllReduce(&red->delta_bits, &red->delta_bits, 1, kNcclUint64, kNcclMax, comm_, st),
               "ncclAllReduce");
    nccl_check(nccl().AllReduce(&red->processed, &red->processed, 3, kNcclUint64, kNcclSum, comm_, st),
               "ncclAllReduce");
    nccl_check(nccl().AllReduce(&red->pend_low, &red->pend_low, 2, kNcclUint32, kNcclSum, comm_, st),
               "ncclAllReduce");
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }
  void barrier() override {}

 private:
  ncclComm_t comm_ = nullptr;
};

}  // namespace

// ---- LocalComm ---------------------------------------------------------------
struct LocalTeam {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  void* staging = nullptr;
  size_t staging_bytes = 0;
  bool aborted = false;
  std::vector<SweepRed> reds;
  explicit LocalTeam(int w) : world(w), reds(w) {}
  ~LocalTeam() {
    if (staging) cudaFree(staging);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) throw Error(DYNPR_RUNTIME_ERROR, "team: another rank failed");
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen || aborted; });
      if (generation == gen) throw Error(DYNPR_RUNTIME_ERROR, "team: another rank failed");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

namespace {

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalTeam> t, int r, int device) : team_(std::move(t)), device_(device) {
    rank = r;
    world = team_->world;
  }
  void allgatherv(void* buf, const uint64_t* off, cudaStream_t st) override {
    const uint64_t total = off[world];
    if (rank == 0) {
      std::lock_guard<std::mutex> lk(team_->m);
      if (team_->staging_bytes < total) {
        if (team_->staging) cudaFree(team_->staging);
        team_->staging = nullptr;
        team_->staging_bytes = 0;
        DYNPR_CK(cudaMalloc(&team_->staging, total));
        team_->staging_bytes = total;
      }
    }
    team_->barrier();
    auto* s = static_cast<uint8_t*>(team_->staging);
    auto* b = static_cast<uint8_t*>(buf);
    const uint64_t mine = off[rank + 1] - off[rank];
    if (mine) DYNPR_CK(cudaMemcpyAsync(s + off[rank], b + off[rank], mine, cudaMemcpyDefault, st));
    DYNPR_CK(cudaStreamSynchronize(st));
    team_->barrier();
    if (total) DYNPR_CK(cudaMemcpyAsync(b, s, total, cudaMemcpyDefault, st));
    DYNPR_CK(cudaStreamSynchronize(st));
    team_->barrier();
  }
  void allreduce_red(SweepRed* red, cudaStream_t st) override {
    SweepRed h;
    DYNPR_CK(cudaMemcpyAsync(&h, red, sizeof h, cudaMemcpyDeviceToHost, st));
    DYNPR_CK(cudaStreamSynchronize(st));
    team_->reds[rank] = h;
    team_->barrier();
    SweepRed t{};
    for (const SweepRed& x : team_->reds) {
      t.delta_bits = x.delta_bits > t.delta_bits ? x.delta_bits : t.delta_bits;
      t.processed += x.processed;
      t.edges += x.edges;
      t.pend_edges += x.pend_edges;
      t.pend_low += x.pend_low;
      t.pend_high += x.pend_high;
    }
    team_->barrier();
    DYNPR_CK(cudaMemcpyAsync(red, &t, sizeof t, cudaMemcpyHostToDevice, st));
    DYNPR_CK(cudaStreamSynchronize(st));
  }
  void barrier() override { team_->barrier(); }
  void abort() override { team_->abort(); }

 private:
  std::shared_ptr<LocalTeam> team_;
  int device_;
};

// ---- HostComm: caller-supplied host transport -------------------------------
class HostComm final : public Comm {
 public:
  HostComm(int r, int w, const dynpr_comm_ops& ops, void* user) : ops_(ops), user_(user) {
    rank = r;
    world = w;
    DYNPR_CK(cudaMallocHost(&small_, 4096));
  }
  ~HostComm() override {
    if (host_) cudaFreeHost(host_);
    if (small_) cudaFreeHost(small_);
  }
  void allgatherv(void* buf, const uint64_t* off, cudaStream_t st) override {
    const uint64_t total = off[world];
    if (total > host_bytes_) {
      if (host_) DYNPR_CK(cudaFreeHost(host_));
      host_ = nullptr;
      host_bytes_ = 0;
      DYNPR_CK(cudaMallocHost(&host_, total));
      host_bytes_ = total;
    }
    auto* h = static_cast<uint8_t*>(host_);
    auto* b = static_cast<uint8_t*>(buf);
    const uint64_t lo = off[rank], hi = off[rank + 1];
    if (hi > lo) DYNPR_CK(cudaMemcpyAsync(h + lo, b + lo, hi - lo, cudaMemcpyDeviceToHost, st));
    DYNPR_CK(cudaStreamSynchronize(st));
    call(ops_.allgatherv(host_, off, world, user_), "allgatherv");
    if (lo) DYNPR_CK(cudaMemcpyAsync(b, h, lo, cudaMemcpyHostToDevice, st));
    if (total > hi) DYNPR_CK(cudaMemcpyAsync(b + hi, h + hi, total - hi, cudaMemcpyHostToDevice, st));
    // the staging buffer is reused by the next collective
    DYNPR_CK(cudaStreamSynchronize(st));
  }
  void allreduce_red(SweepRed* red, cudaStream_t st) override {
    auto* h = static_cast<SweepRed*>(small_);
    DYNPR_CK(cudaMemcpyAsync(h, red, sizeof(SweepRed), cudaMemcpyDeviceToHost, st));
    DYNPR_CK(cudaStreamSynchronize(st));
    uint64_t mx[1] = {h->delta_bits};
    uint64_t sm[5] = {h->processed, h->edges, h->pend_edges, h->pend_low, h->pend_high};
    call(ops_.allreduce_u64(mx, 1, 1, user_), "allreduce (max)");
    call(ops_.allreduce_u64(sm, 5, 0, user_), "allreduce (sum)");
    h->delta_bits = mx[0];
    h->processed = sm[0];
    h->edges = sm[1];
    h->pend_edges = sm[2];
    h->pend_low = static_cast<unsigned>(sm[3]);
    h->pend_high = static_cast<unsigned>(sm[4]);
    DYNPR_CK(cudaMemcpyAsync(red, h, sizeof(SweepRed), cudaMemcpyHostToDevice, st));
    DYNPR_CK(cudaStreamSynchronize(st));
  }
  void barrier() override { call(ops_.barrier(user_), "barrier"); }

 private:
  void call(int rc, const char* what) {
    if (rc != 0) throw Error(DYNPR_RUNTIME_ERROR, std::string("team: host transport ") + what + " failed");
  }
  dynpr_comm_ops ops_;
  void* user_;
  void* host_ = nullptr;
  uint64_t host_bytes_ = 0;
  void* small_ = nullptr;
};

// ---- pending-flag bitmap ------------------------------------------------------
__global__ void k_pack_flags(const uint8_t* __restrict__ flags, uint32_t lo, uint32_t hi,
                             uint32_t* __restrict__ seg) {
  const uint32_t w0 = lo >> 5;
  const uint64_t v = ((uint64_t)w0 << 5) + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = v >= lo && v < hi;
  const unsigned bits = __ballot_sync(0xffffffffu, in && flags[in ? v : lo]);
  if ((threadIdx.x & 31) == 0 && v < hi) seg[(v >> 5) - w0] = bits;  // v = the word's first vertex
}

// bounds: lo_0..lo_world (lo_world = n), then seg_0..seg_world (word offsets)
__global__ void k_unpack_flags(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ bounds, int world,
                               int me, uint32_t n, uint8_t* __restrict__ flags) {
  const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  if (v >= bounds[me] && v < bounds[me + 1]) return;  // own range: already current
  int a = 0, b = world;  // owner q: lo_q <= v < lo_{q+1}
  while (b - a > 1) {
    const int mid = (a + b) >> 1;
    if (v >= bounds[mid]) a = mid; else b = mid;
  }
  const uint32_t word = bounds[world + 1 + a] + (uint32_t)((v >> 5) - (bounds[a] >> 5));
  flags[v] = (uint8_t)((bits[word] >> (v & 31)) & 1u);
}

}  // namespace

FlagBitmapPlan make_flag_bitmap_plan(const std::vector<uint32_t>& v_lo, uint32_t n) {
  const int world = (int)v_lo.size();
  FlagBitmapPlan p;
  p.host_bounds.assign(2 * (world + 1), 0);
  p.byte_off.assign(world + 1, 0);
  uint64_t seg = 0;
  for (int r = 0; r < world; ++r) {
    const uint32_t lo = v_lo[r], hi = r + 1 < world ? v_lo[r + 1] : n;
    p.host_bounds[r] = lo;
    p.host_bounds[world + 1 + r] = (uint32_t)seg;
    p.byte_off[r] = 4 * seg;
    if (hi > lo) seg += ((uint64_t)hi + 31) / 32 - lo / 32;
  }
  p.host_bounds[world] = n;
  p.host_bounds[2 * world + 1] = (uint32_t)seg;
  p.byte_off[world] = 4 * seg;
  p.words = seg;
  return p;
}

void launch_pack_flags(dynpr_context* ctx, const uint8_t* flags, uint32_t lo, uint32_t hi, uint32_t* seg_words) {
  if (hi <= lo) return;
  const uint64_t span = (((uint64_t)hi + 31) / 32 - lo / 32) * 32;
  k_pack_flags<<<(unsigned)((span + 255) / 256), 256, 0, ctx->stream>>>(flags, lo, hi, seg_words);
  ctx->launches += 1;
  check_launch();
}

void launch_unpack_flags(dynpr_context* ctx, const uint32_t* bits, const uint32_t* bounds, int world, int me,
                         uint32_t n, uint8_t* flags) {
  if (!n) return;
  k_unpack_flags<<<(n + 255) / 256, 256, 0, ctx->stream>>>(bits, bounds, world, me, n, flags);
  ctx->launches += 1;
  check_launch();
}

std::unique_ptr<Comm> make_host_comm(int rank, int world, const dynpr_comm_ops& ops, void* user) {
  return std::make_unique<HostComm>(rank, world, ops, user);
}

dynpr_status nccl_unique_id(void* out128) {
  return api_guard([&] {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, 128);
  });
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id128) {
  return std::make_unique<NcclComm>(rank, world, id128);
}

std::shared_ptr<LocalTeam> make_local_team(int world) { return std::make_shared<LocalTeam>(world); }
int local_team_world(const LocalTeam& t) { return t.world; }

std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalTeam> team, int rank, int device) {
  return std::make_unique<LocalComm>(std::move(team), rank, device);
}

}  // namespace dynpr_b200
