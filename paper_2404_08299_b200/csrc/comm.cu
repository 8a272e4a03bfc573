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

}  // namespace

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
