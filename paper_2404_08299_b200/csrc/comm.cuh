// Multi-GPU exchange for the range-partitioned engine.
//
// One process (or, for LocalComm, one host thread) per rank; every rank
// holds the full graph and layout, owns a contiguous edge-balanced range of
// the relabelled vertex space, and per sweep exchanges
//   * allgatherv of the owned slice of the contribution vector (8 B/vertex),
//   * allreduce of the 40-byte SweepRed (max of the L-inf bits, sums),
//   * (DF/DF-P) allgatherv of the owned pending flags (1 B/vertex).
// NcclComm implements this with NCCL over NVLink (grouped ncclBroadcast =
// allgatherv, ncclAllReduce), NCCL resolved at run time with dlopen so the
// library has no link-time NCCL dependency.  LocalComm runs P virtual ranks
// on threads of one process (same device or not) with the identical engine
// code path, which is how the partitioned engine is tested bit-exactly on a
// single GPU.
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace dynpr_b200 {

class Comm {
 public:
  virtual ~Comm() = default;
  int rank = 0;
  int world = 1;
  // In place on `buf` (device): rank r's bytes are [off[r], off[r+1]).
  virtual void allgatherv(void* buf, const uint64_t* off, cudaStream_t st) = 0;
  // In place on a device SweepRed: delta_bits max, the counters summed.
  virtual void allreduce_red(SweepRed* red, cudaStream_t st) = 0;
  virtual void barrier() = 0;
  // A rank that fails between collectives calls abort(): ranks blocked in
  // (or later entering) a host-side barrier of the team throw instead of
  // waiting forever.  No-op for NCCL (its collectives are stream-ordered).
  virtual void abort() {}
};

// A context of a range-partitioned team (world > 1, or the DYNPR_FORCE_TEAM
// test hook on a 1-rank team): its layouts hold only the rank's rows and its
// engines exchange after every sweep.
bool team_forced();
bool is_team(const dynpr_context* ctx);

// 128-byte NCCL unique id (ncclUniqueId) from the rank-0 process.
dynpr_status nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id128);

// P virtual ranks in one process: a shared rendezvous the P rank contexts
// attach to.
struct LocalTeam;
std::shared_ptr<LocalTeam> make_local_team(int world);
int local_team_world(const LocalTeam& t);
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalTeam> team, int rank, int device);

// Caller-supplied host transport (dynpr_comm_ops, e.g. torch.distributed
// gloo, MPI): the collectives are staged through pinned host memory.  Any
// number of processes on any devices -- including several processes on one
// GPU, which NCCL refuses -- so the cross-process engine runs on one GPU.
std::unique_ptr<Comm> make_host_comm(int rank, int world, const dynpr_comm_ops& ops, void* user);

// DF/DF-P pending-flag exchange as a bitmap (n/8 bytes per sweep instead of
// n): rank r packs the flags of its vertex range [lo_r, hi_r) into words
// [lo_r/32, ceil(hi_r/32)) of its segment of the bit buffer (segments
// concatenated in rank order); after the all-gather every rank unpacks the
// other ranks' ranges into its byte flags.
struct FlagBitmapPlan {
  std::vector<uint64_t> byte_off;    // allgatherv offsets of the segments (world + 1)
  std::vector<uint32_t> host_bounds; // lo_0..lo_world (= n), seg_0..seg_world (word offsets)
  uint64_t words = 0;                // total words of the bit buffer
};
FlagBitmapPlan make_flag_bitmap_plan(const std::vector<uint32_t>& v_lo, uint32_t n);
// `bounds` = device copy of host_bounds
void launch_pack_flags(dynpr_context* ctx, const uint8_t* flags, uint32_t lo, uint32_t hi, uint32_t* seg_words);
void launch_unpack_flags(dynpr_context* ctx, const uint32_t* bits, const uint32_t* bounds, int world, int me,
                         uint32_t n, uint8_t* flags);

}  // namespace dynpr_b200
