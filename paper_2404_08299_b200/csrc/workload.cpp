// Host-side workload generation (reference workload.cpp:183-249, rng.hpp).
//
// generateRandomBatch draws from one sequential SplitMix64 stream, so it is
// inherently host work; this restatement reproduces the reference's draws
// exactly while avoiding its O(|E|) candidate copy: the deletion candidates
// (all non-loop edges in CSR order) are addressed virtually through a
// per-vertex prefix of non-loop degrees, and the partial Fisher-Yates shuffle
// records only the positions it swapped.  The host CSR is downloaded once
// per graph snapshot and cached with it.
#include <algorithm>
#include <cmath>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "common.cuh"

namespace dynpr_b200 {
namespace {

struct SplitMix64 {  // rng.hpp:10-41
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  uint64_t bounded(uint64_t bound) {
    unsigned __int128 m = static_cast<unsigned __int128>(next()) * bound;
    uint64_t low = static_cast<uint64_t>(m);
    if (low < bound) {
      const uint64_t threshold = -bound % bound;
      while (low < threshold) {
        m = static_cast<unsigned __int128>(next()) * bound;
        low = static_cast<uint64_t>(m);
      }
    }
    return static_cast<uint64_t>(m >> 64);
  }
};

struct HostCsr {
  std::vector<uint64_t> off;
  std::vector<uint32_t> tgt;
  bool has(uint32_t u, uint32_t v) const {
    const uint32_t* b = tgt.data() + off[u];
    const uint32_t* e = tgt.data() + off[u + 1];
    const uint32_t* p = std::lower_bound(b, e, v);
    return p != e && *p == v;
  }
};

}  // namespace
}  // namespace dynpr_b200

using namespace dynpr_b200;

extern "C" {

uint64_t dynpr_batch_size_from_fraction(double fraction, uint64_t total) {
  const double scaled = fraction * static_cast<double>(total);
  const auto rounded = static_cast<uint64_t>(std::floor(scaled + 0.5));
  return rounded < 1 ? 1 : rounded;
}

uint64_t dynpr_derive_seed(uint64_t seed, uint64_t stream) {
  SplitMix64 r{seed ^ (0xD1B54A32D192ED03ULL * (stream + 1))};
  return r.next();
}

dynpr_status dynpr_generate_random_batch(dynpr_context* ctx, const dynpr_graph* g, uint64_t total,
                                         double insert_fraction, uint64_t seed, uint32_t* ins_src,
                                         uint32_t* ins_dst, uint64_t* n_ins, uint32_t* del_src, uint32_t* del_dst,
                                         uint64_t* n_del) {
  NvtxRange nvtx__("dynpr_generate_random_batch");
  return api_guard([&] {
    if (!ctx || !g || !n_ins || !n_del) invalid("null argument");
    if (total < 1) invalid("generateRandomBatch: totalSize must be >= 1");
    if (insert_fraction < 0.0 || insert_fraction > 1.0)
      invalid("generateRandomBatch: insertFraction must be in [0,1]");
    bind_device(ctx);
    const uint32_t n = g->n;
    HostCsr h;
    h.off.resize((size_t)n + 1);
    h.tgt.resize(g->m ? g->m : 1);
    DYNPR_CK(cudaMemcpy(h.off.data(), g->off, ((size_t)n + 1) * 8, cudaMemcpyDeviceToHost));
    if (g->m) DYNPR_CK(cudaMemcpy(h.tgt.data(), g->tgt, g->m * 4, cudaMemcpyDeviceToHost));
    const auto insertCount = static_cast<uint64_t>(std::ceil(insert_fraction * static_cast<double>(total)));
    const uint64_t deleteCount = total - insertCount;
    SplitMix64 rng{seed};
    if (insertCount > 0 && n < 2)
      throw Error(DYNPR_SIZING_ERROR, "generateRandomBatch: need at least 2 vertices for insertions");
    if (insertCount && (!ins_src || !ins_dst)) invalid("null output array");
    // insertions (workload.cpp:204-220)
    std::unordered_set<uint64_t> chosen;
    chosen.reserve(insertCount * 2 + 1);
    const uint64_t maxAttempts = 100 * std::max<uint64_t>(insertCount, 1);
    uint64_t attempts = 0, have = 0;
    while (have < insertCount) {
      if (++attempts > maxAttempts)
        throw Error(DYNPR_SIZING_ERROR, "generateRandomBatch: could not find enough non-existing edges");
      const auto u = static_cast<uint32_t>(rng.bounded(n));
      const auto v = static_cast<uint32_t>(rng.bounded(n));
      if (u == v || h.has(u, v)) continue;
      if (!chosen.insert((static_cast<uint64_t>(u) << 32) | v).second) continue;
      ins_src[have] = u;
      ins_dst[have] = v;
      ++have;
    }
    *n_ins = insertCount;
    *n_del = 0;
    if (deleteCount == 0) return;
    if (!del_src || !del_dst) invalid("null output array");
    // deletions (workload.cpp:224-241): virtual candidate array
    std::vector<uint64_t> pre((size_t)n + 1, 0);  // non-loop edges before vertex u
    std::vector<int64_t> loopPos(n, -1);           // slice index of (u,u) or -1
    for (uint32_t u = 0; u < n; ++u) {
      const uint64_t b = h.off[u], e = h.off[u + 1];
      const uint32_t* p = std::lower_bound(h.tgt.data() + b, h.tgt.data() + e, u);
      const bool loop = p != h.tgt.data() + e && *p == u;
      if (loop) loopPos[u] = p - (h.tgt.data() + b);
      pre[u + 1] = pre[u] + (e - b) - (loop ? 1 : 0);
    }
    const uint64_t nc = pre[n];
    if (deleteCount > nc)
      throw Error(DYNPR_SIZING_ERROR, "generateRandomBatch: requested " + std::to_string(deleteCount) +
                                          " deletions but only " + std::to_string(nc) + " non-loop edges exist");
    auto edgeAt = [&](uint64_t k, uint32_t& u, uint32_t& v) {
      u = static_cast<uint32_t>(std::upper_bound(pre.begin(), pre.end(), k) - pre.begin() - 1);
      uint64_t r = k - pre[u];
      if (loopPos[u] >= 0 && r >= static_cast<uint64_t>(loopPos[u])) ++r;
      v = h.tgt[h.off[u] + r];
    };
    std::unordered_map<uint64_t, uint64_t> swapped;
    swapped.reserve(deleteCount * 2 + 1);
    auto at = [&](uint64_t i) {
      auto it = swapped.find(i);
      return it == swapped.end() ? i : it->second;
    };
    for (uint64_t i = 0; i < deleteCount; ++i) {
      const uint64_t j = i + rng.bounded(nc - i);
      const uint64_t ci = at(i), cj = at(j);
      swapped[i] = cj;
      swapped[j] = ci;
      uint32_t u, v;
      edgeAt(cj, u, v);
      del_src[i] = u;
      del_dst[i] = v;
    }
    *n_del = deleteCount;
  });
}

}  // extern "C"
