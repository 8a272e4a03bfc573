// Input formats and the experiment harness: the callers either side of the
// hot path.
//
//  * loadMatrixMarket / loadTemporalEdgeList / splitTemporal
//    (workload.cpp:43-181): the file is memory-mapped and tokenised in place
//    with std::from_chars -- same token rules as the reference's
//    getline + istringstream (whitespace = C-locale isspace, one trailing
//    '\r' chomped, comment tests on the raw first byte), same ParseError
//    texts and line numbers -- instead of a stringstream per line.
//  * runExperiment / summarizeRows / emitReport (harness.cpp:68-399): the
//    static, random-batch and temporal protocols driven through this
//    library's device engines.  Every graph lives on the device: the base
//    CSR pair is built there (buildCsr + addSelfLoops + transpose), each
//    batch is ingested with apply_batch_pair (forward and transpose updated
//    together, byte-identical to applyBatch + transpose), the 500-sweep
//    reference ranks (computeReferenceRanks) and the L1 errors are computed
//    on the device, and the chained warm-start ranks never leave it.  Only
//    the report rows come back to the host.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <exception>
#include <thread>
#include <utility>
#include <vector>

#include "common.cuh"

struct dynpr_edge_list {
  uint32_t n = 0;
  std::vector<uint32_t> src, dst;
  std::vector<int64_t> ts;  // empty unless a temporal stream
  bool temporal = false;
};

struct dynpr_report {
  struct Row {
    std::string graph, approach, spec;
    int64_t batch_index = 0;
    double runtime = 0.0;
    int64_t iterations = 0;
    uint64_t affected = 0;
    double l1 = 0.0;
    bool converged = false;
  };
  std::vector<Row> rows;
};

namespace dynpr_b200 {
namespace {

[[noreturn]] void parse_error(const std::string& path, uint64_t line, const std::string& what) {
  throw Error(DYNPR_PARSE_ERROR, path + ":" + std::to_string(line) + ": " + what);
}

// Read-only memory map of a whole file (empty files map to nothing).
struct MappedFile {
  const char* data = nullptr;
  size_t size = 0;
  explicit MappedFile(const std::string& path) {
    int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) throw Error(DYNPR_RUNTIME_ERROR, "cannot open " + path);
    struct stat st;
    if (::fstat(fd, &st) != 0 || S_ISDIR(st.st_mode)) {
      ::close(fd);
      throw Error(DYNPR_RUNTIME_ERROR, "cannot open " + path);
    }
    size = static_cast<size_t>(st.st_size);
    if (size) {
      void* p = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (p == MAP_FAILED) {
        ::close(fd);
        throw Error(DYNPR_RUNTIME_ERROR, "cannot open " + path);
      }
      ::madvise(p, size, MADV_SEQUENTIAL);
      data = static_cast<const char*>(p);
    }
    ::close(fd);
  }
  ~MappedFile() {
    if (data) ::munmap(const_cast<char*>(data), size);
  }
};

// std::getline over the mapped bytes: yields [b, e) without the '\n', then
// chomps one '\r' (workload.cpp:34-36).  A final line without '\n' counts;
// an empty file yields no line.
struct LineReader {
  const char* p;
  const char* end;
  LineReader(const MappedFile& f) : p(f.data), end(f.data + f.size) {}
  bool next(const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(memchr(p, '\n', static_cast<size_t>(end - p)));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    if (e > b && e[-1] == '\r') --e;
    return true;
  }
};

inline bool is_space(char c) {  // isspace in the "C" locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// istream >> std::string: skip whitespace, take the next non-space run
// (empty when the line is exhausted).
struct Tokens {
  const char* p;
  const char* e;
  std::pair<const char*, const char*> next() {
    while (p < e && is_space(*p)) ++p;
    const char* b = p;
    while (p < e && !is_space(*p)) ++p;
    return {b, p};
  }
};

template <class T>
bool parse_num(std::pair<const char*, const char*> tok, T& out) {  // workload.cpp:22-30
  auto [p, ec] = std::from_chars(tok.first, tok.second, out);
  return ec == std::errc() && p == tok.second;
}

std::string lower(std::pair<const char*, const char*> tok) {
  std::string s(tok.first, tok.second);
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// ---- parallel body parsing ----------------------------------------------------
// Files above kParallelBytes are split into line-aligned chunks parsed by
// host threads; every chunk reports its line count and its first error, and
// the chunks are stitched in file order, so the result -- arrays, error
// class, message and line number -- is exactly the sequential reading's.
// DYNPR_PARSE_THREADS overrides the thread count (tests force the parallel
// path on small files with it).
constexpr size_t kParallelBytes = size_t(8) << 20;

unsigned parse_threads(size_t body_bytes) {
  if (const char* e = std::getenv("DYNPR_PARSE_THREADS")) {
    const long t = std::strtol(e, nullptr, 10);
    if (t >= 1) return (unsigned)std::min<long>(t, 256);
  }
  if (body_bytes < kParallelBytes) return 1;
  const unsigned hc = std::thread::hardware_concurrency();
  return std::max(1u, std::min(hc ? hc : 1u, 64u));
}

// [b, e) cut into up to `t` pieces, each ending just after a '\n' (the last
// at e).
std::vector<const char*> split_lines(const char* b, const char* e, unsigned t) {
  std::vector<const char*> cuts{b};
  const size_t len = static_cast<size_t>(e - b);
  for (unsigned k = 1; k < t; ++k) {
    const char* p = b + len * k / t;
    if (p <= cuts.back()) continue;
    const char* nl = static_cast<const char*>(memchr(p, '\n', static_cast<size_t>(e - p)));
    if (!nl) break;
    if (nl + 1 > cuts.back() && nl + 1 < e) cuts.push_back(nl + 1);
  }
  cuts.push_back(e);
  return cuts;
}

template <class F>
void parallel_for(size_t n, F&& f) {
  if (n <= 1) {
    if (n) f(0);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> errs(n);
  for (size_t k = 0; k < n; ++k)
    th.emplace_back([&, k] {
      try {
        f(k);
      } catch (...) {
        errs[k] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& x : errs)
    if (x) std::rethrow_exception(x);
}

// Lines of [b, e) as LineReader yields them.
struct ChunkLines {
  const char* p;
  const char* end;
  bool next(const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(memchr(p, '\n', static_cast<size_t>(end - p)));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    if (e > b && e[-1] == '\r') --e;
    return true;
  }
};

struct MMChunk {
  std::vector<uint32_t> u, v;  // entries (before symmetric expansion)
  uint64_t lines = 0;
  uint64_t err_line = 0;       // 1-based within the chunk; 0 = none
  const char* err_what = nullptr;
};

void parse_mm_chunk(const char* b0, const char* e0, uint64_t rows, uint64_t cols, MMChunk& out) {
  ChunkLines lines{b0, e0};
  const char *b, *e;
  while (lines.next(b, e)) {
    ++out.lines;
    if (e == b || *b == '%') continue;
    Tokens t{b, e};
    auto si = t.next(), sj = t.next();
    uint64_t i = 0, j = 0;
    if (!parse_num(si, i) || !parse_num(sj, j)) {
      out.err_line = out.lines;
      out.err_what = "malformed entry";
      return;
    }
    if (i < 1 || i > rows || j < 1 || j > cols) {
      out.err_line = out.lines;
      out.err_what = "index out of declared bounds";
      return;
    }
    out.u.push_back(static_cast<uint32_t>(i - 1));
    out.v.push_back(static_cast<uint32_t>(j - 1));
  }
}

// loadMatrixMarket -- workload.cpp:43-107.
dynpr_edge_list* load_matrix_market(const std::string& path) {
  MappedFile f(path);
  LineReader lines(f);
  const char *b, *e;
  uint64_t line_no = 0;
  if (!lines.next(b, e)) parse_error(path, 1, "empty file");
  ++line_no;
  Tokens header{b, e};
  const std::string banner = lower(header.next()), object = lower(header.next()),
                    format = lower(header.next());
  header.next();  // field
  const std::string symmetry = lower(header.next());
  if (banner != "%%matrixmarket") parse_error(path, line_no, "missing %%MatrixMarket banner");
  if (object != "matrix" || format != "coordinate")
    parse_error(path, line_no, "only 'matrix coordinate' files are supported");
  const bool symmetric = symmetry == "symmetric" || symmetry == "skew-symmetric" || symmetry == "hermitian";

  uint64_t rows = 0, cols = 0, declared = 0;
  for (;;) {
    if (!lines.next(b, e)) parse_error(path, line_no + 1, "missing size line");
    ++line_no;
    if (e == b || *b == '%') continue;
    Tokens t{b, e};
    auto r = t.next(), c = t.next(), z = t.next();
    if (!parse_num(r, rows) || !parse_num(c, cols) || !parse_num(z, declared))
      parse_error(path, line_no, "malformed size line");
    break;
  }
  auto out = std::make_unique<dynpr_edge_list>();
  out->n = static_cast<uint32_t>(std::max(rows, cols));
  // body: chunks parsed in parallel, stitched in order up to `declared`
  // entries (the reference never reads past them, so a bad line after the
  // last declared entry is not an error)
  const char* body = lines.p;
  const char* end = lines.end;
  const auto cuts = split_lines(body, end, parse_threads(static_cast<size_t>(end - body)));
  std::vector<MMChunk> ch(cuts.size() - 1);
  parallel_for(ch.size(), [&](size_t k) { parse_mm_chunk(cuts[k], cuts[k + 1], rows, cols, ch[k]); });
  uint64_t seen = 0, take_chunks = 0, last_take = 0;
  for (size_t k = 0; k < ch.size(); ++k) {
    const uint64_t need = declared - seen;
    if (ch[k].u.size() >= need) {  // the declared count is reached inside this chunk
      take_chunks = k + 1;
      last_take = need;
      seen = declared;
      break;
    }
    if (ch[k].err_line) parse_error(path, line_no + ch[k].err_line, ch[k].err_what);
    seen += ch[k].u.size();
    line_no += ch[k].lines;
    take_chunks = k + 1;
    last_take = ch[k].u.size();
  }
  if (seen < declared)
    parse_error(path, line_no + 1,
                "expected " + std::to_string(declared) + " entries, got " + std::to_string(seen));
  // output offsets per chunk (symmetric off-diagonal entries emit both
  // directions, in entry order)
  std::vector<uint64_t> base(take_chunks + 1, 0);
  for (size_t k = 0; k < take_chunks; ++k) {
    const uint64_t cnt = k + 1 == take_chunks ? last_take : ch[k].u.size();
    uint64_t edges = cnt;
    if (symmetric)
      for (uint64_t i = 0; i < cnt; ++i) edges += ch[k].u[i] != ch[k].v[i];
    base[k + 1] = base[k] + edges;
  }
  out->src.resize(base[take_chunks]);
  out->dst.resize(base[take_chunks]);
  parallel_for(take_chunks, [&](size_t k) {
    const uint64_t cnt = k + 1 == take_chunks ? last_take : ch[k].u.size();
    uint64_t o = base[k];
    for (uint64_t i = 0; i < cnt; ++i) {
      const uint32_t u = ch[k].u[i], v = ch[k].v[i];
      out->src[o] = u;
      out->dst[o++] = v;
      if (symmetric && u != v) {
        out->src[o] = v;
        out->dst[o++] = u;
      }
    }
  });
  return out.release();
}

// Open-addressing hash map uint64 -> uint64 (linear probing, power-of-two
// capacity, grows at 1/2 load) -- the id compaction's hot structure.
struct U64Map {
  static constexpr uint64_t kEmpty = ~0ull;
  std::vector<uint64_t> keys, vals;
  uint64_t mask = 0, size = 0;
  explicit U64Map(uint64_t cap = 1024) { init(cap); }
  void init(uint64_t cap) {
    uint64_t c = 16;
    while (c < cap) c <<= 1;
    keys.assign(c, kEmpty);
    vals.assign(c, 0);
    mask = c - 1;
    size = 0;
  }
  static uint64_t hash(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    return k;
  }
  // inserts (k, v) if k is absent (the raw id ~0 is kept aside: never a key)
  void emplace(uint64_t k, uint64_t v) {
    if ((size + 1) * 2 > mask + 1) grow();
    uint64_t i = hash(k) & mask;
    while (keys[i] != kEmpty) {
      if (keys[i] == k) return;
      i = (i + 1) & mask;
    }
    keys[i] = k;
    vals[i] = v;
    ++size;
  }
  uint64_t at(uint64_t k) const {
    uint64_t i = hash(k) & mask;
    while (keys[i] != k) i = (i + 1) & mask;
    return vals[i];
  }
  void grow() {
    std::vector<uint64_t> ok = std::move(keys), ov = std::move(vals);
    init((mask + 1) * 2);
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != kEmpty) emplace(ok[i], ov[i]);
  }
};

struct TChunk {
  std::vector<uint64_t> s, d;
  std::vector<int64_t> ts;
  uint64_t lines = 0;
  uint64_t err_line = 0;
};

void parse_temporal_chunk(const char* b0, const char* e0, TChunk& out) {
  ChunkLines lines{b0, e0};
  const char *b, *e;
  while (lines.next(b, e)) {
    ++out.lines;
    if (e == b || *b == '#') continue;
    Tokens t{b, e};
    auto a = t.next(), c = t.next(), z = t.next();
    uint64_t src = 0, dst = 0;
    int64_t stamp = 0;
    if (!parse_num(a, src) || !parse_num(c, dst) || !parse_num(z, stamp)) {
      out.err_line = out.lines;
      return;
    }
    out.s.push_back(src);
    out.d.push_back(dst);
    out.ts.push_back(stamp);
  }
}

// loadTemporalEdgeList -- workload.cpp:109-136.  Raw ids are compacted in
// first-appearance order (source before target within a line): the
// (raw id, position) pairs are hash-partitioned into buckets, each bucket
// keeps the first position of its ids (chunks visited in file order), the
// distinct ids are ranked by first position, and the entries mapped in
// parallel.  The entries are then stably sorted by timestamp.
dynpr_edge_list* load_temporal(const std::string& path) {
  MappedFile f(path);
  const char* body = f.data;
  const char* end = f.data + f.size;
  const unsigned T = parse_threads(f.size);
  const auto cuts = split_lines(body, end, T);
  std::vector<TChunk> ch(cuts.size() - 1);
  const bool dbg = std::getenv("DYNPR_PARSE_DEBUG") != nullptr;
  auto tick = [&, t0 = std::chrono::steady_clock::now()](const char* what) mutable {
    if (!dbg) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "load_temporal %-10s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  parallel_for(ch.size(), [&](size_t k) { parse_temporal_chunk(cuts[k], cuts[k + 1], ch[k]); });
  tick("parse");
  uint64_t line_no = 0, total = 0;
  std::vector<uint64_t> first(ch.size() + 1, 0);
  for (size_t k = 0; k < ch.size(); ++k) {
    if (ch[k].err_line) parse_error(path, line_no + ch[k].err_line, "expected 'src dst timestamp'");
    line_no += ch[k].lines;
    first[k] = total;
    total += ch[k].s.size();
  }
  first[ch.size()] = total;

  auto out = std::make_unique<dynpr_edge_list>();
  out->temporal = true;
  const size_t P = ch.size();
  auto bucket_of = [P](uint64_t raw) {
    return P == 1 ? size_t(0) : static_cast<size_t>((raw * 0x9E3779B97F4A7C15ULL) >> 32) % P;
  };
  // per-bucket maps raw -> first position (2 * entry + {0 src, 1 dst});
  // every bucket thread walks the chunks in file order and keeps its ids.
  // The raw id ~0 (the maps' empty marker) is tracked on the side.
  std::vector<U64Map> firstpos(P);
  uint64_t max_first = ~0ull;  // first position of raw id ~0, if present
  parallel_for(P, [&](size_t bkt) {
    auto& mp = firstpos[bkt];
    for (size_t k = 0; k < ch.size(); ++k)
      for (uint64_t i = 0; i < ch[k].s.size(); ++i) {
        const uint64_t pos = 2 * (first[k] + i);
        const uint64_t a = ch[k].s[i], c = ch[k].d[i];
        if (a != U64Map::kEmpty && bucket_of(a) == bkt) mp.emplace(a, pos);
        if (c != U64Map::kEmpty && bucket_of(c) == bkt) mp.emplace(c, pos + 1);
      }
  });
  tick("firstpos");
  for (size_t k = 0; k < ch.size() && max_first == ~0ull; ++k)
    for (uint64_t i = 0; i < ch[k].s.size(); ++i) {
      const uint64_t pos = 2 * (first[k] + i);
      if (ch[k].s[i] == U64Map::kEmpty) { max_first = pos; break; }
      if (ch[k].d[i] == U64Map::kEmpty) { max_first = pos + 1; break; }
    }
  // dense ids in first-appearance order
  std::vector<std::pair<uint64_t, uint64_t>> order;  // (first pos, raw)
  for (const auto& mp : firstpos)
    for (size_t i = 0; i < mp.keys.size(); ++i)
      if (mp.keys[i] != U64Map::kEmpty) order.emplace_back(mp.vals[i], mp.keys[i]);
  if (max_first != ~0ull) order.emplace_back(max_first, U64Map::kEmpty);
  std::sort(order.begin(), order.end());
  uint32_t id_of_max = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    if (order[i].second == U64Map::kEmpty) {
      id_of_max = (uint32_t)i;
      continue;
    }
    auto& mp = firstpos[bucket_of(order[i].second)];  // reuse: value := dense id
    uint64_t j = U64Map::hash(order[i].second) & mp.mask;
    while (mp.keys[j] != order[i].second) j = (j + 1) & mp.mask;
    mp.vals[j] = i;
  }
  tick("order");
  out->n = static_cast<uint32_t>(order.size());
  std::vector<uint32_t> s(total), d(total);
  std::vector<int64_t> ts(total);
  auto dense = [&](uint64_t raw) -> uint32_t {
    return raw == U64Map::kEmpty ? id_of_max : (uint32_t)firstpos[bucket_of(raw)].at(raw);
  };
  parallel_for(ch.size(), [&](size_t k) {
    for (uint64_t i = 0; i < ch[k].s.size(); ++i) {
      s[first[k] + i] = dense(ch[k].s[i]);
      d[first[k] + i] = dense(ch[k].d[i]);
      ts[first[k] + i] = ch[k].ts[i];
    }
  });
  tick("map");
  const size_t cnt = ts.size();
  if (std::is_sorted(ts.begin(), ts.end())) {
    out->src = std::move(s);
    out->dst = std::move(d);
    out->ts = std::move(ts);
  } else {
    std::vector<uint64_t> perm(cnt);
    for (size_t i = 0; i < cnt; ++i) perm[i] = i;
    std::stable_sort(perm.begin(), perm.end(), [&](uint64_t x, uint64_t y) { return ts[x] < ts[y]; });
    out->src.resize(cnt);
    out->dst.resize(cnt);
    out->ts.resize(cnt);
    for (size_t i = 0; i < cnt; ++i) {
      out->src[i] = s[perm[i]];
      out->dst[i] = d[perm[i]];
      out->ts[i] = ts[perm[i]];
    }
  }
  return out.release();
}

// splitTemporal -- workload.cpp:138-181 (base part; the batches are ranges
// of the stream).
uint64_t split_base_count(const dynpr_edge_list* t, double base_fraction, int32_t batch_count,
                          uint64_t batch_size) {
  if (!(base_fraction > 0.0 && base_fraction < 1.0))
    invalid("splitTemporal: baseFraction must be in (0,1)");
  if (batch_count < 1 || batch_size < 1) invalid("splitTemporal: batchCount and batchSize must be >= 1");
  const uint64_t total = t->src.size();
  const auto base = static_cast<uint64_t>(std::floor(base_fraction * static_cast<double>(total)));
  const uint64_t needed = base + static_cast<uint64_t>(batch_count) * batch_size;
  if (needed > total) {
    const uint64_t fit = (total - std::min(base, total)) / batch_size;
    throw Error(DYNPR_SIZING_ERROR, "splitTemporal: stream has " + std::to_string(total) + " entries; only " +
                                        std::to_string(fit) + " of " + std::to_string(batch_count) +
                                        " batches of size " + std::to_string(batch_size) + " fit after the base");
  }
  return base;
}

dynpr_edge_list* split_base(const dynpr_edge_list* t, uint64_t base) {
  auto out = std::make_unique<dynpr_edge_list>();
  out->n = t->n;
  std::vector<uint64_t> keys(base);
  for (uint64_t i = 0; i < base; ++i) keys[i] = (uint64_t(t->src[i]) << 32) | t->dst[i];
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  out->src.resize(keys.size());
  out->dst.resize(keys.size());
  for (size_t i = 0; i < keys.size(); ++i) {
    out->src[i] = static_cast<uint32_t>(keys[i] >> 32);
    out->dst[i] = static_cast<uint32_t>(keys[i]);
  }
  return out.release();
}

// ---- harness ----------------------------------------------------------------

using Clock = std::chrono::steady_clock;

const char* approach_name(int32_t a) {  // harness.cpp:318-327
  switch (a) {
    case DYNPR_APPROACH_STATIC: return "static";
    case DYNPR_APPROACH_ND: return "nd";
    case DYNPR_APPROACH_DT: return "dt";
    case DYNPR_APPROACH_DF: return "df";
    case DYNPR_APPROACH_DFP: return "dfp";
  }
  invalid("unknown approach");
}

std::string file_stem(const std::string& path) {  // harness.cpp:26-32
  const auto slash = path.find_last_of("/\\");
  std::string name = slash == std::string::npos ? path : path.substr(slash + 1);
  const auto dot = name.find_last_of('.');
  if (dot != std::string::npos && dot > 0) name = name.substr(0, dot);
  return name;
}

double stod_like(const std::string& s) {  // std::stod: leading space, prefix parse
  const char* b = s.c_str();
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(b, &end);
  if (end == b) invalid("stod");
  if (errno == ERANGE && (v == HUGE_VAL || v == -HUGE_VAL)) invalid("stod");
  return v;
}

// Status -> exception, keeping the library's message.
void ck(dynpr_status st) {
  if (st != DYNPR_OK) throw Error(st, dynpr_last_error());
}

struct Graph {  // owning handle
  dynpr_graph* g = nullptr;
  Graph() = default;
  explicit Graph(dynpr_graph* h) : g(h) {}
  Graph(Graph&& o) noexcept : g(o.g) { o.g = nullptr; }
  Graph& operator=(Graph&& o) noexcept {
    if (this != &o) {
      if (g) dynpr_graph_destroy(g);
      g = o.g;
      o.g = nullptr;
    }
    return *this;
  }
  ~Graph() {
    if (g) dynpr_graph_destroy(g);
  }
  uint64_t m() const {
    uint32_t n;
    uint64_t m;
    dynpr_graph_info(g, &n, &m);
    return m;
  }
  uint32_t n() const {
    uint32_t n;
    uint64_t m;
    dynpr_graph_info(g, &n, &m);
    return n;
  }
};

struct Pair {  // harness.cpp:117-127 LoadedGraph
  Graph forward, transposed;
};

Pair augment_and_transpose(dynpr_context* ctx, const std::vector<uint32_t>& s, const std::vector<uint32_t>& d,
                           uint32_t n) {
  dynpr_graph *raw = nullptr, *loops = nullptr, *t = nullptr;
  ck(dynpr_graph_build(ctx, n, s.data(), d.data(), s.size(), &raw));
  Graph graw(raw);
  ck(dynpr_graph_add_self_loops(ctx, raw, &loops));
  Pair p;
  p.forward = Graph(loops);
  ck(dynpr_graph_transpose(ctx, loops, &t));
  p.transposed = Graph(t);
  return p;
}

// Host batch (edge-list pairs) staged once to the device for the engines.
struct Batch {
  std::vector<uint32_t> ds, dd, is, id;
};

struct Runner {
  dynpr_context* ctx;
  const dynpr_experiment_spec& spec;
  const std::string graph_name;
  dynpr_report* rep;
  uint32_t n = 0;

  // Chain ranks per approach (harness.cpp:140-149), device-resident.
  std::map<int32_t, std::unique_ptr<DevBuf>> chain;
  DevBuf reference, result, scratch;

  double* chain_of(int32_t a) { return chain.at(a)->as<double>(n); }

  void reset_chains(const double* from) {
    for (int i = 0; i < spec.n_approaches; ++i) {
      auto& slot = chain[spec.approaches[i]];
      if (!slot) slot = std::make_unique<DevBuf>();
      DYNPR_CK(cudaMemcpyAsync(slot->as<double>(n), from, n * sizeof(double), cudaMemcpyDeviceToDevice,
                               ctx->stream));
    }
    sync(ctx);
  }

  // harness.cpp:34-54 runApproach
  void run_approach(int32_t a, const Pair& p, const Batch& b, const double* prev, double* out, dynpr_stats* st) {
    const dynpr_config* c = &spec.config;
    switch (a) {
      case DYNPR_APPROACH_STATIC:
        ck(dynpr_static_pagerank(ctx, p.transposed.g, p.forward.g, c, out, st, nullptr, nullptr));
        return;
      case DYNPR_APPROACH_ND:
        ck(dynpr_naive_dynamic(ctx, p.transposed.g, p.forward.g, prev, n, c, out, st, nullptr, nullptr));
        return;
      case DYNPR_APPROACH_DT:
        ck(dynpr_dynamic_traversal(ctx, p.forward.g, p.transposed.g, b.ds.data(), b.dd.data(), b.ds.size(),
                                   b.is.data(), b.id.data(), b.is.size(), prev, n, c, out, st, nullptr, nullptr));
        return;
      case DYNPR_APPROACH_DF:
      case DYNPR_APPROACH_DFP:
        ck(dynpr_dynamic_frontier(ctx, p.forward.g, p.transposed.g, b.ds.data(), b.dd.data(), b.ds.size(),
                                  b.is.data(), b.id.data(), b.is.size(), prev, n, c, a == DYNPR_APPROACH_DFP, out,
                                  st, nullptr, nullptr));
        return;
    }
    invalid("unknown approach");
  }

  void reference_ranks(const Pair& p, double* out) {  // harness.cpp:340-349
    ck(dynpr_compute_reference_ranks(ctx, p.transposed.g, p.forward.g, &spec.config, out));
  }

  dynpr_report::Row row(int32_t a, const std::string& size_spec, int64_t index, double ms, const dynpr_stats& st,
                        double l1) {
    dynpr_report::Row r;
    r.graph = graph_name;
    r.approach = approach_name(a);
    r.spec = size_spec;
    r.batch_index = index;
    r.runtime = spec.record_timing ? ms : 0.0;
    r.iterations = st.iterations;
    r.affected = st.affected_vertex_iterations;
    r.l1 = l1;
    r.converged = st.converged != 0;
    return r;
  }

  // harness.cpp:129-155 runBatchStep
  void batch_step(const Pair& p, const Batch& b, const std::string& size_spec, int64_t index) {
    double* ref = reference.as<double>(n);
    reference_ranks(p, ref);
    double* out = result.as<double>(n);
    for (int i = 0; i < spec.n_approaches; ++i) {
      const int32_t a = spec.approaches[i];
      const double* prev = chain_of(a);
      dynpr_stats st{};
      const auto t0 = Clock::now();
      run_approach(a, p, b, prev, out, &st);
      const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
      double l1 = 0.0;
      ck(dynpr_l1_norm_delta(ctx, out, ref, n, &l1));
      rep->rows.push_back(row(a, size_spec, index, ms, st, l1));
      if (a != DYNPR_APPROACH_STATIC) {
        const double* keep = spec.chain_mode == DYNPR_CHAIN_SHARED_REFERENCE ? ref : out;
        DYNPR_CK(cudaMemcpyAsync(chain_of(a), keep, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        sync(ctx);
      }
    }
  }

  // Snapshots are immutable; the engine layout is built once per ingested
  // pair here (like the reference's transpose, outside the timed region).
  void prepare(const Pair& p, bool forward) {
    ck(dynpr_graph_prepare(ctx, p.transposed.g, p.forward.g, spec.config.low_degree_threshold, forward ? 1 : 0,
                           nullptr));
  }

  bool needs_forward() const {
    for (int i = 0; i < spec.n_approaches; ++i)
      if (spec.approaches[i] != DYNPR_APPROACH_STATIC && spec.approaches[i] != DYNPR_APPROACH_ND) return true;
    return false;
  }

  Pair apply(const Pair& p, const Batch& b) {
    dynpr_graph *gf = nullptr, *gt = nullptr;
    ck(dynpr_graph_apply_batch_pair(ctx, p.forward.g, p.transposed.g, b.ds.data(), b.dd.data(), b.ds.size(),
                                    b.is.data(), b.id.data(), b.is.size(), &gf, &gt, nullptr, nullptr));
    Pair q;
    q.forward = Graph(gf);
    q.transposed = Graph(gt);
    return q;
  }

  // harness.cpp:241-270 runStatic
  void run_static() {
    std::unique_ptr<dynpr_edge_list> mm(load_matrix_market(spec.graph_path));
    n = mm->n;
    Pair p = augment_and_transpose(ctx, mm->src, mm->dst, mm->n);
    n = p.forward.n();
    double* ref = reference.as<double>(n);
    reference_ranks(p, ref);
    double* out = result.as<double>(n);
    for (int rep_i = 0; rep_i < spec.repetitions; ++rep_i) {
      dynpr_stats st{};
      const auto t0 = Clock::now();
      ck(dynpr_static_pagerank(ctx, p.transposed.g, p.forward.g, &spec.config, out, &st, nullptr, nullptr));
      const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
      double l1 = 0.0;
      ck(dynpr_l1_norm_delta(ctx, out, ref, n, &l1));
      rep->rows.push_back(row(DYNPR_APPROACH_STATIC, "0", rep_i, ms, st, l1));
    }
  }

  // harness.cpp:211-239 runRandomBatch
  void run_random() {
    std::unique_ptr<dynpr_edge_list> mm(load_matrix_market(spec.graph_path));
    Pair base = augment_and_transpose(ctx, mm->src, mm->dst, mm->n);
    mm.reset();
    n = base.forward.n();
    const uint64_t m = base.forward.m();
    DevBuf base_ranks;
    ck(dynpr_static_pagerank(ctx, base.transposed.g, base.forward.g, &spec.config, base_ranks.as<double>(n),
                             nullptr, nullptr, nullptr));
    for (int si = 0; si < spec.n_batch_size_specs; ++si) {
      const std::string size_spec = spec.batch_size_specs[si];
      const uint64_t size = dynpr_batch_size_from_fraction(stod_like(size_spec), m);
      for (int r = 0; r < spec.repetitions; ++r) {
        const uint64_t sub = dynpr_derive_seed(spec.seed, uint64_t(si) * 1000003ULL + uint64_t(r));
        Batch b;
        b.is.resize(size);
        b.id.resize(size);
        b.ds.resize(size);
        b.dd.resize(size);
        uint64_t ni = 0, nd = 0;
        ck(dynpr_generate_random_batch(ctx, base.forward.g, size, spec.insert_fraction, sub, b.is.data(),
                                       b.id.data(), &ni, b.ds.data(), b.dd.data(), &nd));
        b.is.resize(ni);
        b.id.resize(ni);
        b.ds.resize(nd);
        b.dd.resize(nd);
        Pair p = apply(base, b);
        prepare(p, needs_forward());
        reset_chains(base_ranks.as<double>(n));
        batch_step(p, b, size_spec, r);
      }
    }
  }

  // harness.cpp:157-182 runTemporal
  void run_temporal() {
    std::unique_ptr<dynpr_edge_list> stream(load_temporal(spec.graph_path));
    for (int si = 0; si < spec.n_batch_size_specs; ++si) {
      const std::string size_spec = spec.batch_size_specs[si];
      const uint64_t size = dynpr_batch_size_from_fraction(stod_like(size_spec), stream->src.size());
      const uint64_t base_count = split_base_count(stream.get(), spec.base_fraction, spec.batch_count, size);
      std::unique_ptr<dynpr_edge_list> base(split_base(stream.get(), base_count));
      Pair p = augment_and_transpose(ctx, base->src, base->dst, stream->n);
      base.reset();
      n = p.forward.n();
      DevBuf initial;
      ck(dynpr_static_pagerank(ctx, p.transposed.g, p.forward.g, &spec.config, initial.as<double>(n), nullptr,
                               nullptr, nullptr));
      reset_chains(initial.as<double>(n));
      for (int bi = 0; bi < spec.batch_count; ++bi) {
        Batch b;
        const uint64_t first = base_count + uint64_t(bi) * size;
        b.is.assign(stream->src.begin() + first, stream->src.begin() + first + size);
        b.id.assign(stream->dst.begin() + first, stream->dst.begin() + first + size);
        Pair q = apply(p, b);
        p = std::move(q);
        prepare(p, needs_forward());
        batch_step(p, b, size_spec, bi);
      }
    }
  }
};

// summarizeRows (harness.cpp:56-113): one summary row per (approach, batch
// size spec), in order of first appearance.  Means are accumulated in row
// order as the rows stream past: the geometric means as running log sums
// (exp(sum / count), 0 once a non-positive value is seen), the counters as
// running sums rounded at the end; NaN errors are left out of the error mean
// and a group without errors reports NaN.
struct RunningSummary {
  std::string graph, approach, spec;
  uint64_t rows = 0;
  double log_runtime = 0.0;
  bool runtime_nonpositive = false;
  uint64_t errors = 0;
  double log_error = 0.0;
  bool error_nonpositive = false;
  double iterations = 0.0, affected = 0.0;
  bool converged = true;

  static void add_log(double v, double& log_sum, bool& nonpositive) {
    if (v > 0.0)
      log_sum += std::log(v);
    else
      nonpositive = true;
  }
  void add(const dynpr_report::Row& r) {
    ++rows;
    add_log(r.runtime, log_runtime, runtime_nonpositive);
    if (!std::isnan(r.l1)) {
      ++errors;
      add_log(r.l1, log_error, error_nonpositive);
    }
    iterations += static_cast<double>(r.iterations);
    affected += static_cast<double>(r.affected);
    converged = converged && r.converged;
  }
  static double geo(uint64_t count, double log_sum, bool nonpositive) {
    return (count == 0 || nonpositive) ? 0.0 : std::exp(log_sum / static_cast<double>(count));
  }
  dynpr_report::Row row() const {
    dynpr_report::Row s;
    s.graph = graph;
    s.approach = approach;
    s.spec = spec;
    s.batch_index = -1;
    s.runtime = geo(rows, log_runtime, runtime_nonpositive);
    s.l1 = errors ? geo(errors, log_error, error_nonpositive) : std::nan("");
    s.iterations = static_cast<int64_t>(std::llround(iterations / static_cast<double>(rows)));
    s.affected = static_cast<uint64_t>(std::llround(affected / static_cast<double>(rows)));
    s.converged = converged;
    return s;
  }
};

std::vector<dynpr_report::Row> summarize(const std::vector<dynpr_report::Row>& rows) {
  std::vector<RunningSummary> groups;  // a handful: (approach, spec) pairs
  for (const auto& r : rows) {
    auto g = std::find_if(groups.begin(), groups.end(),
                          [&](const RunningSummary& x) { return x.approach == r.approach && x.spec == r.spec; });
    if (g == groups.end()) {
      groups.emplace_back();
      g = groups.end() - 1;
      g->graph = r.graph;
      g->approach = r.approach;
      g->spec = r.spec;
    }
    g->add(r);
  }
  std::vector<dynpr_report::Row> out;
  out.reserve(groups.size());
  for (const auto& g : groups) out.push_back(g.row());
  return out;
}

// Report schema (proj/README.md:89-115; writers harness.cpp:241-352): nine
// columns, floats as %.17g, a NaN error as an empty CSV field / JSON null.
// Each row is first turned into its nine (name, text, quoted) cells; the CSV
// and JSON writers only differ in how they join them.
struct Cell {
  const char* name;
  std::string text;
  bool quoted;  // JSON string value
};

std::string g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::vector<Cell> cells_of(const dynpr_report::Row& r) {
  return {{"graphName", r.graph, true},
          {"approach", r.approach, true},
          {"batchSizeSpec", r.spec, true},
          {"batchIndex", std::to_string(r.batch_index), false},
          {"runtimeMillis", g17(r.runtime), false},
          {"iterations", std::to_string(r.iterations), false},
          {"affectedVertexIterations", std::to_string(r.affected), false},
          {"l1ErrorVsReference", std::isnan(r.l1) ? std::string() : g17(r.l1), false},
          {"converged", r.converged ? "true" : "false", false}};
}

std::string json_quote(const std::string& s) {
  std::string q = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') q += '\\';
    q += c;
  }
  return q + '"';
}

std::string render(const std::vector<dynpr_report::Row>& rows, int32_t format) {
  const bool csv = format == DYNPR_REPORT_CSV;
  std::string out;
  if (csv) {
    const dynpr_report::Row header_row{};
    const auto header = cells_of(header_row);
    for (size_t i = 0; i < header.size(); ++i) out += std::string(i ? "," : "") + header[i].name;
    out += '\n';
  } else {
    out += "[\n";
  }
  for (size_t k = 0; k < rows.size(); ++k) {
    const auto cells = cells_of(rows[k]);
    if (!csv) out += "  {";
    for (size_t i = 0; i < cells.size(); ++i) {
      if (i) out += ',';
      if (csv) {
        out += cells[i].text;
      } else {
        out += json_quote(cells[i].name) + ':';
        out += cells[i].quoted ? json_quote(cells[i].text) : (cells[i].text.empty() ? "null" : cells[i].text);
      }
    }
    out += csv ? "\n" : (k + 1 < rows.size() ? "},\n" : "}\n");
  }
  if (!csv) out += "]\n";
  return out;
}

}  // namespace
}  // namespace dynpr_b200

using namespace dynpr_b200;

extern "C" {

dynpr_status dynpr_load_matrix_market(const char* path, dynpr_edge_list** out) {
  return api_guard([&] {
    if (!path || !out) invalid("null argument");
    *out = load_matrix_market(path);
  });
}

dynpr_status dynpr_load_temporal_edge_list(const char* path, dynpr_edge_list** out) {
  return api_guard([&] {
    if (!path || !out) invalid("null argument");
    *out = load_temporal(path);
  });
}

dynpr_status dynpr_split_temporal(const dynpr_edge_list* stream, double base_fraction, int32_t batch_count,
                                  uint64_t batch_size, dynpr_edge_list** base, uint64_t* base_count) {
  return api_guard([&] {
    if (!stream || !base || !base_count) invalid("null argument");
    const uint64_t bc = split_base_count(stream, base_fraction, batch_count, batch_size);
    *base = split_base(stream, bc);
    *base_count = bc;
  });
}

dynpr_status dynpr_edge_list_info(const dynpr_edge_list* e, uint32_t* vertex_count, uint64_t* count,
                                  int* has_timestamps) {
  return api_guard([&] {
    if (!e) invalid("null edge list");
    if (vertex_count) *vertex_count = e->n;
    if (count) *count = e->src.size();
    if (has_timestamps) *has_timestamps = e->temporal ? 1 : 0;
  });
}

dynpr_status dynpr_edge_list_create(uint32_t vertex_count, const uint32_t* src, const uint32_t* dst,
                                    const int64_t* ts, uint64_t count, dynpr_edge_list** out) {
  return api_guard([&] {
    if (!out) invalid("null argument");
    if (count && (!src || !dst)) invalid("null array argument");
    auto e = std::make_unique<dynpr_edge_list>();
    e->n = vertex_count;
    e->src.assign(src, src + count);
    e->dst.assign(dst, dst + count);
    if (ts) {
      e->ts.assign(ts, ts + count);
      e->temporal = true;
    }
    *out = e.release();
  });
}

dynpr_status dynpr_edge_list_copy(const dynpr_edge_list* e, uint64_t first, uint64_t count, uint32_t* src,
                                  uint32_t* dst, int64_t* ts) {
  return api_guard([&] {
    if (!e) invalid("null edge list");
    if (first > e->src.size() || count > e->src.size() - first) invalid("edge list range out of bounds");
    if (count && (!src || !dst)) invalid("null output array");
    std::memcpy(src, e->src.data() + first, count * sizeof(uint32_t));
    std::memcpy(dst, e->dst.data() + first, count * sizeof(uint32_t));
    if (ts && count) {
      if (!e->temporal) invalid("edge list has no timestamps");
      std::memcpy(ts, e->ts.data() + first, count * sizeof(int64_t));
    }
  });
}

dynpr_status dynpr_edge_list_destroy(dynpr_edge_list* e) {
  delete e;
  return DYNPR_OK;
}

dynpr_status dynpr_compute_reference_ranks(dynpr_context* ctx, const dynpr_graph* gT, const dynpr_graph* gF,
                                           const dynpr_config* cfg, double* ranks_out) {
  NvtxRange nvtx__("dynpr_compute_reference_ranks");
  return api_guard([&] {
    if (!cfg) invalid("null config");
    dynpr_config c = *cfg;  // harness.cpp:340-349
    c.convergence_check_disabled = 1;
    ck(dynpr_static_pagerank(ctx, gT, gF, &c, ranks_out, nullptr, nullptr, nullptr));
  });
}

void dynpr_experiment_spec_default(dynpr_experiment_spec* s) {
  if (!s) return;
  std::memset(s, 0, sizeof *s);
  s->mode = DYNPR_MODE_STATIC;
  s->seed = 1;
  s->repetitions = 1;
  s->base_fraction = 0.9;
  s->batch_count = 100;
  s->insert_fraction = 0.8;
  s->chain_mode = DYNPR_CHAIN_PER_APPROACH;
  s->record_timing = 1;
  dynpr_config_default(&s->config);
}

// harness.cpp:351-381 runExperiment
dynpr_status dynpr_run_experiment(dynpr_context* ctx, const dynpr_experiment_spec* spec, dynpr_report** out) {
  NvtxRange nvtx__("dynpr_run_experiment");
  return api_guard([&] {
    if (!ctx || !spec || !out) invalid("null argument");
    ck(dynpr_config_validate(&spec->config));
    const std::string path = spec->graph_path ? spec->graph_path : "";
    const std::string name =
        spec->graph_name && spec->graph_name[0] ? std::string(spec->graph_name) : file_stem(path);
    if (spec->n_approaches < 1 || !spec->approaches) invalid("runExperiment: no approaches requested");
    for (int i = 0; i < spec->n_approaches; ++i) approach_name(spec->approaches[i]);
    if (spec->mode != DYNPR_MODE_STATIC && (spec->n_batch_size_specs < 1 || !spec->batch_size_specs))
      invalid("runExperiment: no batch sizes requested");
    if (spec->repetitions < 1) invalid("runExperiment: repetitions must be >= 1");
    if (spec->mode != DYNPR_MODE_STATIC && spec->mode != DYNPR_MODE_TEMPORAL && spec->mode != DYNPR_MODE_RANDOM)
      invalid("runExperiment: unknown mode");
    bind_device(ctx);
    auto rep = std::make_unique<dynpr_report>();
    Runner r{ctx, *spec, name, rep.get()};
    switch (spec->mode) {
      case DYNPR_MODE_STATIC: r.run_static(); break;
      case DYNPR_MODE_TEMPORAL: r.run_temporal(); break;
      case DYNPR_MODE_RANDOM: r.run_random(); break;
    }
    auto sums = summarize(rep->rows);
    rep->rows.insert(rep->rows.end(), sums.begin(), sums.end());
    *out = rep.release();
  });
}

dynpr_status dynpr_report_create(dynpr_report** out) {
  return api_guard([&] {
    if (!out) invalid("null argument");
    *out = new dynpr_report();
  });
}

dynpr_status dynpr_report_append(dynpr_report* r, const dynpr_experiment_row* row) {
  return api_guard([&] {
    if (!r || !row) invalid("null argument");
    dynpr_report::Row x;
    x.graph = row->graph_name ? row->graph_name : "";
    x.approach = row->approach ? row->approach : "";
    x.spec = row->batch_size_spec ? row->batch_size_spec : "";
    x.batch_index = row->batch_index;
    x.runtime = row->runtime_millis;
    x.iterations = row->iterations;
    x.affected = row->affected_vertex_iterations;
    x.l1 = row->l1_error_vs_reference;
    x.converged = row->converged != 0;
    r->rows.push_back(std::move(x));
  });
}

dynpr_status dynpr_report_size(const dynpr_report* r, uint64_t* rows) {
  return api_guard([&] {
    if (!r || !rows) invalid("null argument");
    *rows = r->rows.size();
  });
}

dynpr_status dynpr_report_row(const dynpr_report* r, uint64_t i, dynpr_experiment_row* out) {
  return api_guard([&] {
    if (!r || !out) invalid("null argument");
    if (i >= r->rows.size()) invalid("report row out of range");
    const auto& x = r->rows[i];
    out->graph_name = x.graph.c_str();
    out->approach = x.approach.c_str();
    out->batch_size_spec = x.spec.c_str();
    out->batch_index = x.batch_index;
    out->runtime_millis = x.runtime;
    out->iterations = x.iterations;
    out->affected_vertex_iterations = x.affected;
    out->l1_error_vs_reference = x.l1;
    out->converged = x.converged ? 1 : 0;
  });
}

dynpr_status dynpr_report_summarize(const dynpr_report* r, dynpr_report** out) {
  return api_guard([&] {
    if (!r || !out) invalid("null argument");
    auto s = std::make_unique<dynpr_report>();
    s->rows = summarize(r->rows);
    *out = s.release();
  });
}

// harness.cpp:380-396 emitReport
dynpr_status dynpr_report_emit(const dynpr_report* r, int32_t format, const char* path) {
  return api_guard([&] {
    if (!r || !path) invalid("null argument");
    if (r->rows.empty()) invalid("emitReport: no rows");
    if (format != DYNPR_REPORT_CSV && format != DYNPR_REPORT_JSON) invalid("emitReport: unknown format");
    const std::string text = render(r->rows, format);
    const std::string p = path;
    if (p == "-") {
      std::cout << text;
      std::cout.flush();
      if (!std::cout) throw Error(DYNPR_RUNTIME_ERROR, "emitReport: write failed");
      return;
    }
    std::ofstream f(p);
    if (!f) throw Error(DYNPR_RUNTIME_ERROR, "emitReport: cannot open " + p);
    f << text;
    if (!f) throw Error(DYNPR_RUNTIME_ERROR, "emitReport: write failed");
  });
}

dynpr_status dynpr_report_destroy(dynpr_report* r) {
  delete r;
  return DYNPR_OK;
}

}  // extern "C"
