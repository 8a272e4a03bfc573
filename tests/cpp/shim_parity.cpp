// C++ drop-in parity check: the reference's own types and engines
// (dynpr::CsrGraph, dynpr::staticPageRank, dynpr::dynamicFrontier) against
// the same calls routed through include/dynpr_b200.hpp onto the B200
// engine.  Built by oracle/Makefile (it needs the reference headers and
// library) into oracle/_ref/shim_parity; run by tests/test_gpu_cpp.py.
// Prints one line per check and exits non-zero on any mismatch.
#include <cstdio>
#include <cstdlib>
#include <span>
#include <vector>

#include <fstream>
#include <sstream>
#include <string>

#include "dynpr/engine.hpp"
#include "dynpr/graph.hpp"
#include "dynpr/harness.hpp"
#include "dynpr/partition.hpp"
#include "dynpr/rng.hpp"
#include "dynpr/workload.hpp"
#include "dynpr_b200.hpp"
#include "oracles.hpp"

using namespace dynpr;

static int failures = 0;
static void expect(bool ok, const char* what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what);
  if (!ok) ++failures;
}

int main() {
  SplitMix64 rng(2024);
  const CsrGraph g = oracles::randomGraph(rng, 20000, 200000);
  const CsrGraph gt = transpose(g);
  EngineConfig cfg;

  // staticPageRank(gT, gF, cfg) with the reference signature
  const RankResult ref = staticPageRank(gt, g, cfg);
  const RankResult dev = dynpr_b200::staticPageRank<RankResult>(gt, g, cfg);
  expect(ref.iterations == dev.iterations, "static: iterations equal");
  expect(ref.ranks == dev.ranks, "static: ranks bitwise equal");
  expect(ref.converged == dev.converged && ref.finalDelta == dev.finalDelta, "static: converged/finalDelta");

  // observer semantics (engine.hpp:24-27)
  int seen = 0;
  dynpr_b200::staticPageRank<RankResult>(gt, g, cfg, [&](int it, std::span<const double> r) {
    seen = it;
    (void)r;
  });
  expect(seen == ref.iterations, "static: observer called per iteration");

  // device-side graph construction equals the reference's bytes
  EdgeList raw;
  for (uint32_t u = 0; u < g.vertexCount(); ++u)
    for (Vertex v : g.out(u)) raw.emplace_back(u, v);
  const auto dg = dynpr_b200::addSelfLoops(dynpr_b200::buildCsr(raw, g.vertexCount()));
  expect(dg.download<CsrGraph>() == g, "buildCsr+addSelfLoops: CSR bytes equal");
  expect(dynpr_b200::transpose(dg).download<CsrGraph>() == gt, "transpose: CSR bytes equal");

  // DF-P on a random 80/20 batch
  const BatchUpdate batch = generateRandomBatch(g, 200, 0.8, 7);
  BatchApplyStats st1, st2;
  const CsrGraph g2 = applyBatch(g, batch, &st1);
  const CsrGraph gt2 = transpose(g2);
  const auto dg2 = dynpr_b200::applyBatch(dg, batch, &st2);
  expect(dg2.download<CsrGraph>() == g2, "applyBatch: CSR bytes equal");
  expect(st1.missingDeletions == st2.missingDeletions && st1.duplicateInsertions == st2.duplicateInsertions,
         "applyBatch: stats equal");
  for (bool pruning : {false, true}) {
    const RankResult r1 = dynamicFrontier(g2, gt2, batch.deletions, batch.insertions, ref.ranks, cfg, pruning);
    const RankResult r2 = dynpr_b200::dynamicFrontier<RankResult>(g2, gt2, batch.deletions, batch.insertions,
                                                                 std::span<const double>(ref.ranks), cfg, pruning);
    expect(r1.iterations == r2.iterations && r1.affectedVertexIterations == r2.affectedVertexIterations,
           pruning ? "DF-P: iterations / work equal" : "DF: iterations / work equal");
    expect(r1.ranks == r2.ranks, pruning ? "DF-P: ranks bitwise equal" : "DF: ranks bitwise equal");
  }

  // partitionByDegree
  const DegreePartition p1 = partitionByDegree(gt, 32);
  const DegreePartition p2 = dynpr_b200::partitionByDegree<DegreePartition>(dynpr_b200::transpose(dg), 32);
  expect(p1.order == p2.order && p1.lowCount == p2.lowCount, "partitionByDegree: bit-exact");

  // exceptions keep the reference's types and texts
  try {
    EngineConfig bad;
    bad.dampingFactor = 1.5;
    dynpr_b200::staticPageRank<RankResult>(gt, g, bad);
    expect(false, "invalid config throws std::invalid_argument");
  } catch (const std::invalid_argument& e) {
    expect(std::string(e.what()) == "EngineConfig: dampingFactor must be in (0,1)",
           "invalid config throws std::invalid_argument with the reference text");
  }
  // harness: the reference's runExperiment + emitReport vs the same spec
  // through the shim (device engines) -- report bytes (criterion 9 shape)
  {
    const std::string stream = "/tmp/dynpr_shim_stream.txt";
    {
      std::ofstream f(stream);
      f << "# synthetic temporal stream\n";
      SplitMix64 r(99);
      for (int i = 0; i < 4000; ++i)
        f << r.bounded(600) * 7 << ' ' << r.bounded(600) * 7 << ' ' << (1000 + i / 3) << '\n';
    }
    ExperimentSpec spec;
    spec.graphPath = stream;
    spec.mode = ExperimentMode::Temporal;
    spec.batchSizeSpecs = {"1e-3"};
    spec.approaches = {Approach::Static, Approach::NaiveDynamic, Approach::DynamicTraversal,
                       Approach::DynamicFrontier, Approach::DynamicFrontierPrune};
    spec.batchCount = 50;
    spec.recordTiming = false;
    const auto want = runExperiment(spec);
    emitReport(want, ReportFormat::Csv, "/tmp/dynpr_shim_ref.csv");
    const auto got = dynpr_b200::runExperiment<ExperimentRow>(spec);
    dynpr_b200::emitReport(got, 0, "/tmp/dynpr_shim_dev.csv");
    auto slurp = [](const char* p) {
      std::ifstream f(p);
      std::stringstream ss;
      ss << f.rdbuf();
      return ss.str();
    };
    const std::string a = slurp("/tmp/dynpr_shim_ref.csv"), b = slurp("/tmp/dynpr_shim_dev.csv");
    expect(!a.empty() && a == b, "runExperiment (temporal, 5 approaches): report bytes identical");
    expect(want.size() == got.size() && want.size() == 255, "runExperiment: 250 rows + 5 summaries");
    // computeReferenceRanks on the device, bitwise
    const auto r1 = computeReferenceRanks(gt, g, cfg);
    const auto r2 = dynpr_b200::computeReferenceRanks(gt, g, cfg);
    expect(r1 == r2, "computeReferenceRanks: bitwise equal");
    // loadMatrixMarket
    {
      std::ofstream f("/tmp/dynpr_shim.mtx");
      f << "%%MatrixMarket matrix coordinate real symmetric\n% c\n50 50 120\n";
      SplitMix64 q(5);
      for (int i = 0; i < 120; ++i) f << 1 + q.bounded(50) << ' ' << 1 + q.bounded(50) << " 1.0\n";
    }
    const auto m1 = loadMatrixMarket("/tmp/dynpr_shim.mtx");
    const auto m2 = dynpr_b200::loadMatrixMarket<MatrixMarketGraph>("/tmp/dynpr_shim.mtx");
    expect(m1.edges == m2.edges && m1.vertexCount == m2.vertexCount, "loadMatrixMarket: edges equal");
    try {
      ExperimentSpec bad = spec;
      bad.batchSizeSpecs = {"1e-1"};
      dynpr_b200::runExperiment<ExperimentRow>(bad);
      expect(false, "sizing error raised");
    } catch (const dynpr_b200::SizingError& e) {
      expect(std::string(e.what()).rfind("splitTemporal: stream has 4000 entries", 0) == 0,
             "runExperiment: SizingError with the reference text");
    }
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
