// dynpr_bench -- the reference's benchmark CLI surface (tools/dynpr_bench.cpp:
// subcommands static | temporal | random and their flags), parsed by hand
// instead of CLI11 (absent in this image), driving the reference API that
// libdynpr_compat.so implements on the B200.  It exists so the reference's
// unmodified acceptance suite (criteria 9 and 10 shell out to this binary,
// acceptance.cpp:367-375) runs end to end against the GPU engines.
#include <cstdlib>
#include <exception>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "dynpr/harness.hpp"

namespace {

using namespace dynpr;

std::vector<std::string> split_list(const std::string& s) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

int usage(const char* msg) {
  std::cerr << "dynpr_bench: " << msg << "\n"
            << "usage: dynpr_bench static|temporal|random --graph PATH [--batch-sizes F,..] [--approaches A,..]\n"
               "       [--seed N] [--reps N] [--threads N] [--partition-strategy none|transpose|both]\n"
               "       [--dp-threshold N] [--alpha X] [--tol X] [--frontier-tol X] [--prune-tol X]\n"
               "       [--max-iters N] [--out PATH] [--format csv|json] [--no-timing]\n"
               "       temporal: [--batch-count N] [--base-fraction X] [--chain-mode per-approach|shared-reference]\n"
               "       random:   [--insert-fraction X]\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage("a subcommand is required");
  const std::string cmd = argv[1];
  ExperimentSpec spec;
  if (cmd == "static")
    spec.mode = ExperimentMode::Static;
  else if (cmd == "temporal")
    spec.mode = ExperimentMode::Temporal;
  else if (cmd == "random")
    spec.mode = ExperimentMode::RandomBatch;
  else
    return usage(("unknown subcommand '" + cmd + "'").c_str());

  std::map<std::string, std::string> opt{{"--approaches", "static,nd,dt,df,dfp"},
                                         {"--out", "-"},
                                         {"--format", "csv"},
                                         {"--partition-strategy", "both"},
                                         {"--chain-mode", "per-approach"}};
  bool no_timing = false;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--no-timing") {
      no_timing = true;
      continue;
    }
    if (a.rfind("--", 0) != 0 || i + 1 >= argc) return usage(("bad argument '" + a + "'").c_str());
    opt[a] = argv[++i];
  }
  if (!opt.count("--graph")) return usage("--graph is required");
  if (spec.mode != ExperimentMode::Static && !opt.count("--batch-sizes")) return usage("--batch-sizes is required");

  try {
    auto& cfg = spec.config;
    for (const auto& [k, v] : opt) {
      if (k == "--graph") spec.graphPath = v;
      else if (k == "--batch-sizes") spec.batchSizeSpecs = split_list(v);
      else if (k == "--seed") spec.seed = std::stoull(v);
      else if (k == "--reps") spec.repetitions = std::stoi(v);
      else if (k == "--threads") spec.threads = std::stoi(v);
      else if (k == "--dp-threshold") cfg.lowDegreeThreshold = static_cast<uint32_t>(std::stoul(v));
      else if (k == "--alpha") cfg.dampingFactor = std::stod(v);
      else if (k == "--tol") cfg.iterationTolerance = std::stod(v);
      else if (k == "--frontier-tol") cfg.frontierTolerance = std::stod(v);
      else if (k == "--prune-tol") cfg.pruneTolerance = std::stod(v);
      else if (k == "--max-iters") cfg.maxIterations = std::stoi(v);
      else if (k == "--batch-count" && spec.mode == ExperimentMode::Temporal) spec.batchCount = std::stoi(v);
      else if (k == "--base-fraction" && spec.mode == ExperimentMode::Temporal) spec.baseFraction = std::stod(v);
      else if (k == "--insert-fraction" && spec.mode == ExperimentMode::RandomBatch)
        spec.insertFraction = std::stod(v);
      else if (k != "--approaches" && k != "--out" && k != "--format" && k != "--partition-strategy" &&
               k != "--chain-mode")
        return usage(("unknown option '" + k + "'").c_str());
    }
    spec.recordTiming = !no_timing;
    for (const auto& name : split_list(opt["--approaches"])) spec.approaches.push_back(approachFromName(name));
    const std::string& ps = opt["--partition-strategy"];
    if (ps == "none") cfg.partitionStrategy = PartitionStrategy::DontPartition;
    else if (ps == "transpose") cfg.partitionStrategy = PartitionStrategy::PartitionTranspose;
    else if (ps == "both") cfg.partitionStrategy = PartitionStrategy::PartitionBoth;
    else throw std::invalid_argument("unknown partition strategy '" + ps + "'");
    const std::string& cm = opt["--chain-mode"];
    if (cm == "per-approach") spec.chainMode = ChainMode::PerApproach;
    else if (cm == "shared-reference") spec.chainMode = ChainMode::SharedReference;
    else throw std::invalid_argument("unknown chain mode '" + cm + "'");
    const std::string& f = opt["--format"];
    ReportFormat format;
    if (f == "csv") format = ReportFormat::Csv;
    else if (f == "json") format = ReportFormat::Json;
    else throw std::invalid_argument("unknown report format '" + f + "'");
    const auto rows = runExperiment(spec);
    emitReport(rows, format, opt["--out"]);
    return 0;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
