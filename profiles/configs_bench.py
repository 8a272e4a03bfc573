#!/usr/bin/env python
"""BASELINE.json configs sweep (one GPU): every config that is not bench.py's
headline line, each next to the reference CPU library (oracle/_ref, all host
cores) on the same inputs, with a parity check on the compared solves.

    python profiles/configs_bench.py [--configs 0,1,3,4] [--out gpurun_out/configs.json]

  configs[0]  Static, RMAT-18: ms/solve, iterations, GTEPS; reference full
              solve on the same CSR bytes; ranks bitwise compared.
  configs[1]  DF-P on RMAT-20, 80/20 random batches of 1e-7..1e-3 |E| (the
              reference generator), 5 reps per size: DF-P and Static ms/solve
              on the same updated graph; the reference's DF-P + Static for the
              first rep of every size (parity: iterations, ranks bitwise).
  configs[3]  Static + DF-P (1e-4 batch) on Kronecker scale-27 (~2.1 B edges;
              Graph500 initiator with the seeded vertex-id scramble,
              dynpr_graph_kronecker)
              on ONE B200 (the box has one GPU; the partitioned engine is
              exercised by bench.py --gpus N); reference: a bounded sample of
              static sweeps.
  configs[4]  Temporal stream: uniform-random graph (n = 2^20, 16n pairs)
              written as a SNAP `src dst ts` file, run through
              run_experiment(TEMPORAL, 100 insert-only batches, chained) on
              the device: DF-P vs Static per batch (geometric means), plus the
              load/parse time.  The reference harness would need ~100 x 500
              CPU sweeps per spec; its DF-P/Static are timed on batch 0 only.

Timing: device ms are the library's CUDA-event time of each engine call
(dynpr_stats.device_ms); the reference is steady_clock around its call, as in
harness.cpp:133-135.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker + CPU baseline only)
import paper_2404_08299_b200 as dp  # noqa: E402


def ref_lib():
    kind = "ref" if oracle.available("ref") else "port"
    O = oracle.Oracle(kind)
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    return O, ("reference" if kind == "ref" else "port"), (threads if kind == "ref" else 1)


def to_ref(O, g):
    return O.graph_from_csr(g.vertex_count, g.offsets, g.targets)


def timed_ref(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, (time.perf_counter() - t0) * 1e3


def config0(O, kind, cores, reps=5):
    g = dp.rmat_graph(18)
    gt = dp.transpose(g)
    dp.prepare(gt, g, frontier=False)
    res = [dp.static_pagerank(gt, g) for _ in range(reps + 1)][1:]
    ms = statistics.mean(r.device_ms for r in res)
    it = res[0].iterations
    og, ogt = to_ref(O, g), to_ref(O, gt)
    O.static(ogt, og)
    rr, rms = timed_ref(lambda: O.static(ogt, og))
    return {"workload": "configs[0] Static RMAT-18", "n": g.vertex_count, "m": g.edge_count,
            "ours": {"ms_per_solve": ms, "iterations": it, "gteps": g.edge_count * it / (ms * 1e-3) / 1e9},
            "reference": {"ms_per_solve": rms, "iterations": rr.iterations, "kind": kind, "cores": cores,
                          "gteps": g.edge_count * rr.iterations / (rms * 1e-3) / 1e9},
            "speedup": rms / ms,
            "parity": {"iterations_equal": rr.iterations == it,
                       "ranks_bitwise_equal": bool(np.array_equal(rr.ranks, res[0].ranks))}}


def config1(O, kind, cores, reps=5, seed=42):
    g0 = dp.rmat_graph(20, seed=seed)
    gt0 = dp.transpose(g0)
    base = dp.static_pagerank(gt0, g0)
    og0 = to_ref(O, g0)
    rows = []
    for si, frac in enumerate([1e-7, 1e-6, 1e-5, 1e-4, 1e-3]):
        size = dp.batch_size_from_fraction(frac, g0.edge_count)
        st_ms, df_ms, st_it, df_it, aff = [], [], [], [], []
        ref_row = None
        for rep in range(reps):
            b = dp.generate_random_batch(g0, size, 0.8, dp.derive_seed(seed, si * 1000003 + rep))
            g, gt = dp.apply_batch_pair(g0, gt0, b)
            dp.prepare(gt, g)
            s = dp.static_pagerank(gt, g)
            d = dp.dynamic_frontier(g, gt, b.deletions, b.insertions, base.ranks, pruning=True)
            st_ms.append(s.device_ms)
            df_ms.append(d.device_ms)
            st_it.append(s.iterations)
            df_it.append(d.iterations)
            aff.append(d.affected_vertex_iterations)
            if rep == 0:
                og, ogt = to_ref(O, g), to_ref(O, gt)
                rs, rs_ms = timed_ref(lambda: O.static(ogt, og))
                rd, rd_ms = timed_ref(lambda: O.dynamic_frontier(og, ogt, b.deletions, b.insertions, base.ranks,
                                                                 pruning=True))
                ref_row = {"static_ms": rs_ms, "dfp_ms": rd_ms, "dfp_iterations": rd.iterations,
                           "speedup_dfp_vs_static": rs_ms / rd_ms,
                           "parity": {"static_iterations_equal": rs.iterations == s.iterations,
                                      "static_ranks_bitwise_equal": bool(np.array_equal(rs.ranks, s.ranks)),
                                      "dfp_iterations_equal": rd.iterations == d.iterations,
                                      "dfp_affected_equal": rd.affected_vertex_iterations
                                      == d.affected_vertex_iterations,
                                      "dfp_ranks_bitwise_equal": bool(np.array_equal(rd.ranks, d.ranks))},
                           "ours_vs_reference_dfp": rd_ms / d.device_ms}
            del g, gt
        rows.append({"fraction": frac, "batch_size": size,
                     "static_ms": statistics.mean(st_ms), "static_iterations": statistics.mean(st_it),
                     "dfp_ms": statistics.mean(df_ms), "dfp_iterations": statistics.mean(df_it),
                     "dfp_affected_vertex_iterations": statistics.mean(aff),
                     "speedup_dfp_vs_static": statistics.mean(st_ms) / statistics.mean(df_ms),
                     "static_ms_reps": st_ms, "dfp_ms_reps": df_ms,
                     "reference_rep0": ref_row})
    return {"workload": "configs[1] DF-P RMAT-20, 80/20 random batches, %d reps per size" % reps,
            "n": g0.vertex_count, "m": g0.edge_count, "reference_kind": kind, "reference_cores": cores,
            "sizes": rows}


def config3(O, kind, cores, scale=27, seed=42, ref_sweeps=3):
    t0 = time.perf_counter()
    g0 = dp.kronecker_graph(scale, seed=seed)  # Graph500 initiator + id scramble
    gt0 = dp.transpose(g0)
    build_s = time.perf_counter() - t0
    n, m = g0.vertex_count, g0.edge_count
    dp.prepare(gt0, g0)  # the base snapshot of a DF-P stream: layout + relabelled forward rows
    base = dp.static_pagerank(gt0, g0)
    size = dp.batch_size_from_fraction(1e-4, m)
    b = dp.generate_random_batch(g0, size, 0.8, dp.derive_seed(seed, 1000003))
    # the first ingest of a new graph size grows the device memory pool
    # (cudaMallocAsync maps ~35 GB of fresh pages, ~1 s); report it apart
    # from the warm ingest every later batch pays
    t0 = time.perf_counter()
    g, gt = dp.apply_batch_pair(g0, gt0, b)
    lay_cold = dp.prepare(gt, g)
    ingest_cold_ms = (time.perf_counter() - t0) * 1e3
    del g, gt
    t0 = time.perf_counter()
    g, gt = dp.apply_batch_pair(g0, gt0, b)
    lay = dp.prepare(gt, g)
    ingest_ms = (time.perf_counter() - t0) * 1e3
    # warm (first calls on a new graph size allocate workspace / instantiate
    # the loop graph); report the median of 3 warm solves each
    prev_dev = base.ranks
    dp.static_pagerank(gt, g)
    dp.dynamic_frontier(g, gt, b.deletions, b.insertions, prev_dev, pruning=True)
    ss = sorted((dp.static_pagerank(gt, g) for _ in range(3)), key=lambda r: r.device_ms)
    ds = sorted((dp.dynamic_frontier(g, gt, b.deletions, b.insertions, prev_dev, pruning=True) for _ in range(3)),
                key=lambda r: r.device_ms)
    s, d = ss[1], ds[1]
    out = {"workload": "configs[3] Kronecker-%d (Graph500 initiator, scrambled ids) on one B200" % scale,
           "n": n, "m": m,
           "build_s": build_s, "ingest_ms": ingest_ms, "layout_ms": lay,
           "ingest_cold_ms": ingest_cold_ms, "layout_cold_ms": lay_cold,
           "static": {"ms_per_solve": s.device_ms, "iterations": s.iterations,
                      "gteps": m * s.iterations / (s.device_ms * 1e-3) / 1e9},
           "dfp": {"ms_per_solve": d.device_ms, "iterations": d.iterations,
                   "affected_vertex_iterations": d.affected_vertex_iterations,
                   "speedup_vs_static": s.device_ms / d.device_ms}}
    del g0, gt0
    if ref_sweeps:
        og, ogt = to_ref(O, g), to_ref(O, gt)
        cfg = oracle.default_config(max_iterations=ref_sweeps, convergence_check_disabled=1)
        rr, rms = timed_ref(lambda: O.static(ogt, og, cfg))
        mine = dp.static_pagerank(gt, g, dp.EngineConfig(max_iterations=ref_sweeps,
                                                         convergence_check_disabled=True))
        out["reference_sample"] = {"kind": kind, "cores": cores, "sweeps": ref_sweeps, "ms": rms,
                                   "gteps": m * ref_sweeps / (rms * 1e-3) / 1e9,
                                   "ranks_bitwise_equal": bool(np.array_equal(rr.ranks, mine.ranks))}
    return out


def write_uniform_stream(path, n, pairs, seed=7):
    rng = np.random.default_rng(seed)
    with open(path, "w") as f:
        f.write("# uniform random temporal stream, SNAP layout: src dst unixts\n")
        chunk = 1 << 22
        t = 1_000_000_000
        for lo in range(0, pairs, chunk):
            k = min(chunk, pairs - lo)
            s = rng.integers(0, n, k)
            d = rng.integers(0, n, k)
            ts = t + lo + np.arange(k)
            f.write("\n".join(f"{a} {b} {c}" for a, b, c in zip(s.tolist(), d.tolist(), ts.tolist())))
            f.write("\n")


def config4(O, kind, cores, scale=20, specs=("1e-5", "1e-4", "1e-3")):
    n = 1 << scale
    path = os.path.join(tempfile.gettempdir(), "dynpr_uniform_stream.txt")
    write_uniform_stream(path, n, 16 * n)
    t0 = time.perf_counter()
    s, d, ts, nv = dp.load_temporal_edge_list_arrays(path)
    load_s = time.perf_counter() - t0
    size_mb = os.path.getsize(path) / 1e6
    spec = dp.ExperimentSpec(graph_path=path, mode=dp.ExperimentMode.TEMPORAL, batch_size_specs=list(specs),
                             approaches=[dp.Approach.STATIC, dp.Approach.DYNAMIC_FRONTIER_PRUNE], batch_count=100)
    t0 = time.perf_counter()
    rows = dp.run_experiment(spec)
    total_s = time.perf_counter() - t0
    summ = {}
    for r in rows:
        if r.batch_index == -1:
            summ.setdefault(r.batch_size_spec, {})[r.approach] = {
                "geomean_ms": r.runtime_millis, "mean_iterations": r.iterations,
                "mean_affected_vertex_iterations": r.affected_vertex_iterations,
                "geomean_l1_vs_reference": r.l1_error_vs_reference, "all_converged": r.converged}
    for k, v in summ.items():
        v["speedup_dfp_vs_static"] = v["static"]["geomean_ms"] / v["dfp"]["geomean_ms"]
    out = {"workload": "configs[4] temporal stream, uniform random n=2^%d, %d pairs, 100 insert-only batches "
                       "per spec (chained DF-P)" % (scale, 16 * n),
           "file_mb": size_mb, "load_s": load_s, "load_mb_per_s": size_mb / load_s, "vertices": nv,
           "experiment_wall_s": total_s, "per_spec": summ,
           "note": "runtimes are the harness's host wall clock around each device engine call "
                   "(harness.cpp:133-135); each batch also ingests (apply_batch_pair) and computes the "
                   "500-sweep reference ranks on the device"}
    # reference on batch 0 of the first spec only (one CPU Static + DF-P)
    bs = dp.batch_size_from_fraction(float(specs[-1]), len(s))
    (bsrc, bdst), batches = dp.split_temporal(path, 0.9, 1, bs)
    og = O.add_self_loops(O.build_csr((bsrc, bdst), nv))
    ogt = O.transpose(og)
    prev = O.static(ogt, og).ranks
    ins = batches[0]
    og2, _, _ = O.apply_batch(og, [], ins)
    ogt2 = O.transpose(og2)
    rs, rs_ms = timed_ref(lambda: O.static(ogt2, og2))
    rd, rd_ms = timed_ref(lambda: O.dynamic_frontier(og2, ogt2, [], ins, prev, pruning=True))
    out["reference_batch0"] = {"spec": specs[-1], "kind": kind, "cores": cores, "static_ms": rs_ms,
                               "dfp_ms": rd_ms, "speedup_dfp_vs_static": rs_ms / rd_ms}
    os.unlink(path)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,4")
    ap.add_argument("--kron-scale", type=int, default=27)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    args = ap.parse_args()
    O, kind, cores = ref_lib()
    out = {}
    for c in args.configs.split(","):
        t0 = time.perf_counter()
        if c == "0":
            out["configs[0]"] = config0(O, kind, cores)
        elif c == "1":
            out["configs[1]"] = config1(O, kind, cores)
        elif c == "3":
            out["configs[3]"] = config3(O, kind, cores, scale=args.kron_scale)
        elif c == "4":
            out["configs[4]"] = config4(O, kind, cores)
        print(f"config {c} done in {time.perf_counter() - t0:.1f} s", flush=True)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
