"""Profiling driver (run under ncu on the GPU box; never a bench number).

    python profiles/prof_driver.py --scale 24 [--dfp]

Builds the RMAT graph pair on the device, runs one Static solve and (with
--dfp) one DF-P solve on a 1e-4|E| batch, printing the engine's own timings.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2404_08299_b200 as dp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--dfp", action="store_true")
    ap.add_argument("--static-iters", type=int, default=0)
    ap.add_argument("--frac", type=float, default=1e-4)
    a = ap.parse_args()
    g = dp.rmat_graph(a.scale)
    gt = dp.transpose(g)
    cfg = dp.EngineConfig(max_iterations=a.static_iters, convergence_check_disabled=True) \
        if a.static_iters else dp.EngineConfig()
    dp.prepare(gt, g)
    base = dp.static_pagerank(gt, g, cfg)  # warms the workspace
    ctx = dp.default_context()
    ctx.set_profiling(True)
    base = dp.static_pagerank(gt, g, cfg)
    ms, sweeps, nbytes = ctx.sweep_times()
    ctx.set_profiling(False)
    print(f"static: {base.iterations} it, {base.device_ms:.3f} ms; sweep {ms / max(sweeps, 1):.3f} ms, "
          f"{nbytes / max(sweeps, 1) / (ms / max(sweeps, 1)) / 1e6:.0f} GB/s algorithmic")
    if a.dfp:
        b = dp.generate_random_batch(g, dp.batch_size_from_fraction(a.frac, g.edge_count), 0.8, 7)
        g2, gt2 = dp.apply_batch_pair(g, gt, b)
        r = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
        print(f"dfp: {r.iterations} it, {r.affected_vertex_iterations} affected, {r.device_ms:.3f} ms")


if __name__ == "__main__":
    main()
