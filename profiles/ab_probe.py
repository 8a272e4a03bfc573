"""A/B of the split (3-kernel) and fused sweeps in one process: mean sweep
time (CUDA events) of Static solves, alternating, per RMAT scale."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
ctx = dp.default_context()
for scale in [int(x) for x in sys.argv[1:]] or [18, 20, 22, 24]:
    g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
    cfg = dp.EngineConfig(max_iterations=20, convergence_check_disabled=True)
    res = {"split": [], "fused": [], "wide": []}
    for rep in range(6):
        for mode in ("split", "fused", "wide"):
            os.environ["DYNPR_SWEEP"] = mode
            ctx.set_profiling(True)
            dp.static_pagerank(gt, g, cfg)
            ms, n, _ = ctx.sweep_times()
            if rep:
                res[mode].append(1e3 * ms / n)
    print(scale, {k: "%.1f us" % statistics.median(v) for k, v in res.items()}, flush=True)
    del g, gt
