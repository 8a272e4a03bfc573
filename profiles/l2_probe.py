"""Experiment: L2 persistence of the hot prefix of the contribution vector
(host loop, per-sweep CUDA events), RMAT-24."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DYNPR_HOST_LOOP"] = "1"
import paper_2404_08299_b200 as dp
ctx = dp.default_context()
g = dp.rmat_graph(int(os.environ.get("SCALE", "24"))); gt = dp.transpose(g); dp.prepare(gt, g)
cfg = dp.EngineConfig(max_iterations=20, convergence_check_disabled=True)
for mb in [None, "16", "32", "48", "64", "96", None]:
    if mb is None:
        os.environ.pop("DYNPR_L2_HOT_MB", None)
    else:
        os.environ["DYNPR_L2_HOT_MB"] = mb
    ts = []
    for rep in range(3):
        ctx.set_profiling(True)
        dp.static_pagerank(gt, g, cfg)
        ms, n, _ = ctx.sweep_times()
        ts.append(1e3 * ms / n)
    print(mb, "%.1f us" % statistics.median(ts), flush=True)
