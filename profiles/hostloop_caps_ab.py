"""Per-sweep time of the host-driven loop (ctx.set_profiling: CUDA events
around each sweep, as bench.py's roofline leg) vs the device loop's
per-iteration time, with and without the split-grid caps
(DYNPR_MSEG_BPS / DYNPR_SINGLE_BPS = 0 disables them)."""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
ctx = dp.default_context()
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
cfg = dp.EngineConfig(max_iterations=20, convergence_check_disabled=True)
for caps in ("default", "off"):
    for k in ("DYNPR_MSEG_BPS", "DYNPR_SINGLE_BPS"):
        if caps == "off":
            os.environ[k] = "0"
        else:
            os.environ.pop(k, None)
    host, dev = [], []
    for rep in range(4):
        ctx.set_profiling(True)
        dp.static_pagerank(gt, g, cfg)
        ms, n, _ = ctx.sweep_times()
        ctx.set_profiling(False)
        r = dp.static_pagerank(gt, g, cfg)
        if rep:
            host.append(1e3 * ms / n)
            dev.append(1e3 * r.device_ms / r.iterations)
    print("caps %s: host-loop sweep %.1f us (events), device loop %.1f us per iteration" % (
        caps, statistics.median(host), statistics.median(dev)), flush=True)
