"""Per-iteration overhead probe: engine device time vs summed sweep time
(CUDA events around each sweep) for Static on RMAT-18..24, and per-rep DF-P
times on RMAT-20 batches (1e-5 outlier hunt)."""
import os, sys, json, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp

ctx = dp.default_context()
out = {}
for scale in (18, 20, 22, 24):
    g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
    dp.static_pagerank(gt, g)
    os.environ["DYNPR_HOST_LOOP"] = "1"
    rh = dp.static_pagerank(gt, g)
    os.environ["DYNPR_HOST_LOOP"] = "0"
    rd = dp.static_pagerank(gt, g)
    ctx.set_profiling(True)
    r = dp.static_pagerank(gt, g)
    sw = ctx.sweep_times()
    ctx.set_profiling(False)
    out[scale] = {"device_loop_ms": rd.device_ms, "host_loop_ms": rh.device_ms, "device_ms": r.device_ms, "it": r.iterations, "sweep_ms": sw[0], "sweeps": sw[1],
                  "per_iter_us": 1e3 * r.device_ms / r.iterations, "sweep_us": 1e3 * sw[0] / max(sw[1], 1)}
    print(scale, out[scale], flush=True)
    if scale == 20:
        base = dp.static_pagerank(gt, g)
        for frac in (1e-6, 1e-5, 1e-4):
            size = dp.batch_size_from_fraction(frac, g.edge_count)
            for rep in range(5):
                b = dp.generate_random_batch(g, size, 0.8, dp.derive_seed(42, int(frac * 1e7) * 1000003 + rep))
                g2, gt2 = dp.apply_batch_pair(g, gt, b)
                dp.prepare(gt2, g2)
                ts = []
                for hl in ("1", "0", "1", "0"):
                    os.environ["DYNPR_HOST_LOOP"] = hl
                    d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
                    ts.append(round(d.device_ms, 3))
                print("dfp", frac, rep, ts, d.iterations, d.affected_vertex_iterations, d.processed_edges,
                      "pull", ctx.pull_expansions if hasattr(ctx, "pull_expansions") else None, flush=True)
    del g, gt
