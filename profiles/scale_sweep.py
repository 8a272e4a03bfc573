"""Static GTEPS and DF-P speed-up across RMAT scales on one B200 (device
loop, warm solves; median of 3).  Writes gpurun_out/scale_sweep.json."""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp

out = []
for scale in [int(x) for x in sys.argv[1:]] or [16, 18, 20, 22, 24, 26]:
    g0 = dp.rmat_graph(scale); gt0 = dp.transpose(g0)
    base = dp.static_pagerank(gt0, g0)
    b = dp.generate_random_batch(g0, dp.batch_size_from_fraction(1e-4, g0.edge_count), 0.8, dp.derive_seed(42, 7))
    g, gt = dp.apply_batch_pair(g0, gt0, b)
    dp.prepare(gt, g)
    dp.static_pagerank(gt, g); dp.dynamic_frontier(g, gt, b.deletions, b.insertions, base.ranks, pruning=True)
    s = sorted((dp.static_pagerank(gt, g) for _ in range(3)), key=lambda r: r.device_ms)[1]
    d = sorted((dp.dynamic_frontier(g, gt, b.deletions, b.insertions, base.ranks, pruning=True) for _ in range(3)),
               key=lambda r: r.device_ms)[1]
    row = {"scale": scale, "n": g.vertex_count, "m": g.edge_count, "static_ms": s.device_ms,
           "static_iterations": s.iterations, "static_gteps": g.edge_count * s.iterations / s.device_ms / 1e6,
           "dfp_ms": d.device_ms, "dfp_iterations": d.iterations, "dfp_speedup": s.device_ms / d.device_ms}
    print(json.dumps(row), flush=True)
    out.append(row)
    del g0, gt0, g, gt
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "scale_sweep.json"), "w"), indent=1)
