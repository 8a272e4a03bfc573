"""DF-P fixed per-solve cost on RMAT-20 (BASELINE configs[1]): for each batch
fraction, a fresh batch is ingested and prepared, then DF-P is solved
`reps` times; prints every call's device ms (dynpr_stats.device_ms: the
engine's own events) and host wall ms, with host numpy arrays and with
device-resident tensors (prev / out on the GPU), plus Static on the same
graph for the ratio.
    python profiles/dfp_fixed_probe.py [scale] [fractions] [reps]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2404_08299_b200 as dp

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
fracs = [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1e-7", "1e-6", "1e-5", "1e-4", "1e-3"])]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = dp.rmat_graph(scale); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
prev_dev = torch.from_numpy(base.ranks).cuda()
for k, f in enumerate(fracs):
    b = dp.generate_random_batch(g, dp.batch_size_from_fraction(f, g.edge_count), 0.8, dp.derive_seed(42, k))
    g2, gt2 = dp.apply_batch_pair(g, gt, b)
    dp.prepare(gt2, g2)
    out = torch.empty_like(prev_dev)
    for kind in ("host", "device"):
        dev, wall = [], []
        for r in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if kind == "host":
                d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
            else:
                d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, prev_dev, pruning=True, out=out)
            wall.append((time.perf_counter() - t0) * 1e3)
            dev.append(d.device_ms)
        print("frac %g %-6s it %2d device ms %s | wall ms %s" % (
            f, kind, d.iterations, " ".join("%.3f" % x for x in dev), " ".join("%.3f" % x for x in wall)), flush=True)
    st = [dp.static_pagerank(gt2, g2).device_ms for _ in range(3)]
    print("frac %g static device ms %s" % (f, " ".join("%.3f" % x for x in st)), flush=True)
