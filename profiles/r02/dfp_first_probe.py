"""Bench-like steps on RMAT-S (ingest + prepare, Static, DF-P from the base
ranks) with the DF-P solve repeated on the same snapshot: is the first DF-P
solve of a snapshot slower than a warm repeat?
    python profiles/r02/dfp_first_probe.py [scale] [steps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
g0 = dp.rmat_graph(scale); gt0 = dp.transpose(g0); dp.prepare(gt0, g0)
base = dp.static_pagerank(gt0, g0)
size = dp.batch_size_from_fraction(1e-4, g0.edge_count)
for k in range(steps):
    b = dp.generate_random_batch(g0, size, 0.8, dp.derive_seed(42, 1000003 + k))
    g, gt = dp.apply_batch_pair(g0, gt0, b); dp.prepare(gt, g)
    s = dp.static_pagerank(gt, g)
    d = [dp.dynamic_frontier(g, gt, b.deletions, b.insertions, base.ranks, pruning=True) for _ in range(3)]
    print("step %d static %.3f ms (%d it)  dfp %s ms (%d it)" % (
        k, s.device_ms, s.iterations, " / ".join("%.3f" % x.device_ms for x in d), d[0].iterations), flush=True)
