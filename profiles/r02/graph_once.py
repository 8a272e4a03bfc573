"""One full device-loop Static solve and one DF-P solve (1e-4 batch) on a
prepared RMAT-S pair, for `ncu --graph-profiling graph`: the whole loop graph
(split kernels running concurrently, loop bookkeeping, expansions) is one
profiled workload, so its request-pipe metrics describe the shipped
execution rather than serialised single kernels.
    python profiles/r02/graph_once.py [scale]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(1e-4, g.edge_count), 0.8, 11)
g2, gt2 = dp.apply_batch_pair(g, gt, b); dp.prepare(gt2, g2)
r = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
print("static", base.iterations, "%.3f ms" % base.device_ms, "dfp", r.iterations, "%.3f ms" % r.device_ms)
