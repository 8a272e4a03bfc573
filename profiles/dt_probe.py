"""DT (dynamicTraversal) vs DF-P on RMAT-20, 1e-4 batch: device ms."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
g = dp.rmat_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 20); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(1e-4, g.edge_count), 0.8, 3)
g2, gt2 = dp.apply_batch_pair(g, gt, b); dp.prepare(gt2, g2)
for _ in range(2):
    t = dp.dynamic_traversal(g2, gt2, b.deletions, b.insertions, base.ranks)
    d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
    nd = dp.naive_dynamic(gt2, g2, base.ranks)
print("dt %.3f ms (%d it, %d aff)  dfp %.3f ms (%d it)  nd %.3f ms (%d it)" % (t.device_ms, t.iterations,
      t.affected_vertex_iterations, d.device_ms, d.iterations, nd.device_ms, nd.iterations))
import time, numpy as np, torch
seeds = np.unique(np.concatenate([b.insertions.src, b.deletions.src, b.deletions.dst]))
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    va = dp.mark_reachable(g2, seeds)
    torch.cuda.synchronize()
print("markReachable %.3f ms, %d reached" % ((time.perf_counter() - t0) * 1e3, int(va.sum())))
