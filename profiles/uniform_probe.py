"""DF-P vs Static on a uniform random graph (the temporal config's graph
class): n = 2^20, 16n pairs, insert-only batches."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2404_08299_b200 as dp
n = 1 << 20
rng = np.random.default_rng(7)
s = rng.integers(0, n, 16 * n, dtype=np.uint32); d = rng.integers(0, n, 16 * n, dtype=np.uint32)
g = dp.add_self_loops(dp.build_csr((s, d), n)); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
for bs in (17, 168, 1678, 16777):
    ins = (rng.integers(0, n, bs, dtype=np.uint32), rng.integers(0, n, bs, dtype=np.uint32))
    b = dp.BatchUpdate(([], []), ins)
    g2, gt2 = dp.apply_batch_pair(g, gt, dp.BatchUpdate(dp.EdgeArray([], []), dp.EdgeArray(*ins)))
    dp.prepare(gt2, g2)
    for _ in range(2):
        st = dp.static_pagerank(gt2, g2)
        df = dp.dynamic_frontier(g2, gt2, dp.EdgeArray([], []), dp.EdgeArray(*ins), base.ranks, pruning=True)
    print("batch %6d: static %.3f ms (%d it)  dfp %.3f ms (%d it, %d affected, %.1f%% of n*it)" % (
        bs, st.device_ms, st.iterations, df.device_ms, df.iterations, df.affected_vertex_iterations,
        100.0 * df.affected_vertex_iterations / (n * df.iterations)), flush=True)
