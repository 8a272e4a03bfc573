"""One prepared DF-P solve for a profiler (ncu --nvtx --nvtx-include
"dynpr_dynamic_frontier/"): RMAT-S, frac*|E| batch, solved twice (the
second is the steady-state one).
    python profiles/dfp_once.py [scale] [frac]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-7
g = dp.rmat_graph(scale); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(frac, g.edge_count), 0.8, dp.derive_seed(42, 0))
g2, gt2 = dp.apply_batch_pair(g, gt, b)
dp.prepare(gt2, g2)
for _ in range(2):
    d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
print("dfp", d.iterations, d.device_ms)
