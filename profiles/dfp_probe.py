"""DF-P small-batch timeline probe (RMAT-20, 1e-7|E| batch): run under ncu
--metrics gpu__time_duration.sum to list the kernels of one DF-P call."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
frac = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-7
scale = int(os.environ.get("SCALE", "20"))
g = dp.rmat_graph(scale); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(frac, g.edge_count), 0.8, 5)
g2, gt2 = dp.apply_batch_pair(g, gt, b)
dp.prepare(gt2, g2)
if os.environ.get("HOSTLOOP_DFP"):
    os.environ["DYNPR_HOST_LOOP"] = "1"
for _ in range(int(os.environ.get("REPS", "3"))):
    t0 = time.perf_counter()
    d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
    print("dfp device_ms %.3f wall_ms %.3f it %d affected %d" % (d.device_ms, (time.perf_counter() - t0) * 1e3,
                                                              d.iterations, d.affected_vertex_iterations))
