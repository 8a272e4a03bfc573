"""Static vs DF-P sweeps on RMAT-24 under ncu: one host-loop Static solve
(3 sweeps) and one host-loop DF-P solve on the bench workload's first batch,
so the per-kernel metrics of the two sweep kinds can be compared.
    DYNPR_HOST_LOOP=1 ncu --kernel-name regex:k_sweep --metrics ... python profiles/sweep_compare_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp  # noqa: E402

g0 = dp.rmat_graph(24)
gt0 = dp.transpose(g0)
base = dp.static_pagerank(gt0, g0, dp.EngineConfig(max_iterations=60, convergence_check_disabled=True))
b = dp.generate_random_batch(g0, dp.batch_size_from_fraction(1e-4, g0.edge_count), 0.8, dp.derive_seed(42, 1000003))
g, gt = dp.apply_batch_pair(g0, gt0, b)
dp.prepare(gt, g)
print("MARK static")
s = dp.static_pagerank(gt, g, dp.EngineConfig(max_iterations=3, convergence_check_disabled=True))
print("MARK dfp")
d = dp.dynamic_frontier(g, gt, b.deletions, b.insertions, base.ranks, pruning=True)
print("dfp iterations", d.iterations, "edges", d.processed_edges, "static edges/sweep", g.edge_count)
