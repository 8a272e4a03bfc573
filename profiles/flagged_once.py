"""One host-loop DF solve with every vertex affected (for ncu: the flagged
single-slice kernel on RMAT-S)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
n = g.vertex_count
base = dp.static_pagerank(gt, g, dp.EngineConfig(max_iterations=3, convergence_check_disabled=True))
cfg = dp.EngineConfig(max_iterations=3, convergence_check_disabled=True)
dp.dynamic_frontier_from_flags(g, gt, np.ones(n, np.uint8), np.zeros(n, np.uint8), base.ranks, cfg, False)
