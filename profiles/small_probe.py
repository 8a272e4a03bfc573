import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1])
g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
cfg = dp.EngineConfig(max_iterations=3, convergence_check_disabled=True)
dp.static_pagerank(gt, g, cfg)
