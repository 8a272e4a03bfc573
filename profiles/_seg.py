import sys; sys.path.insert(0, '/root/repo')
import paper_2404_08299_b200 as dp
g = dp.rmat_graph(8); gt = dp.transpose(g)
print("static", dp.static_pagerank(gt, g).iterations, flush=True)
