"""Batch-ingest timing (apply_batch_pair + engine layout) on RMAT-S, 1e-4|E| batches."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = dp.rmat_graph(scale); gt = dp.transpose(g)
for k in range(6):
    b = dp.generate_random_batch(g, dp.batch_size_from_fraction(1e-4, g.edge_count), 0.8, dp.derive_seed(42, k))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g2, gt2 = dp.apply_batch_pair(g, gt, b)
    t1 = time.perf_counter()
    lay = dp.prepare(gt2, g2)
    t2 = time.perf_counter()
    print("apply_pair %.2f ms, prepare %.2f ms (layout device %.2f ms)" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, lay))
    del g2, gt2
