"""Batch-ingest timing (apply_batch_pair + engine layout) on RMAT-S, 1e-4|E|
batches into a prepared base pair (so the new layout is derived
incrementally, layout.cu build_incremental), and the same with the base
unprepared (layout built from scratch)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROOT = os.environ.get("DYNPR_PKG_ROOT", ROOT)  # (A/B: another build of the package)
sys.path.insert(0, ROOT)
import torch
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
g = dp.rmat_graph(scale); gt = dp.transpose(g)
for base_prepared in (False, True):
    if base_prepared:
        dp.prepare(gt, g)
    for k in range(reps):
        b = dp.generate_random_batch(g, dp.batch_size_from_fraction(1e-4, g.edge_count), 0.8, dp.derive_seed(42, k))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g2, gt2 = dp.apply_batch_pair(g, gt, b)
        t1 = time.perf_counter()
        lay = dp.prepare(gt2, g2)
        t2 = time.perf_counter()
        print("base prepared %d: apply_pair %.2f ms, prepare %.2f ms (layout device %.2f ms, generation %d)" % (
            base_prepared, (t1 - t0) * 1e3, (t2 - t1) * 1e3, lay, dp.layout_info(gt2)["generation"]))
        del g2, gt2
