"""Host-side cost of one small DF-P call (RMAT-20, 1e-7 batch): wall clock vs
the engine's device time with host arrays (numpy prev ranks in, numpy ranks
out -- the reference binding's shape) and with device arrays (torch CUDA
tensors for prev and out), plus a cProfile of the host-array call.
    python profiles/host_overhead_probe.py"""
import cProfile
import os
import pstats
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2404_08299_b200 as dp  # noqa: E402

g = dp.rmat_graph(20)
gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
prev_host = np.asarray(base.ranks, np.float64)
prev_dev = torch.from_numpy(prev_host).cuda()
out_dev = torch.empty_like(prev_dev)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(1e-7, g.edge_count), 0.8, 5)
g2, gt2 = dp.apply_batch_pair(g, gt, b)
dp.prepare(gt2, g2)


def run(label, call, reps=20):
    call()
    wall, dev = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = call()
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(r.device_ms)
    print("%-28s wall %.3f ms  device %.3f ms" % (label, statistics.median(wall), statistics.median(dev)), flush=True)


run("host prev, host out", lambda: dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, prev_host, pruning=True))
run("device prev, device out",
    lambda: dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, prev_dev, pruning=True, out=out_dev))
run("device prev, host out", lambda: dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, prev_dev, pruning=True))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, prev_host, pruning=True)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
