"""First-call cost of a DF-P solve in a fresh process (RMAT-20, 1e-7 batch):
device ms of the first, second and third DF-P calls on three prepared
snapshots, and the same under CUDA_MODULE_LOADING=EAGER (run by the parent
as a second child) -- separates lazy module loading from the loop graph's
first capture + instantiation."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time
sys.path.insert(0, sys.argv[1])
import paper_2404_08299_b200 as dp
g = dp.rmat_graph(20); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
snaps = []
for k in range(3):
    b = dp.generate_random_batch(g, dp.batch_size_from_fraction(1e-7, g.edge_count), 0.8, dp.derive_seed(42, k))
    g2, gt2 = dp.apply_batch_pair(g, gt, b)
    dp.prepare(gt2, g2)
    snaps.append((g2, gt2, b))
out = []
for g2, gt2, b in snaps:
    t0 = time.perf_counter()
    d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
    out.append("%.3f/%.3f" % (d.device_ms, (time.perf_counter() - t0) * 1e3))
print("device/wall ms of DF-P calls 1..3:", " ".join(out))
'''
for eager in (False, True):
    env = dict(os.environ)
    if eager:
        env["CUDA_MODULE_LOADING"] = "EAGER"
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, env=env, cwd="/tmp")
    print("EAGER" if eager else "default", r.stdout.strip() or r.stderr[-400:], flush=True)
