"""A/B of DF-P solve time on RMAT-20: the package under _ab_old/ (a previous
build, copied there by hand) vs the working tree, on the same batches
(dfp_probe.py's), fractions 1e-7..1e-3.  One process per (side, fraction),
sides alternated twice; prints the min and median device ms of 8 solves.
    python profiles/ab_dfp.py [scale] [fractions,comma-separated]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, statistics
sys.path.insert(0, sys.argv[1])
import paper_2404_08299_b200 as dp
g = dp.rmat_graph(int(sys.argv[3])); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(float(sys.argv[2]), g.edge_count), 0.8, 5)
g2, gt2 = dp.apply_batch_pair(g, gt, b)
dp.prepare(gt2, g2)
ms = []
for _ in range(9):
    d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
    ms.append(d.device_ms)
ms = ms[1:]
print("%.3f %.3f it %d  %s" % (min(ms), statistics.median(ms), d.iterations, dp.__file__))
'''
scale = sys.argv[1] if len(sys.argv) > 1 else "20"
fracs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["1e-7", "1e-6", "1e-5", "1e-4", "1e-3"]
for f in fracs:
    for side in ("old", "new", "old", "new"):
        path = os.path.join(ROOT, "_ab_old") if side == "old" else ROOT
        out = subprocess.run([sys.executable, "-c", CHILD, path, f, scale], capture_output=True, text=True, cwd="/tmp")
        print(f, side, out.stdout.strip() or out.stderr[-300:], flush=True)
