"""Static device ms on small RMAT graphs: the package under _ab_old/ (a
previous build) vs the working tree, alternating processes."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import sys, statistics
sys.path.insert(0, sys.argv[1])
import paper_2404_08299_b200 as dp
g = dp.rmat_graph(int(sys.argv[2])); gt = dp.transpose(g); dp.prepare(gt, g)
ms = [dp.static_pagerank(gt, g).device_ms for _ in range(8)][1:]
print("%.3f %.3f" % (min(ms), statistics.median(ms)))
'''
for scale in sys.argv[1:] or ["18", "20"]:
    for side in ("old", "new", "old", "new"):
        path = os.path.join(ROOT, "_ab_old") if side == "old" else ROOT
        out = subprocess.run([sys.executable, "-c", CHILD, path, scale], capture_output=True, text=True, cwd="/tmp")
        print(scale, side, out.stdout.strip() or out.stderr[-300:], flush=True)
