"""DF-P device ms (min / median of 6 warm solves, same batch) for several
package builds, one process per (build, graph, fraction), interleaved.
    python profiles/r02/dfp_bisect_ab.py scale:frac[,scale:frac] DIR[:VAR=value] ...
(scale uS: a uniform random graph of 2^S vertices)"""
import os, subprocess, sys
CHILD = r'''
import sys, statistics
sys.path.insert(0, sys.argv[1])
import paper_2404_08299_b200 as dp
if sys.argv[2].startswith("u"):  # uniform: 2^S vertices, 16 x 2^S random pairs + self-loops
    import numpy as np
    S = int(sys.argv[2][1:]); rng = np.random.default_rng(1)
    g = dp.add_self_loops(dp.build_csr((rng.integers(0, 1 << S, 16 << S, dtype=np.uint32),
                                        rng.integers(0, 1 << S, 16 << S, dtype=np.uint32)), 1 << S))
else:
    g = dp.rmat_graph(int(sys.argv[2]))
gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(float(sys.argv[3]), g.edge_count), 0.8, 11)
g2, gt2 = dp.apply_batch_pair(g, gt, b); dp.prepare(gt2, g2)
ms = [dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True).device_ms for _ in range(7)][1:]
print("%.3f %.3f" % (min(ms), statistics.median(ms)))
'''
cases = [c.split(":") for c in sys.argv[1].split(",")]
for scale, frac in cases:
    for rep in range(2):
        for spec in sys.argv[2:]:
            d, _, kv = spec.partition(":")
            env = dict(os.environ)
            for item in filter(None, kv.split("+")):  # VAR=value[+VAR2=value2]
                k, v = item.split("=")
                env[k] = v
            out = subprocess.run([sys.executable, "-c", CHILD, os.path.abspath(d), scale, frac], capture_output=True,
                                 text=True, cwd="/tmp", env=env)
            print(scale, frac, spec, out.stdout.strip() or out.stderr[-300:], flush=True)
