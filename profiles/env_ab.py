"""DF-P device ms under alternative settings of one environment knob read per
solve (e.g. DYNPR_INIT_PULL_DIV, DYNPR_PULL_FUSED), same process, same
batch, settings alternated; results must be bitwise equal.
    python profiles/env_ab.py scale frac reps VAR=v1,v2,..."""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp

arg, frac, reps = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
var, vals = sys.argv[4].split("=")
vals = vals.split(",")
if arg.startswith("u"):  # uniform random graph, 2^S vertices, 16 x 2^S pairs + self-loops
    import numpy as np
    scale = int(arg[1:])
    rng = np.random.default_rng(1)
    src = rng.integers(0, 1 << scale, 16 << scale, dtype=np.uint32)
    dst = rng.integers(0, 1 << scale, 16 << scale, dtype=np.uint32)
    g = dp.add_self_loops(dp.build_csr((src, dst), 1 << scale))
else:
    scale = int(arg)
    g = dp.rmat_graph(scale)
gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(frac, g.edge_count), 0.8, dp.derive_seed(42, 0))
g2, gt2 = dp.apply_batch_pair(g, gt, b)
dp.prepare(gt2, g2)
res = {v: [] for v in vals}
ref = None
for _ in range(reps):
    for v in vals:
        os.environ[var] = v
        d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
        res[v].append(d.device_ms)
        key = (d.iterations, d.affected_vertex_iterations, d.ranks.tobytes())
        assert ref is None or key == ref, "settings differ"
        ref = key
print("scale %d frac %g it %d: " % (scale, frac, d.iterations) + " | ".join(
    "%s=%s min %.3f med %.3f" % (var, v, min(res[v]), statistics.median(res[v])) for v in vals), flush=True)
