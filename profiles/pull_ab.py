"""In-sweep pull A/B (SweepArgs::pull_fused): DF-P device ms with the pull
folded into the next sweep (DYNPR_PULL_FUSED=1, default) vs the separate
pull kernels (=0), same process, same batches, alternated; plus Static on
the same updated graph.
    python profiles/pull_ab.py [scale] [fractions,comma-separated] [reps]"""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
fracs = [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1e-4"])]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
g = dp.rmat_graph(scale); gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
for f in fracs:
    b = dp.generate_random_batch(g, dp.batch_size_from_fraction(f, g.edge_count), 0.8, dp.derive_seed(42, 0))
    g2, gt2 = dp.apply_batch_pair(g, gt, b)
    dp.prepare(gt2, g2)
    st = [dp.static_pagerank(gt2, g2).device_ms for _ in range(3)]
    res = {"1": [], "0": []}
    ref = None
    for _ in range(reps):
        for mode in ("1", "0"):
            os.environ["DYNPR_PULL_FUSED"] = mode
            d = dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True)
            res[mode].append(d.device_ms)
            key = (d.iterations, d.affected_vertex_iterations, d.ranks.tobytes())
            assert ref is None or key == ref, "pull modes differ"
            ref = key
    print("scale %d frac %g: static %.3f ms | DF-P it %d: fused min %.3f med %.3f | separate min %.3f med %.3f | "
          "speedup vs static fused %.2fx separate %.2fx" % (
              scale, f, min(st), d.iterations, min(res["1"]), statistics.median(res["1"]), min(res["0"]),
              statistics.median(res["0"]), min(st) / min(res["1"]), min(st) / min(res["0"])), flush=True)
