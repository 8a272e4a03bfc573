"""Split-sweep co-residency A/B: Static device ms (device loop) on RMAT-S with
the persistent grids of k_sweep_mseg / k_sweep_single capped to a number of
blocks per SM (DYNPR_MSEG_BPS / DYNPR_SINGLE_BPS; "-" = occupancy default),
so the two concurrently launched kernels can share every SM instead of the
first one filling the GPU.  Combos alternated; results must be identical.
    python profiles/grid_ab.py scale mseg:single[,mseg:single...]"""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_08299_b200 as dp

arg = sys.argv[1]  # S (RMAT) or kS (Kronecker)
scale = int(arg.lstrip("k"))
combos = [c.split(":") for c in sys.argv[2].split(",")]
g = dp.kronecker_graph(scale) if arg.startswith("k") else dp.rmat_graph(scale)
gt = dp.transpose(g); dp.prepare(gt, g)
res = {tuple(c): [] for c in combos}
ref = None
for rep in range(4):
    for c in combos:
        for var, v in zip(("DYNPR_MSEG_BPS", "DYNPR_SINGLE_BPS"), c):
            if v == "-":
                os.environ.pop(var, None)
            else:
                os.environ[var] = v
        r = dp.static_pagerank(gt, g)
        if rep:
            res[tuple(c)].append(r.device_ms)
        key = r.ranks.tobytes()
        assert ref is None or key == ref
        ref = key
for c, v in res.items():
    print("%s mseg %s single %s: min %.3f med %.3f ms" % (arg, c[0], c[1], min(v), statistics.median(v)),
          flush=True)
