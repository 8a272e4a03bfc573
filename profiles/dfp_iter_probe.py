"""Per-iteration timeline of device-loop solves (dynpr_debug_loop_trace):
for Static and DF-P on RMAT-S with a frac*|E| batch, each iteration's
duration (difference of the globaltimer stamps k_loop_end writes; the first
iteration is measured from a marker solve-start event), gathered edges,
processed vertices, pending out-edges and the expansion decided after it.
    python profiles/dfp_iter_probe.py [scale] [frac]"""
import ctypes as C
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROOT = os.environ.get("DYNPR_PKG_ROOT", ROOT)  # (A/B: another build of the package)
sys.path.insert(0, ROOT)
import numpy as np
import paper_2404_08299_b200 as dp
from paper_2404_08299_b200 import _native as N

arg = sys.argv[1] if len(sys.argv) > 1 else "24"
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
if len(sys.argv) > 3:
    os.environ["DYNPR_SWEEP"] = sys.argv[3]  # split | fused
if arg.startswith("u"):  # uniform random graph (configs[4]'s kind): 2^S vertices, 16 x 2^S pairs + self-loops
    scale = int(arg[1:])
    rng = np.random.default_rng(1)
    nv = 1 << scale
    src = rng.integers(0, nv, 16 * nv, dtype=np.uint32)
    dst = rng.integers(0, nv, 16 * nv, dtype=np.uint32)
    g = dp.add_self_loops(dp.build_csr((src, dst), nv))
else:
    scale = int(arg)
    g = dp.rmat_graph(scale)
gt = dp.transpose(g)
base = dp.static_pagerank(gt, g)
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(frac, g.edge_count), 0.8, dp.derive_seed(42, 0))
g2, gt2 = dp.apply_batch_pair(g, gt, b)
dp.prepare(gt2, g2)


def trace(n_it):
    cnt = C.c_uint64()
    N.lib().dynpr_debug_loop_trace(None, 0, C.byref(cnt))
    buf = np.zeros(cnt.value, np.uint64)
    N.lib().dynpr_debug_loop_trace(buf.ctypes.data, cnt.value, None)
    return buf.reshape(-1, 4)[:n_it]


for name, fn in (("static", lambda: dp.static_pagerank(gt2, g2)),
                 ("dfp", lambda: dp.dynamic_frontier(g2, gt2, b.deletions, b.insertions, base.ranks, pruning=True))):
    fn()
    r = fn()
    t = trace(r.iterations)
    dt = np.diff(t[:, 0].astype(np.int64)) / 1e6
    print("%s: %d it, device %.3f ms, sum of iterations 2..%d %.3f ms (first ~%.3f ms incl. init)" % (
        name, r.iterations, r.device_ms, r.iterations, dt.sum(), r.device_ms - dt.sum()))
    for i in range(r.iterations):
        d = dt[i - 1] if i else float("nan")
        w = int(t[i, 3])
        pend = w & ((1 << 62) - 1)
        ex = {0: "-", 1: "push", 2: "pull", 3: "push (lists collected)"}[(w >> 62) & 3]
        print("  it %2d  %7.3f ms  edges %11d (%.2f m)  processed %9d  pending-out %11d  -> %s" % (
            i + 1, d, int(t[i, 1]), int(t[i, 1]) / g2.edge_count, int(t[i, 2]), pend, ex))
