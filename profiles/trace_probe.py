"""Per-warp timeline of one fused sweep (DYNPR_TRACE=1): the last sweep of a
3-sweep Static solve, or with a second argument `dfp [fraction]` the last
sweep of a DF-P solve after a random batch of that size.
    python profiles/trace_probe.py SCALE [dfp [1e-7]]"""
import os, sys, ctypes as C
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DYNPR_TRACE"] = "1"
import paper_2404_08299_b200 as dp
from paper_2404_08299_b200 import _native as N
scale = int(sys.argv[1])
g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
if len(sys.argv) > 2 and sys.argv[2] == "dfp":
    frac = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-7
    base = dp.static_pagerank(gt, g)
    b = dp.generate_random_batch(g, dp.batch_size_from_fraction(frac, g.edge_count), 0.8, 5)
    g, gt = dp.apply_batch_pair(g, gt, b)
    dp.prepare(gt, g)
    for _ in range(2):
        d = dp.dynamic_frontier(g, gt, b.deletions, b.insertions, base.ranks, pruning=True)
    print("dfp iterations", d.iterations, "affected", d.affected_vertex_iterations, "device_ms %.3f" % d.device_ms)
else:
    cfg = dp.EngineConfig(max_iterations=3, convergence_check_disabled=True)
    dp.static_pagerank(gt, g, cfg)
cnt = C.c_uint64()
N.lib().dynpr_debug_sweep_trace(None, 0, C.byref(cnt))
buf = np.zeros(cnt.value, np.uint64)
N.lib().dynpr_debug_sweep_trace(buf.ctypes.data, cnt.value, None)
t = buf.reshape(-1, 6).astype(np.int64)
t = t[t[:, 1] > 0]
t0 = t[:, 1].min()
st, en, th = (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 5] - t0) / 1e3
nh, nl = t[:, 3] & 0xffffffff, t[:, 3] >> 32
print("warps", len(t), "kernel span us %.1f" % en.max(), "start spread %.1f" % st.max())
print("heavy phase end: median %.1f max %.1f" % (np.median(th), th.max()))
print("warp end: median %.1f p90 %.1f max %.1f" % (np.median(en), np.percentile(en, 90), en.max()))
i = np.argsort(-en)[:12]
for k in i:
    print("  sm %3d start %.1f heavy_end %.1f end %.1f heavy %d light %d first %d" % (t[k, 0], st[k], th[k], en[k], nh[k], nl[k], t[k, 4]))
# per-SM busy
sm = t[:, 0]
print("items heavy total", nh.sum(), "light total", nl.sum())
