"""Flagged-sweep overhead: per-iteration device-loop times (k_loop_end
trace) of Static vs DF started with every vertex affected
(dynamic_frontier_from_flags, all-ones vertexAffected, no pruning) on the
same RMAT-S graph -- the same gathers, plus the frontier epilogue (flags,
copy-through bookkeeping, pending lists / sign bits)."""
import ctypes as C
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2404_08299_b200 as dp
from paper_2404_08299_b200 import _native as N

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = dp.rmat_graph(scale); gt = dp.transpose(g); dp.prepare(gt, g)
n = g.vertex_count


def trace(n_it):
    cnt = C.c_uint64()
    N.lib().dynpr_debug_loop_trace(None, 0, C.byref(cnt))
    buf = np.zeros(cnt.value, np.uint64)
    N.lib().dynpr_debug_loop_trace(buf.ctypes.data, cnt.value, None)
    t = buf.reshape(-1, 4)[:n_it]
    return np.diff(t[:, 0].astype(np.int64)) / 1e3


base = dp.static_pagerank(gt, g)
cfg = dp.EngineConfig(max_iterations=12, convergence_check_disabled=True)
for name, fn in (("static", lambda: dp.static_pagerank(gt, g, cfg)),
                 ("df all-affected", lambda: dp.dynamic_frontier_from_flags(
                     g, gt, np.ones(n, np.uint8), np.zeros(n, np.uint8), base.ranks, cfg, False)),
                 ("dfp all-affected", lambda: dp.dynamic_frontier_from_flags(
                     g, gt, np.ones(n, np.uint8), np.zeros(n, np.uint8), base.ranks, cfg, True))):
    fn()
    r = fn()
    dt = trace(r.iterations)
    print("%-18s iterations 2..%d: median %.1f us, min %.1f us" % (name, r.iterations, np.median(dt), dt.min()),
          flush=True)
