"""A/B: Static solve time on the base pair's layout (built from scratch) vs
on a batch snapshot's layout derived from it (layout.cu build_incremental)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2404_08299_b200 as dp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = dp.rmat_graph(scale); gt = dp.transpose(g)
dp.prepare(gt, g)
out = torch.empty(g.vertex_count, dtype=torch.float64, device="cuda")
def t(gt_, g_, k=3):
    return [round(dp.static_pagerank(gt_, g_, out=out).device_ms if False else _solve(gt_, g_), 3) for _ in range(k)]
from paper_2404_08299_b200 import _native as N
import ctypes as C
def _solve(gt_, g_):
    st = N.Stats(); cfg = dp.EngineConfig()._c()
    dp._check(N.lib().dynpr_static_pagerank(C.c_void_p(g_.ctx.h), C.c_void_p(gt_.h), C.c_void_p(g_.h), C.byref(cfg),
                                            C.c_void_p(out.data_ptr()), C.byref(st), N.OBSERVER(0), None))
    return st.device_ms
print("base (gen 0):", t(gt, g))
b = dp.generate_random_batch(g, dp.batch_size_from_fraction(1e-4, g.edge_count), 0.8, 5)
g2, gt2 = dp.apply_batch_pair(g, gt, b)
dp.prepare(gt2, g2)
print("derived gen %d:" % dp.layout_info(gt2)["generation"], t(gt2, g2))
g3 = dp.CsrGraph.from_csr(g2.vertex_count, g2.offsets, g2.targets); gt3 = dp.transpose(g3)
dp.prepare(gt3, g3)
print("same graph rebuilt (gen %d):" % dp.layout_info(gt3)["generation"], t(gt3, g3))
print("base again:", t(gt, g))
