"""Per-iteration cost of the team path on one GPU (RMAT-24 Static): the
single-GPU device loop, the single-GPU host loop (DYNPR_HOST_LOOP=1), and a
1-rank NCCL team forced onto the team path (DYNPR_FORCE_TEAM=1: range plan,
record all-reduce per sweep, speculative host loop), with and without the
fused exchange buffers attached.
    python profiles/team_overhead_probe.py [scale]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2404_08299_b200 as dp  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24


def timed(label, gt, g, reps=3):
    dp.static_pagerank(gt, g)
    ms = [dp.static_pagerank(gt, g).device_ms for _ in range(reps)]
    r = dp.static_pagerank(gt, g)
    print("%-34s %.2f ms  (%d it, %.1f us/it)" % (label, statistics.median(ms), r.iterations,
                                                   1e3 * statistics.median(ms) / r.iterations), flush=True)


g = dp.rmat_graph(scale)
gt = dp.transpose(g)
dp.prepare(gt, g)
timed("single GPU, device loop", gt, g)
os.environ["DYNPR_HOST_LOOP"] = "1"
timed("single GPU, host loop", gt, g)
del os.environ["DYNPR_HOST_LOOP"]
ctx = dp.Context.nccl(0, 0, 1, dp.nccl_unique_id())
h = dp.CsrGraph.from_csr(g.vertex_count, g.offsets, g.targets, ctx=ctx)
ht = dp.transpose(h)
dp.prepare(ht, h)
os.environ["DYNPR_FORCE_TEAM"] = "1"
timed("1-rank NCCL team, all-gather", ht, h)
bufs = [torch.empty(g.vertex_count, dtype=torch.float64, device="cuda:0") for _ in range(2)]
ctx.attach_peers([bufs[0].data_ptr()], [bufs[1].data_ptr()], g.vertex_count)
timed("1-rank NCCL team, fused exchange", ht, h)
