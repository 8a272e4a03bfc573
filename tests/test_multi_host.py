"""Host side of the multi-GPU path on CPU: torch.distributed (gloo), world 2.

* the NCCL bootstrap: rank 0's ncclGetUniqueId shared over the process group
  (paper_2404_08299_b200.share_nccl_unique_id) reaches every rank intact;
* the exchange protocol of the range-partitioned engine: each
  rank updates only its edge-balanced range of vertices, the new
  contributions are all-gathered and the L-inf delta all-reduced (max) after
  every sweep -- restated here in plain Python over the oracle's CSR, it
  reproduces the reference staticPageRank bit for bit (the device engine's
  own partitioned path is tested against the single-GPU engine in
  tests/test_gpu_multi.py);
* bench.py's max-over-ranks timing reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def edge_balanced_cuts(indeg, world):
    """Contiguous vertex ranges holding ~m/world in-edges each (the cut rule of
    csrc/sweep.cu plan_ranges, without the SELL slice alignment)."""
    pre = np.concatenate([[0], np.cumsum(indeg, dtype=np.int64)])
    m = pre[-1]
    cuts = [0] + [int(np.searchsorted(pre, m * r / world, side="left")) for r in range(1, world)] + [len(indeg)]
    return cuts


def partitioned_static(rank, world, off_t, tgt_t, outdeg, alpha=0.85, tol=1e-10, max_iter=500):
    n = len(outdeg)
    indeg = np.diff(off_t)
    cuts = edge_balanced_cuts(indeg, world)
    lo, hi = cuts[rank], cuts[rank + 1]
    ranks = [1.0 / n] * n
    teleport = (1.0 - alpha) / n  # rank.cpp:85
    iters = 0
    import torch
    for it in range(max_iter):
        contrib = [ranks[u] / float(outdeg[u]) for u in range(n)]
        mine = []
        delta = 0.0
        for v in range(lo, hi):  # owned rows; flat sums (in-degree <= 32 here)
            c = 0.0
            for u in tgt_t[off_t[v]:off_t[v + 1]]:
                c += contrib[u]
            r = teleport + alpha * c
            delta = max(delta, abs(r - ranks[v]))
            mine.append(r)
        # allgather of the owned slices (padded to equal length) + allreduce(max)
        width = max(cuts[i + 1] - cuts[i] for i in range(world))
        buf = torch.zeros(width, dtype=torch.float64)
        buf[: len(mine)] = torch.tensor(mine, dtype=torch.float64)
        parts = [torch.zeros(width, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, buf)
        new = []
        for i in range(world):
            new.extend(parts[i][: cuts[i + 1] - cuts[i]].tolist())
        d = torch.tensor([delta], dtype=torch.float64)
        dist.all_reduce(d, op=dist.ReduceOp.MAX)
        ranks = new
        iters = it + 1
        if d.item() <= tol:
            break
    return np.array(ranks), iters


def worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import bench
        import oracle
        import paper_2404_08299_b200 as dp
        res = {}
        uid = dp.share_nccl_unique_id()
        ids = [None] * WORLD
        dist.all_gather_object(ids, uid)
        res["uid_ok"] = len(uid) == 128 and all(i == ids[0] for i in ids)

        O = oracle.Oracle("port")
        g = O.random_graph(O.rng(77), 400, 3000)
        gl = O.add_self_loops(g)
        gt = O.transpose(gl)
        off_t, tgt_t = gt.csr()
        off_f, _ = gl.csr()
        ranks, iters = partitioned_static(rank, WORLD, off_t, tgt_t, np.diff(off_f))
        ref = O.static(gt, gl)
        res["ranks_equal"] = bool(np.array_equal(ranks, ref.ranks))
        res["iters_equal"] = iters == ref.iterations

        # the host transport of the cross-process team engine
        # (Context.hostcomm): the C callbacks dynpr_comm_ops, called exactly
        # as libdynpr_cuda.so's HostComm calls them
        import ctypes as C
        t = dp.TorchDistTransport()
        mx = (C.c_uint64 * 2)(2**63 + rank, 7)
        sm = (C.c_uint64 * 3)(rank + 1, 2**64 - 1, 10)
        rc = [t.ops.allreduce_u64(mx, 2, 1, None), t.ops.allreduce_u64(sm, 3, 0, None)]
        res["allreduce"] = (rc, list(mx), list(sm))
        gathered = []
        for off in ([0, 3, 8], [0, 0, 4], [0, 5, 5]):
            buf = (C.c_uint8 * max(off[-1], 1))()
            for i in range(off[rank], off[rank + 1]):
                buf[i] = 10 * rank + i
            o = (C.c_uint64 * 3)(*off)
            rc = t.ops.allgatherv(C.addressof(buf), o, WORLD, None)
            gathered.append((rc, list(buf)[: off[-1]]))
        res["allgatherv"] = gathered
        res["barrier"] = t.ops.barrier(None)
        res["max_over_ranks"] = bench.max_over_ranks(float(rank + 1), WORLD)
        res["sum_over_ranks"] = bench.sum_over_ranks(float(rank + 1), WORLD)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_multi_rank_host_protocol_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=540) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(WORLD):
        assert got[r]["uid_ok"]
        assert got[r]["ranks_equal"]
        assert got[r]["iters_equal"]
        rc, mx, sm = got[r]["allreduce"]
        assert rc == [0, 0]
        assert mx == [2**63 + 1, 7]  # unsigned max
        assert sm == [3, 2**64 - 2, 20]  # sum mod 2^64
        expect = []
        for off in ([0, 3, 8], [0, 0, 4], [0, 5, 5]):
            expect.append((0, [10 * q + i for q in range(WORLD) for i in range(off[q], off[q + 1])]))
        assert got[r]["allgatherv"] == expect
        assert got[r]["barrier"] == 0
        assert got[r]["max_over_ranks"] == float(WORLD)
        assert got[r]["sum_over_ranks"] == float(WORLD * (WORLD + 1) // 2)
