"""The range-partitioned engine as N PROCESSES on one B200.

Two processes, one torch.distributed (gloo) process group, both on cuda:0:
each creates a team context whose collectives go through the process group
(`Context.hostcomm` + `TorchDistTransport`: dynpr_context_create_hostcomm,
the same engine team path the NCCL context takes -- range plan, record
all-reduce, contribution all-gather, pending-flag bitmap exchange, graph
identity check, speculative host loop).  With `IpcExchange` the two
processes map each other's contribution buffers through CUDA IPC and every
sweep stores into both copies (the fused exchange across processes).  NCCL
itself refuses two ranks on one GPU; on a multi-GPU box the same engine
code runs over NCCL (bench.py --gpus N).

Every rank must return exactly the single-GPU result (itself bitwise equal
to the reference library, tests/test_gpu_engine.py), and the reference
library is checked directly on one case.
"""
import os
import socket
import traceback

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _same(a, b, what):
    assert a.iterations == b.iterations, (what, a.iterations, b.iterations)
    assert a.converged == b.converged, what
    assert a.affected_vertex_iterations == b.affected_vertex_iterations, what
    assert a.final_delta == b.final_delta, what
    assert np.array_equal(a.ranks, b.ranks), what


def _worker(rank, port, case, scale, q):
    try:
        import sys
        sys.path.insert(0, ROOT)
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
        import paper_2404_08299_b200 as dp
        _run_case(dp, dist, rank, case, scale)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, None))
    except BaseException:  # pragma: no cover - reported by the parent
        q.put((rank, traceback.format_exc()))


def _graphs(dp, scale, ctx):
    g = dp.rmat_graph(scale, ctx=ctx)
    return g, dp.transpose(g)


def _run_case(dp, dist, rank, case, scale):
    plain = dp.Context(0)
    team = dp.context_from_process_group(0, transport="host")
    assert (team.rank, team.world) == (rank, WORLD)
    g1, gt1 = _graphs(dp, scale, plain)
    g2, gt2 = _graphs(dp, scale, team)
    ipc = dp.IpcExchange(team, g2.vertex_count) if case.endswith("fused") else None
    try:
        if case.startswith("engines"):
            ref = dp.static_pagerank(gt1, g1)
            got = dp.static_pagerank(gt2, g2)
            _same(got, ref, "static")
            # a batch identical on both ranks (same seed): DF-P, DF, ND
            batch = dp.generate_random_batch(g1, dp.batch_size_from_fraction(1e-3, g1.edge_count), 0.8, 11)
            h1, ht1 = dp.apply_batch_pair(g1, gt1, batch)
            h2, ht2 = dp.apply_batch_pair(g2, gt2, batch)
            for pruning in (True, False):
                a = dp.dynamic_frontier(h1, ht1, batch.deletions, batch.insertions, ref.ranks, pruning=pruning)
                b = dp.dynamic_frontier(h2, ht2, batch.deletions, batch.insertions, ref.ranks, pruning=pruning)
                _same(b, a, f"df pruning={pruning}")
                assert b.affected_vertex_iterations < b.iterations * h1.vertex_count  # a real frontier
            a = dp.naive_dynamic(ht1, h1, ref.ranks)
            b = dp.naive_dynamic(ht2, h2, ref.ranks)
            _same(b, a, "nd")
            a = dp.dynamic_traversal(h1, ht1, batch.deletions, batch.insertions, ref.ranks)
            b = dp.dynamic_traversal(h2, ht2, batch.deletions, batch.insertions, ref.ranks)
            _same(b, a, "dt")
            # iteration caps: odd / even exits of the speculative team loop
            for cap in (1, 2, 7):
                cfg = dp.EngineConfig(max_iterations=cap)
                _same(dp.static_pagerank(gt2, g2, cfg), dp.static_pagerank(gt1, g1, cfg), f"cap {cap}")
        elif case == "reference":
            import oracle
            O = oracle.Oracle("ref") if oracle.available("ref") else oracle.Oracle("port")
            off, tgt = g2.offsets, g2.targets
            og = O.graph_from_csr(g2.vertex_count, off, tgt)
            ogt = O.transpose(og)
            ref = O.static(ogt, og)
            got = dp.static_pagerank(gt2, g2)
            assert got.iterations == ref.iterations
            assert np.array_equal(got.ranks, ref.ranks)
            dels, ins = O.generate_random_batch(og, O.batch_size_from_fraction(1e-3, og.m), 0.8, 5)
            og2, _, _ = O.apply_batch(og, dels, ins)
            ogt2 = O.transpose(og2)
            rd = O.dynamic_frontier(og2, ogt2, dels, ins, ref.ranks, pruning=True)
            h2, ht2 = dp.apply_batch_pair(g2, gt2, dp.BatchUpdate(dels, ins))
            d = dp.dynamic_frontier(h2, ht2, dels, ins, got.ranks, pruning=True)
            assert d.iterations == rd.iterations
            assert d.affected_vertex_iterations == rd.affected_vertex_iterations
            assert np.array_equal(d.ranks, rd.ranks)
        elif case == "csr_entry":
            # the by-value entry (host CSR pair -> upload -> solve) on a team:
            # the forward targets' side upload is joined before the identity
            # fingerprint (no race between them)
            import ctypes as C
            from paper_2404_08299_b200 import _native as N
            ref = dp.static_pagerank(gt1, g1)
            n, m = g1.vertex_count, g1.edge_count
            off_t, tgt_t = gt1.offsets, gt1.targets
            off_f, tgt_f = g1.offsets, g1.targets
            for _ in range(3):
                out = np.empty(n, dtype=np.float64)
                st = N.Stats()
                cfg = dp.EngineConfig()._c()
                dp._check(N.lib().dynpr_static_pagerank_csr(
                    C.c_void_p(team.h), n, off_t.ctypes.data_as(C.c_void_p), tgt_t.ctypes.data_as(C.c_void_p),
                    off_f.ctypes.data_as(C.c_void_p), tgt_f.ctypes.data_as(C.c_void_p), m, C.byref(cfg),
                    out.ctypes.data_as(C.c_void_p), C.byref(st), N.OBSERVER(0), None))
                assert st.iterations == ref.iterations
                assert np.array_equal(out, ref.ranks)
        elif case == "mismatch":
            # rank 1 holds a different graph of the same size: every rank
            # raises instead of combining ranges of two graphs
            if rank == 1:
                off, tgt = g2.offsets.copy(), g2.targets.copy()
                v = int(np.argmax(np.diff(off) > 2))
                row = set(tgt[off[v]:off[v + 1]].tolist())
                new = next(u for u in range(g2.vertex_count) if u not in row)
                row.discard(max(u for u in row if u != v))  # move one edge, keep the self-loop
                row.add(new)
                tgt[off[v]:off[v + 1]] = np.array(sorted(row), dtype=np.uint32)
                g2 = dp.CsrGraph.from_csr(g2.vertex_count, off, tgt, ctx=team)
                gt2 = dp.transpose(g2)
            with pytest.raises(ValueError, match="ranks hold different graphs"):
                dp.static_pagerank(gt2, g2)
        else:
            raise AssertionError(case)
    finally:
        if ipc is not None:
            ipc.close()


def _spawn(case, scale):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, case, scale, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(WORLD):
            r, err = q.get(timeout=600)
            results[r] = err
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    errs = {r: e for r, e in results.items() if e}
    assert not errs, "\n".join(f"rank {r}:\n{e}" for r, e in errs.items())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


@pytest.mark.parametrize("case", ["engines-allgather", "engines-fused"])
@pytest.mark.parametrize("scale", [10, 14])
def test_two_processes_equal_single_gpu(case, scale):
    _spawn(case, scale)


def test_two_processes_equal_reference_library():
    _spawn("reference", 13)


def test_two_processes_host_csr_entry():
    _spawn("csr_entry", 12)


def test_two_processes_reject_different_graphs():
    _spawn("mismatch", 10)
