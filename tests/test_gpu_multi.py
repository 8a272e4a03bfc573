"""The range-partitioned multi-GPU engine on one B200.

A LocalTeam runs P virtual ranks of the partitioned engine on host threads
of this process, all on cuda:0, through the same engine code path as the
NCCL team (each rank sweeps its edge-balanced vertex range; contributions,
pending flags and the reduction record are exchanged after every sweep).
Every rank must return exactly the single-GPU result, which itself equals
the reference's (tests/test_gpu_engine.py).  NCCL cannot put two ranks on
one GPU, so the NCCL transport itself is exercised only on multi-GPU boxes
(bench.py --gpus N).
"""
import os
import threading

import numpy as np
import pytest

from helpers import rand_pair

pytestmark = pytest.mark.gpu


def run_team(dp, world, fn, fused_n=0):
    """fn(ctx, rank) on `world` threads with virtual-rank contexts; with
    fused_n > 0 the ranks get peer contribution buffers (fused exchange:
    each sweep stores into every rank's copy, no all-gather)."""
    team = dp.LocalTeam(world)
    ctxs = [team.context(0, r) for r in range(world)]
    if fused_n:
        import torch
        bufs = [[torch.empty(fused_n, dtype=torch.float64, device="cuda:0") for _ in range(world)] for _ in range(2)]
        ptrs = [[b.data_ptr() for b in bufs[k]] for k in range(2)]
        for c in ctxs:
            c.attach_peers(ptrs[0], ptrs[1], fused_n)
        ctxs.append(bufs)  # keep the buffers alive with the contexts
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(ctxs[r], r)
        except BaseException as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    assert all(o is not None for o in out)
    return out, ctxs


def same(a, b):
    assert a.iterations == b.iterations
    assert a.converged == b.converged
    assert a.affected_vertex_iterations == b.affected_vertex_iterations
    assert a.final_delta == b.final_delta
    assert np.array_equal(a.ranks, b.ranks)


def test_attach_peers_validates(dp):
    team = dp.LocalTeam(2)
    c = team.context(0, 0)
    with pytest.raises(ValueError, match="world does not match"):
        c.attach_peers([1, 2, 3], [4, 5, 6], 10)
    c.attach_peers([], [], 0)  # detach is always allowed


def test_team_reports_rank_and_world(dp):
    team = dp.LocalTeam(3)
    ctxs = [team.context(0, r) for r in range(3)]
    assert [(c.rank, c.world) for c in ctxs] == [(0, 3), (1, 3), (2, 3)]
    assert (dp.default_context().rank, dp.default_context().world) == (0, 1)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("scale", [10, 13])
@pytest.mark.parametrize("fused", [False, True], ids=["allgather", "fused-peer-stores"])
def test_partitioned_static_and_dfp_equal_single_gpu(dp, oracle_lib, world, scale, fused):
    O = oracle_lib
    src, dst = O.rmat_edges(scale, 16 << scale)
    og = O.add_self_loops(O.build_csr((src, dst), 1 << scale))
    off, tgt = og.csr()
    n = og.n
    dels, ins = O.generate_random_batch(og, O.batch_size_from_fraction(1e-3, og.m), 0.8, 5)
    og2, _, _ = O.apply_batch(og, dels, ins)
    off2, tgt2 = og2.csr()

    g = dp.CsrGraph.from_csr(n, off, tgt)
    gt = dp.transpose(g)
    base = dp.static_pagerank(gt, g)
    g2 = dp.CsrGraph.from_csr(n, off2, tgt2)
    gt2 = dp.transpose(g2)
    single = {
        "static": base,
        "nd": dp.naive_dynamic(gt2, g2, base.ranks),
        "df": dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=False),
        "dfp": dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=True),
    }
    # the checker agrees with the single-GPU engine (bitwise)
    ref = O.dynamic_frontier(og2, O.transpose(og2), dels, ins, O.static(O.transpose(og), og).ranks,
                             pruning=True)
    assert np.array_equal(single["dfp"].ranks, ref.ranks)

    def fn(ctx, r):
        h = dp.CsrGraph.from_csr(n, off, tgt, ctx=ctx)
        ht = dp.transpose(h)
        b = dp.static_pagerank(ht, h)
        h2 = dp.CsrGraph.from_csr(n, off2, tgt2, ctx=ctx)
        ht2 = dp.transpose(h2)
        return {
            "static": b,
            "nd": dp.naive_dynamic(ht2, h2, b.ranks),
            "df": dp.dynamic_frontier(h2, ht2, dels, ins, b.ranks, pruning=False),
            "dfp": dp.dynamic_frontier(h2, ht2, dels, ins, b.ranks, pruning=True),
        }

    out, _ = run_team(dp, world, fn, fused_n=n if fused else 0)
    for r in range(world):
        for k in single:
            same(out[r][k], single[k])


def test_partitioned_observer_sees_full_iterates(dp, oracle_lib):
    O = oracle_lib
    og, ogt = rand_pair(O, 23, 3000, 40000)
    off, tgt = og.csr()
    seen_single = []
    g = dp.CsrGraph.from_csr(og.n, off, tgt)
    dp.static_pagerank(dp.transpose(g), g, observer=lambda it, r: seen_single.append(r.copy()))

    def fn(ctx, r):
        seen = []
        h = dp.CsrGraph.from_csr(og.n, off, tgt, ctx=ctx)
        dp.static_pagerank(dp.transpose(h), h, observer=lambda it, x: seen.append(x.copy()))
        return seen

    out, _ = run_team(dp, 2, fn)
    for seen in out:
        assert len(seen) == len(seen_single)
        for a, b in zip(seen, seen_single):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("fused", [False, True], ids=["allgather", "fused-peer-stores"])
@pytest.mark.parametrize("max_it,check_off", [(1, False), (2, False), (5, True), (6, True), (500, False)])
def test_team_speculative_loop_limits(dp, oracle_lib, fused, max_it, check_off):
    """The team loop enqueues iteration k+1 before reading iteration k's
    record: every exit (convergence on either parity, max iterations, check
    disabled) must still return exactly the single-GPU result."""
    O = oracle_lib
    og, ogt = rand_pair(O, 29, 4000, 50000)
    off, tgt = og.csr()
    n = og.n
    dels, ins = O.generate_random_batch(og, 40, 0.8, 11)
    og2, _, _ = O.apply_batch(og, dels, ins)
    off2, tgt2 = og2.csr()
    cfg = dp.EngineConfig(max_iterations=max_it, convergence_check_disabled=check_off)
    g = dp.CsrGraph.from_csr(n, off, tgt)
    base = dp.static_pagerank(dp.transpose(g), g)
    g2 = dp.CsrGraph.from_csr(n, off2, tgt2)
    gt2 = dp.transpose(g2)
    single = {"static": dp.static_pagerank(gt2, g2, cfg),
              "dfp": dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, cfg, True)}

    def fn(ctx, r):
        h2 = dp.CsrGraph.from_csr(n, off2, tgt2, ctx=ctx)
        ht2 = dp.transpose(h2)
        return {"static": dp.static_pagerank(ht2, h2, cfg),
                "dfp": dp.dynamic_frontier(h2, ht2, dels, ins, base.ranks, cfg, True)}

    out, _ = run_team(dp, 3, fn, fused_n=n if fused else 0)
    for r in range(3):
        for k in single:
            same(out[r][k], single[k])


@pytest.mark.parametrize("fused", [False, True], ids=["allgather", "fused-peer-stores"])
def test_team_rejects_ranks_with_different_graphs(dp, oracle_lib, fused):
    """A team sweeps ONE replicated graph.  Ranks holding different graphs of
    the same size (same n and m, one edge moved) must all fail the solve
    instead of combining ranges of different graphs; identical graphs pass."""
    O = oracle_lib
    og, _ = rand_pair(O, 31, 3000, 30000)
    off, tgt = og.csr()
    n = og.n
    tgt_b = np.array(tgt, copy=True)
    # move one edge of vertex 0 to a target it does not have yet (same n, m)
    row = set(tgt_b[off[0]:off[1]].tolist())
    new_t = next(t for t in range(1, n) if t not in row)
    k = int(off[0]) + next(i for i, t in enumerate(tgt_b[off[0]:off[1]].tolist()) if t != 0)
    tgt_b[k] = new_t
    tgt_b[off[0]:off[1]] = np.sort(tgt_b[off[0]:off[1]])

    def fn_for(graphs):
        def fn(ctx, r):
            h = dp.CsrGraph.from_csr(n, off, graphs[r], ctx=ctx)
            ht = dp.transpose(h)
            try:
                return dp.static_pagerank(ht, h)
            except ValueError as e:
                return e
        return fn

    out, _ = run_team(dp, 2, fn_for([tgt, tgt_b]), fused_n=n if fused else 0)
    assert all(isinstance(o, ValueError) and "different graphs" in str(o) for o in out), out
    out, _ = run_team(dp, 2, fn_for([tgt, tgt]), fused_n=n if fused else 0)
    single = dp.static_pagerank(dp.transpose(dp.CsrGraph.from_csr(n, off, tgt)), dp.CsrGraph.from_csr(n, off, tgt))
    for o in out:
        same(o, single)


def test_nccl_context_single_rank(dp, oracle_lib):
    """The NCCL plumbing of the one-process-per-GPU path on this one-GPU box:
    libnccl is found, a 1-rank communicator initialises and is torn down
    with its context, and solves through it equal the plain context's
    (a 1-rank team sweeps the whole vertex range, no collectives)."""
    ctx = dp.Context.nccl(0, 0, 1, dp.nccl_unique_id())
    assert (ctx.rank, ctx.world) == (0, 1)
    O = oracle_lib
    og, _ = rand_pair(O, 37, 2000, 20000)
    off, tgt = og.csr()
    n = og.n
    g = dp.CsrGraph.from_csr(n, off, tgt, ctx=ctx)
    gt = dp.transpose(g)
    p = dp.CsrGraph.from_csr(n, off, tgt)
    pt = dp.transpose(p)
    same(dp.static_pagerank(gt, g), dp.static_pagerank(pt, p))
    # DYNPR_FORCE_TEAM: the 1-rank communicator takes the team path, so the
    # real NCCL collectives (record all-reduce, broadcast-based all-gather,
    # graph identity check) and the speculative host loop run here too
    dels, ins = O.generate_random_batch(og, 30, 0.8, 5)
    og2, _, _ = O.apply_batch(og, dels, ins)
    off2, tgt2 = og2.csr()
    g2 = dp.CsrGraph.from_csr(n, off2, tgt2, ctx=ctx)
    gt2 = dp.transpose(g2)
    p2 = dp.CsrGraph.from_csr(n, off2, tgt2)
    pt2 = dp.transpose(p2)
    base = dp.static_pagerank(pt, p)
    want = {"static": dp.static_pagerank(pt2, p2),
            "dfp": dp.dynamic_frontier(p2, pt2, dels, ins, base.ranks, pruning=True),
            "dt": dp.dynamic_traversal(p2, pt2, dels, ins, base.ranks)}
    os.environ["DYNPR_FORCE_TEAM"] = "1"
    try:
        got = {"static": dp.static_pagerank(gt2, g2),
               "dfp": dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=True),
               "dt": dp.dynamic_traversal(g2, gt2, dels, ins, base.ranks)}
    finally:
        del os.environ["DYNPR_FORCE_TEAM"]
    for k in want:
        same(got[k], want[k])
    del g, gt, g2, gt2


@pytest.mark.parametrize("n", [1, 5, 40, 97])
def test_tiny_graphs_on_a_wide_team(dp, n):
    """Range plan edge cases (device prefix scan + binary search): fewer
    vertices or slices than ranks leaves trailing ranks empty; every rank
    still returns exactly the single-GPU result."""
    edges = [(u, (u * 7 + 3) % n) for u in range(n)] + [(u, (u + 1) % n) for u in range(0, n, 3)]
    g = dp.add_self_loops(dp.build_csr(edges, n))
    gt = dp.transpose(g)
    single = dp.static_pagerank(gt, g)

    def fn(ctx, r):
        h = dp.add_self_loops(dp.build_csr(edges, n, ctx=ctx))
        return dp.static_pagerank(dp.transpose(h), h)

    out, _ = run_team(dp, 4, fn)
    for o in out:
        same(o, single)


@pytest.mark.parametrize("world", [2, 4])
def test_team_layout_holds_only_owned_rows(dp, world):
    """SURVEY 8e ownership: a team rank's engine layout holds only its own
    in-CSR rows (SELL slices of its edge-balanced vertex range), so the
    per-rank layout memory is ~1/world of the single-GPU one; the owned
    ranges tile the vertex space; team DF/DF-P expand by pull and never
    build the relabelled forward CSR."""
    scale = 14
    g = dp.rmat_graph(scale)
    gt = dp.transpose(g)
    dp.prepare(gt, g)
    whole = dp.layout_info(gt)
    assert whole["v_lo"] == 0 and whole["v_hi"] == g.vertex_count and whole["has_forward"]

    def fn(ctx, r):
        h = dp.rmat_graph(scale, ctx=ctx)
        ht = dp.transpose(h)
        dp.prepare(ht, h)
        info = dp.layout_info(ht)
        batch = dp.generate_random_batch(h, 200, 0.8, 3)
        h2, ht2 = dp.apply_batch_pair(h, ht, batch)
        b = dp.static_pagerank(ht, h)
        d = dp.dynamic_frontier(h2, ht2, batch.deletions, batch.insertions, b.ranks, pruning=True)
        with pytest.raises(ValueError, match="team context"):
            dp.update_ranks(ht, h, b.ranks)
        return info, dp.layout_info(ht2), d

    out, _ = run_team(dp, world, fn)
    infos = [o[0] for o in out]
    assert infos[0]["v_lo"] == 0 and infos[-1]["v_hi"] == g.vertex_count
    for a, b in zip(infos, infos[1:]):
        assert a["v_hi"] == b["v_lo"]
    total = sum(i["sell_words"] for i in infos)
    assert whole["sell_words"] <= total <= whole["sell_words"] * 1.02  # boundary slices only
    for i in infos:
        assert i["sell_words"] <= whole["sell_words"] / world * 1.25
        assert not i["has_forward"]
    for _, after, _ in out:
        assert not after["has_forward"]
    batch = dp.generate_random_batch(g, 200, 0.8, 3)
    g2, gt2 = dp.apply_batch_pair(g, gt, batch)
    single = dp.dynamic_frontier(g2, gt2, batch.deletions, batch.insertions, dp.static_pagerank(gt, g).ranks,
                                 pruning=True)
    for _, _, d in out:
        same(d, single)
