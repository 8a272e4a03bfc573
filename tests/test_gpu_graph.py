"""Device CSR build / transpose / self-loops / batch ingest vs the reference.

Known answers restate proj/tests/unit/test_graph.cpp; random cases compare the
device CSR bytes with the oracle (the reference library when oracle/_ref is
built) -- CsrGraph equality is byte equality (graph.hpp:43).
"""
import numpy as np
import pytest

import oracle

from helpers import rand_pair, same_csr, to_dev

pytestmark = pytest.mark.gpu


def test_build_csr_empty_graph(dp):  # test_graph.cpp:12-17
    g = dp.build_csr([], 0)
    assert g.vertex_count == 0 and g.edge_count == 0
    assert g.offsets.tolist() == [0]


def test_build_csr_collapses_duplicates(dp):  # test_graph.cpp:19-23
    g = dp.build_csr([(0, 1), (0, 1), (1, 0)], 2)
    assert g.offsets.tolist() == [0, 1, 2]
    assert g.targets.tolist() == [1, 0]


def test_build_csr_rejects_out_of_range(dp):  # test_graph.cpp:25-28
    with pytest.raises(ValueError, match=r"buildCsr: vertex id out of range \(0,5\) for \|V\|=3"):
        dp.build_csr([(0, 1), (0, 5), (7, 7)], 3)
    with pytest.raises(ValueError):
        dp.build_csr([(0, 0)], 0)


@pytest.mark.parametrize("n,pairs,seed", [(20, 100, 11), (1000, 8000, 3), (70000, 500000, 5)])
def test_build_csr_matches_oracle(dp, oracle_lib, n, pairs, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, pairs, dtype=np.uint32)
    dst = rng.integers(0, n, pairs, dtype=np.uint32)
    g = dp.build_csr((src, dst), n)
    assert same_csr(g, oracle_lib.build_csr((src, dst), n))


def test_transpose_reverses_a_path(dp):  # test_graph.cpp:48-53
    t = dp.transpose(dp.build_csr([(0, 1), (1, 2)], 3))
    assert t.offsets.tolist() == [0, 0, 1, 2]
    assert t.targets.tolist() == [0, 1]


def test_transpose_fixes_self_loop_only_graphs(dp):  # test_graph.cpp:55-58
    g = dp.build_csr([(0, 0), (1, 1), (2, 2)], 3)
    assert dp.transpose(g) == g


@pytest.mark.parametrize("seed,n,pairs", [(5, 50, 300), (9, 3000, 40000)])
def test_transpose_matches_oracle_and_is_involutive(dp, oracle_lib, seed, n, pairs):
    g, gt = rand_pair(oracle_lib, seed, n, pairs)
    dg = to_dev(dp, g)
    dt = dp.transpose(dg)
    assert same_csr(dt, gt)
    assert dp.transpose(dt) == dg  # test_graph.cpp:60-67


def test_add_self_loops(dp):  # test_graph.cpp:69-80
    g = dp.add_self_loops(dp.build_csr([], 3))
    assert g.edge_count == 3 and all(g.has_self_loop(v) for v in range(3))
    bare = dp.build_csr([(0, 1), (1, 1), (2, 0)], 3)
    a = dp.add_self_loops(bare)
    assert a.edge_count == bare.edge_count + 2
    assert dp.add_self_loops(a) == a


def test_add_self_loops_matches_oracle(dp, oracle_lib):
    rng = np.random.default_rng(1)
    src = rng.integers(0, 5000, 30000, dtype=np.uint32)
    dst = rng.integers(0, 5000, 30000, dtype=np.uint32)
    og = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), 5000))
    assert same_csr(dp.add_self_loops(dp.build_csr((src, dst), 5000)), og)


def test_apply_batch_replaces_an_edge(dp):  # test_graph.cpp:82-90
    g = dp.add_self_loops(dp.build_csr([(0, 1)], 2))
    nxt = dp.apply_batch(g, dp.BatchUpdate(deletions=[(0, 1)], insertions=[(1, 0)]))
    assert nxt.offsets.tolist() == [0, 1, 3]
    assert nxt.targets.tolist() == [0, 0, 1]


def test_apply_batch_with_empty_batch_equals_add_self_loops(dp):  # test_graph.cpp:92-97
    bare = dp.build_csr([(0, 1), (2, 1)], 3)
    assert dp.apply_batch(bare, dp.BatchUpdate()) == dp.add_self_loops(bare)
    aug = dp.add_self_loops(bare)
    assert dp.apply_batch(aug, dp.BatchUpdate()) == aug


def test_apply_batch_matches_the_reference(dp, oracle_lib):  # test_graph.cpp:99-121
    rng = oracle_lib.rng(99)
    for _ in range(50):
        g = oracle_lib.random_graph(rng, 30, 150)
        dels, ins, used = [], [], set()
        for _ in range(14):
            u, v = rng.bounded(30), rng.bounded(30)
            if u == v or (u, v) in used:
                continue
            used.add((u, v))
            if oracle_lib.has_edge(g, u, v):
                dels.append((u, v))
            elif rng.bounded(3) == 0:
                dels.append((u, v))
            else:
                ins.append((u, v))
        ref, miss, dup = oracle_lib.apply_batch(g, dels, ins)
        st = dp.BatchApplyStats()
        nxt = dp.apply_batch(to_dev(dp, g), dp.BatchUpdate(dels, ins), st)
        assert same_csr(nxt, ref)
        assert (st.missing_deletions, st.duplicate_insertions) == (miss, dup)


def test_apply_batch_tallies_noops(dp):  # test_graph.cpp:123-134
    g = dp.add_self_loops(dp.build_csr([(0, 1)], 3))
    st = dp.BatchApplyStats()
    nxt = dp.apply_batch(g, dp.BatchUpdate([(1, 2), (1, 2)], [(0, 1), (0, 2)]), st)
    assert st.missing_deletions == 2 and st.duplicate_insertions == 1
    assert nxt.has_edge(0, 2) and nxt.has_edge(0, 1)


def test_apply_batch_validates(dp):  # test_graph.cpp:136-150
    g = dp.add_self_loops(dp.build_csr([(0, 1)], 2))
    with pytest.raises(ValueError, match="self-loops cannot be deleted"):
        dp.apply_batch(g, dp.BatchUpdate(deletions=[(1, 1)]))
    with pytest.raises(ValueError, match="appears in both deletions and insertions"):
        dp.apply_batch(g, dp.BatchUpdate([(0, 1)], [(0, 1)]))
    with pytest.raises(ValueError, match=r"applyBatch insertions: vertex id out of range \(0,7\) for \|V\|=2"):
        dp.apply_batch(g, dp.BatchUpdate(insertions=[(0, 7)]))
    # range errors in the deletions come before self-loop errors (graph.cpp:116-120)
    with pytest.raises(ValueError, match="applyBatch deletions: vertex id out of range"):
        dp.apply_batch(g, dp.BatchUpdate(deletions=[(1, 1), (5, 0)]))


@pytest.mark.parametrize("scale,size,seed", [(12, 200, 3), (14, 3000, 8)])
def test_random_batch_ingest_pair_matches_reference(dp, oracle_lib, scale, size, seed):
    """generateRandomBatch (80/20) -> applyBatch + transpose, on RMAT."""
    src, dst = oracle_lib.rmat_edges(scale, 16 << scale)
    g = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), 1 << scale))
    gt = oracle_lib.transpose(g)
    dels, ins = oracle_lib.generate_random_batch(g, size, 0.8, seed)
    g2, miss, dup = oracle_lib.apply_batch(g, dels, ins)
    gt2 = oracle_lib.transpose(g2)
    st = dp.BatchApplyStats()
    dg2, dgt2 = dp.apply_batch_pair(to_dev(dp, g), to_dev(dp, gt), dp.BatchUpdate(dels, ins), st)
    assert same_csr(dg2, g2) and same_csr(dgt2, gt2)
    assert (st.missing_deletions, st.duplicate_insertions) == (miss, dup)


@pytest.mark.parametrize("scale", [8, 12, 16])
def test_rmat_generator_matches_oracle(dp, oracle_lib, scale):
    src, dst = oracle_lib.rmat_edges(scale, 16 << scale)
    og = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), 1 << scale))
    assert same_csr(dp.rmat_graph(scale), og)


@pytest.mark.parametrize("scale", [1, 6, 13])
def test_kronecker_generator_matches_oracle(dp, oracle_lib, scale):
    """Graph500-style Kronecker (RMAT draws + seeded id bijection) on the
    device == the C port's edges through the reference buildCsr/addSelfLoops;
    the scramble permutes ids, so the degree multisets equal RMAT's."""
    src, dst = oracle_lib.kronecker_edges(scale, 16 << scale, seed=7)
    og = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), 1 << scale))
    kg = dp.kronecker_graph(scale, seed=7)
    assert same_csr(kg, og)
    rg = dp.rmat_graph(scale, seed=7)
    assert kg.edge_count == rg.edge_count
    assert np.array_equal(np.sort(np.diff(kg.offsets)), np.sort(np.diff(rg.offsets)))


@pytest.mark.parametrize("n,off,tgt,msg", [
    (2, [0, 1, 3], [1, 0], "malformed offsets"),
    (3, [0, 1, 0, 2], [1, 0], "non-decreasing"),
    (3, [0, 2, 1, 2], [1, 0], "sorted and deduplicated"),  # vertex 0 fails first
    (2, [0, 1, 2], [1, 5], "target id out of range"),
    (2, [0, 2, 2], [1, 1], "sorted and deduplicated"),
    (3, [0, 2, 2, 3], [2, 9, 0], "target id out of range"),
])
def test_from_csr_validation(dp, oracle_lib, n, off, tgt, msg):  # graph.cpp:30-49
    with pytest.raises(oracle.OracleError) as ref_err:
        oracle_lib.graph_from_csr(n, off, tgt)
    assert msg in str(ref_err.value)
    with pytest.raises(ValueError) as err:
        dp.CsrGraph.from_csr(n, off, tgt)
    assert str(err.value) == str(ref_err.value)


def test_from_csr_accessors(dp):
    g = dp.CsrGraph.from_csr(2, [0, 1, 2], [1, 0])
    assert g.out(0) == [1] and g.out(1) == [0] and g.degree(0) == 1


@pytest.mark.parametrize("scale,frac,ins,seed", [(10, 1e-3, 0.8, 1), (14, 1e-4, 0.8, 42), (12, 1e-2, 0.5, 9),
                                                 (10, 1e-3, 1.0, 3), (10, 1e-3, 0.0, 4)])
def test_generate_random_batch_matches_reference(dp, oracle_lib, scale, frac, ins, seed):
    """workload.cpp:183-243 -- identical draws (virtual Fisher-Yates)."""
    src, dst = oracle_lib.rmat_edges(scale, 16 << scale)
    og = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), 1 << scale))
    size = oracle_lib.batch_size_from_fraction(frac, og.m)
    assert dp.batch_size_from_fraction(frac, og.m) == size
    s = oracle_lib.derive_seed(seed, 5)
    assert dp.derive_seed(seed, 5) == s
    dels, inss = oracle_lib.generate_random_batch(og, size, ins, s)
    b = dp.generate_random_batch(dp.rmat_graph(scale), size, ins, s)
    assert np.array_equal(b.deletions.src, dels[0]) and np.array_equal(b.deletions.dst, dels[1])
    assert np.array_equal(b.insertions.src, inss[0]) and np.array_equal(b.insertions.dst, inss[1])


def test_generate_random_batch_errors(dp):
    g = dp.add_self_loops(dp.build_csr([(0, 1)], 2))
    with pytest.raises(dp.SizingError, match="requested 3 deletions but only 1 non-loop edges exist"):
        dp.generate_random_batch(g, 3, 0.0, 1)
    with pytest.raises(ValueError, match="insertFraction must be in"):
        dp.generate_random_batch(g, 3, 1.5, 1)


def test_static_pagerank_csr_host_pair(dp, oracle_lib):
    """dynpr_static_pagerank_csr: one call on a host CSR pair (gF's targets
    uploaded + validated on a side stream during the solve) -- same ranks and
    counters as constructing both graphs and calling the engine, and the
    reference's error order (graph construction first, engine checks next)."""
    import ctypes as C
    from paper_2404_08299_b200 import _native as N
    O = oracle_lib
    from helpers import rand_pair
    og, ogt = rand_pair(O, 61, 5000, 50000)
    offF, tgtF = og.csr()
    offT, tgtT = ogt.csr()
    n, m = og.n, og.m
    ctx = dp.default_context()
    L = N.lib()

    def run(oT, tT, oF, tF, cfg=None, nn=n, mm=m):
        c = (cfg or dp.EngineConfig())._c()
        r = np.zeros(max(nn, 1), np.float64)
        st = N.Stats()
        rc = L.dynpr_static_pagerank_csr(C.c_void_p(ctx.h), nn, oT.ctypes.data, tT.ctypes.data, oF.ctypes.data,
                                         tF.ctypes.data, mm, C.byref(c), r.ctypes.data, C.byref(st), N.OBSERVER(0),
                                         None)
        return rc, r, st

    rc, r, st = run(offT, tgtT, offF, tgtF)
    assert rc == 0
    ref = O.static(ogt, og)
    assert st.iterations == ref.iterations and np.array_equal(r[:n], ref.ranks)
    bad = tgtF.copy()
    bad[offF[10]], bad[offF[10] + 1] = bad[offF[10] + 1], bad[offF[10]]  # unsorted slice in gF
    rc, _, _ = run(offT, tgtT, offF, bad)
    assert rc == N.DYNPR_INVALID_ARGUMENT and "sorted and deduplicated" in N.last_error()
    rc, _, _ = run(offT, tgtT, offF, bad, cfg=dp.EngineConfig(damping_factor=2.0))
    assert rc == N.DYNPR_INVALID_ARGUMENT and "sorted and deduplicated" in N.last_error()  # construction first
    rc, _, _ = run(offT, tgtT, offF, tgtF, cfg=dp.EngineConfig(damping_factor=2.0))
    assert rc == N.DYNPR_INVALID_ARGUMENT and "dampingFactor" in N.last_error()
    badT = tgtT.copy()
    badT[5] = n + 3
    rc, _, _ = run(offT, badT, offF, tgtF)
    assert rc == N.DYNPR_INVALID_ARGUMENT and "out of range" in N.last_error()
    rc, r2, _ = run(offT, tgtT, offF, tgtF)  # the context is still healthy
    assert rc == 0 and np.array_equal(r2[:n], ref.ranks)


@pytest.mark.parametrize("case", ["empty", "first_last", "every_row", "hub_rows"])
def test_apply_batch_pair_run_boundaries(dp, oracle_lib, case):
    """The ingest copies untouched rows as runs between touched rows: batches
    touching the first / last row, every row, no row, or only hub rows must
    still give the reference's bytes for both the forward and the transpose."""
    O = oracle_lib
    src, dst = O.rmat_edges(12, 16 << 12)
    og = O.add_self_loops(O.build_csr((src, dst), 1 << 12))
    n = og.n
    off, tgt = og.csr()
    rng = np.random.default_rng(5)
    if case == "empty":
        dels, ins = [], []
    elif case == "first_last":
        dels = [(0, int(t)) for t in tgt[off[0]:off[1]] if t != 0][:3] + \
               [(n - 1, int(t)) for t in tgt[off[n - 1]:off[n]] if t != n - 1][:1]
        ins = [(0, n - 1), (n - 1, 0), (n - 1, 1)]
        ins = [e for e in ins if not og_has(off, tgt, *e)]
    elif case == "every_row":
        ins = [(u, int((u * 7 + 3) % n)) for u in range(n)]
        ins = [e for e in ins if e[0] != e[1] and not og_has(off, tgt, *e)]
        dels = []
    else:
        deg = np.diff(off)
        hubs = np.argsort(-deg)[:4]
        dels = [(int(h), int(t)) for h in hubs for t in tgt[off[h]:off[h + 1]][::7] if t != h]
        ins = []
    og2, miss1, dup1 = O.apply_batch(og, dels, ins)
    g = dp.CsrGraph.from_csr(n, off, tgt)
    gt = dp.transpose(g)
    st = dp.BatchApplyStats()
    g2, gt2 = dp.apply_batch_pair(g, gt, dp.BatchUpdate(dels, ins), st)
    o2, t2 = og2.csr()
    ot2, tt2 = O.transpose(og2).csr()
    assert np.array_equal(g2.offsets, o2) and np.array_equal(g2.targets, t2)
    assert np.array_equal(gt2.offsets, ot2) and np.array_equal(gt2.targets, tt2)
    assert (st.missing_deletions, st.duplicate_insertions) == (miss1, dup1)


def og_has(off, tgt, u, v):
    row = tgt[off[u]:off[u + 1]]
    i = np.searchsorted(row, v)
    return i < len(row) and row[i] == v


def test_context_destroyed_before_its_graphs(dp):
    """Finalisers of a garbage cycle run in any order: a context destroyed
    while graphs still live defers its teardown to the last graph's
    destroy (include/dynpr_cuda.h), so neither order crashes."""
    for order in ("ctx_first", "graphs_first"):
        ctx = dp.Context(0)
        g = dp.build_csr([(0, 1), (1, 2), (2, 0)], 3, ctx=ctx)
        gt = dp.transpose(g)
        r = dp.static_pagerank(gt, g)
        assert r.converged
        if order == "ctx_first":
            ctx._fin()
            g._fin()
            gt._fin()
        else:
            gt._fin()
            g._fin()
            ctx._fin()
    # the default context is unaffected
    g = dp.add_self_loops(dp.build_csr([(0, 1)], 2))
    assert dp.static_pagerank(dp.transpose(g), g).converged
