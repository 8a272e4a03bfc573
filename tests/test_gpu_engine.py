"""Static / ND / DF / DF-P engines on the device vs the reference.

Parity bar (BASELINE.json north_star): affected-vertex sets bit-exact per
iteration, iteration counts equal, ranks within L-inf 1e-9 -- the device path
reproduces the reference's accumulation order, so the tests assert bitwise
rank equality, which implies the 1e-9 tolerance.  Known answers restate
proj/tests/unit/test_engine.cpp.
"""
import numpy as np
import pytest

import oracle
from helpers import dev_cfg, rand_pair, to_dev

pytestmark = pytest.mark.gpu
LINF_TOL = 1e-9  # north_star tolerance; bitwise equality is asserted as well


def dev_pair(dp, og, ogt):
    return to_dev(dp, og), to_dev(dp, ogt)


def assert_same_result(d, r):
    assert d.iterations == r.iterations
    assert d.converged == r.converged
    assert d.affected_vertex_iterations == r.affected_vertex_iterations
    assert np.max(np.abs(d.ranks - r.ranks)) <= LINF_TOL
    assert np.array_equal(d.ranks, r.ranks)
    assert d.final_delta == r.final_delta


def test_static_single_vertex(dp):  # test_engine.cpp:29-35
    g = dp.add_self_loops(dp.build_csr([], 1))
    r = dp.static_pagerank(dp.transpose(g), g)
    assert r.converged and r.iterations <= 2 and abs(r.ranks[0] - 1.0) <= 1e-12


def test_static_matches_dense_oracle(dp, oracle_lib):  # test_engine.cpp:37-45
    og, ogt = rand_pair(oracle_lib, 101, 100, 500)
    g, gt = dev_pair(dp, og, ogt)
    r = dp.static_pagerank(gt, g)
    off, tgt = og.csr()
    assert r.converged
    assert np.max(np.abs(r.ranks - oracle.dense_pagerank(off, tgt, 100))) <= 1e-8


def test_static_rejects_mismatched_pairs(dp):  # test_engine.cpp:47-53
    g = dp.add_self_loops(dp.build_csr([(0, 1)], 2))
    other = dp.add_self_loops(dp.build_csr([(0, 1), (1, 2)], 3))
    with pytest.raises(ValueError, match="not mutually transposed"):
        dp.static_pagerank(other, g)
    e = dp.build_csr([], 0)
    with pytest.raises(ValueError, match="engine: empty graph"):
        dp.static_pagerank(e, e)
    with pytest.raises(ValueError, match="dampingFactor must be in"):
        dp.static_pagerank(dp.transpose(g), g, dp.EngineConfig(damping_factor=1.5))


@pytest.mark.parametrize("seed,n,pairs", [(101, 100, 500), (149, 200, 2000), (7, 5000, 60000),
                                          (11, 60000, 300000)])
def test_static_bitwise_vs_reference(dp, oracle_lib, seed, n, pairs):
    og, ogt = rand_pair(oracle_lib, seed, n, pairs)
    g, gt = dev_pair(dp, og, ogt)
    ref = oracle_lib.static(ogt, og)
    assert_same_result(dp.static_pagerank(gt, g), ref)


def test_naive_dynamic(dp, oracle_lib):  # test_engine.cpp:55-103
    og, ogt = rand_pair(oracle_lib, 103, 60, 240)
    g, gt = dev_pair(dp, og, ogt)
    base = dp.static_pagerank(gt, g)
    warm = dp.naive_dynamic(gt, g, base.ranks)
    assert warm.converged and warm.iterations == 1
    assert np.max(np.abs(warm.ranks - base.ranks)) <= 1e-10
    og, ogt = rand_pair(oracle_lib, 107, 80, 400)
    g, gt = dev_pair(dp, og, ogt)
    a = dp.static_pagerank(gt, g)
    b = dp.naive_dynamic(gt, g, np.full(80, 1.0 / 80))
    assert a.iterations == b.iterations and np.array_equal(a.ranks, b.ranks)  # bitwise
    with pytest.raises(ValueError, match="naiveDynamic: previousRanks length mismatch"):
        dp.naive_dynamic(gt, g, [1.0])


def test_dynamic_frontier_empty_batch(dp, oracle_lib):  # test_engine.cpp:121-138
    og, ogt = rand_pair(oracle_lib, 113, 40, 160)
    g, gt = dev_pair(dp, og, ogt)
    prev = np.full(40, 1.0 / 40) * (1.0 + 0.01 * np.random.default_rng(0).random(40))
    for pruning in (False, True):
        r = dp.dynamic_frontier(g, gt, [], [], prev, pruning=pruning)
        assert r.converged and r.iterations == 1 and r.affected_vertex_iterations == 0
        assert np.array_equal(r.ranks, prev)


def test_full_frontier_df_matches_nd_per_iteration(dp, oracle_lib):  # test_engine.cpp:140-167
    og, ogt = rand_pair(oracle_lib, 127, 70, 350)
    g, gt = dev_pair(dp, og, ogt)
    start = np.full(70, 1.0 / 70)
    nd_it, df_it = [], []
    nd = dp.naive_dynamic(gt, g, start, observer=lambda it, r: nd_it.append(r))
    df = dp.dynamic_frontier_from_flags(g, gt, np.ones(70, np.uint8), np.zeros(70, np.uint8), start,
                                        dp.EngineConfig(frontier_tolerance=0.0), False,
                                        observer=lambda it, r, f: df_it.append(r))
    assert nd.iterations == df.iterations
    for a, b in zip(nd_it, df_it):
        assert np.max(np.abs(a - b)) <= 1e-12
    assert df.affected_vertex_iterations == df.iterations * 70


def batch_case(O, seed, n, pairs, size, ins_frac, bseed):
    og, ogt = rand_pair(O, seed, n, pairs)
    base = O.static(ogt, og)
    dels, ins = O.generate_random_batch(og, size, ins_frac, bseed)
    og2, _, _ = O.apply_batch(og, dels, ins)
    return og2, O.transpose(og2), dels, ins, base.ranks


@pytest.mark.parametrize("pruning", [False, True])
@pytest.mark.parametrize("case", [(131, 400, 4000, 8, 0.8, 2024), (137, 300, 1200, 3, 1.0, 77),
                                  (139, 150, 2500, 6, 0.8, 5), (149, 200, 2000, 10, 0.8, 11),
                                  (3, 20000, 200000, 200, 0.8, 9)])
def test_frontier_engines_bitwise_with_affected_sets(dp, oracle_lib, pruning, case):
    og2, ogt2, dels, ins, prev = batch_case(oracle_lib, *case)
    g2, gt2 = dev_pair(dp, og2, ogt2)
    trace = []
    ref = oracle_lib.dynamic_frontier(og2, ogt2, dels, ins, prev, pruning=pruning, trace=trace)
    got = []
    d = dp.dynamic_frontier(g2, gt2, dels, ins, prev, pruning=pruning,
                            observer=lambda it, r, f: got.append((it, r, f)))
    assert_same_result(d, ref)
    assert len(got) == len(trace)
    for (it, r, f), (rit, rr, rf) in zip(got, trace):
        assert it == rit
        assert np.array_equal(f, rf), f"affected set differs at iteration {it}"
        assert np.array_equal(r, rr)


def test_frontier_engines_stay_close_to_the_oracle(dp, oracle_lib):  # test_engine.cpp:169-197
    og2, ogt2, dels, ins, prev = batch_case(oracle_lib, 131, 400, 4000, 8, 0.8, 2024)
    g2, gt2 = dev_pair(dp, og2, ogt2)
    off, tgt = og2.csr()
    dense = oracle.dense_pagerank(off, tgt, og2.n)
    nd = dp.naive_dynamic(gt2, g2, prev)
    df = dp.dynamic_frontier(g2, gt2, dels, ins, prev, pruning=False)
    dfp = dp.dynamic_frontier(g2, gt2, dels, ins, prev, pruning=True)
    for r in (nd, df, dfp):
        assert np.sum(np.abs(r.ranks - dense)) <= 1e-5
    assert df.affected_vertex_iterations < nd.affected_vertex_iterations
    assert dfp.affected_vertex_iterations <= df.affected_vertex_iterations


def test_partition_strategies_agree_bitwise(dp, oracle_lib):  # test_engine.cpp:232-253
    og2, ogt2, dels, ins, prev = batch_case(oracle_lib, 139, 150, 2500, 6, 0.8, 5)
    g2, gt2 = dev_pair(dp, og2, ogt2)
    res = []
    for s in dp.PartitionStrategy:
        cfg = dp.EngineConfig(partition_strategy=s, low_degree_threshold=8)
        res.append(dp.dynamic_frontier(g2, gt2, dels, ins, prev, cfg, pruning=True))
        ref = oracle_lib.dynamic_frontier(og2, ogt2, dels, ins, prev,
                                          oracle.default_config(partition_strategy=int(s),
                                                                low_degree_threshold=8), pruning=True)
        assert_same_result(res[-1], ref)
    assert np.array_equal(res[0].ranks, res[1].ranks) and np.array_equal(res[1].ranks, res[2].ranks)


def test_engines_are_deterministic(dp, oracle_lib):  # test_engine.cpp:255-271
    og2, ogt2, dels, ins, prev = batch_case(oracle_lib, 149, 200, 2000, 10, 0.8, 11)
    g2, gt2 = dev_pair(dp, og2, ogt2)
    a = dp.dynamic_frontier(g2, gt2, dels, ins, prev, pruning=True)
    b = dp.dynamic_frontier(g2, gt2, dels, ins, prev, pruning=True)
    assert np.array_equal(a.ranks, b.ranks) and a.affected_vertex_iterations == b.affected_vertex_iterations


def test_iteration_cap(dp, oracle_lib):  # test_engine.cpp:273-282
    og, ogt = rand_pair(oracle_lib, 151, 100, 600)
    g, gt = dev_pair(dp, og, ogt)
    r = dp.static_pagerank(gt, g, dp.EngineConfig(max_iterations=3))
    assert not r.converged and r.iterations == 3 and r.final_delta > 1e-10


def test_convergence_check_disabled_runs_max_iterations(dp, oracle_lib):  # harness.cpp:340-349
    og, ogt = rand_pair(oracle_lib, 5, 300, 2000)
    g, gt = dev_pair(dp, og, ogt)
    cfg = dp.EngineConfig(max_iterations=120, convergence_check_disabled=True)
    r = dp.static_pagerank(gt, g, cfg)
    ref = oracle_lib.static(ogt, og, oracle.default_config(max_iterations=120, convergence_check_disabled=1))
    assert r.iterations == 120 and not r.converged
    assert_same_result(r, ref)


def test_frontier_input_validation(dp, oracle_lib):
    og, ogt = rand_pair(oracle_lib, 5, 30, 90)
    g, gt = dev_pair(dp, og, ogt)
    prev = np.full(30, 1.0 / 30)
    with pytest.raises(ValueError, match="dynamicFrontier: previousRanks length mismatch"):
        dp.dynamic_frontier(g, gt, [], [], prev[:5])
    with pytest.raises(ValueError, match="initialAffected deletions: vertex id out of range"):
        dp.dynamic_frontier(g, gt, [(0, 99)], [], prev)
    with pytest.raises(ValueError, match="initialAffected insertions: vertex id out of range"):
        dp.dynamic_frontier(g, gt, [], [(99, 0)], prev)
    with pytest.raises(ValueError, match="flags length mismatch"):
        dp.dynamic_frontier_from_flags(g, gt, np.ones(3, np.uint8), np.zeros(3, np.uint8), prev)


@pytest.mark.parametrize("scale,frac", [(14, 1e-4), (16, 1e-3), (16, 1e-5)])
def test_rmat_static_and_dfp_bitwise(dp, oracle_lib, scale, frac):
    """RMAT (Graph500 a,b,c) Static + DF-P 80/20 batch, full parity."""
    src, dst = oracle_lib.rmat_edges(scale, 16 << scale)
    og = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), 1 << scale))
    ogt = oracle_lib.transpose(og)
    g, gt = dp.rmat_graph(scale), None
    gt = dp.transpose(g)
    base_ref = oracle_lib.static(ogt, og)
    base = dp.static_pagerank(gt, g)
    assert_same_result(base, base_ref)
    size = oracle_lib.batch_size_from_fraction(frac, og.m)
    dels, ins = oracle_lib.generate_random_batch(og, size, 0.8, oracle_lib.derive_seed(42, 0))
    og2, _, _ = oracle_lib.apply_batch(og, dels, ins)
    ogt2 = oracle_lib.transpose(og2)
    g2, gt2 = dp.apply_batch_pair(g, gt, dp.BatchUpdate(dels, ins))
    trace = []
    ref = oracle_lib.dynamic_frontier(og2, ogt2, dels, ins, base_ref.ranks, pruning=True, trace=trace)
    got = []
    d = dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=True,
                            observer=lambda it, r, f: got.append(f))
    assert_same_result(d, ref)
    for f, (_, _, rf) in zip(got, trace):
        assert np.array_equal(f, rf)


@pytest.mark.parametrize("scale,frac", [(14, 1e-3), (16, 1e-4)])
def test_kronecker_static_and_dfp_bitwise(dp, oracle_lib, scale, frac):
    """Graph500-style Kronecker graph (scrambled ids: hubs spread over the
    id space, so the degree relabel and the SELL slices mix ids unlike
    RMAT's) -- Static and DF-P bitwise vs the reference."""
    src, dst = oracle_lib.kronecker_edges(scale, 16 << scale, seed=5)
    og = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), 1 << scale))
    ogt = oracle_lib.transpose(og)
    g = dp.kronecker_graph(scale, seed=5)
    gt = dp.transpose(g)
    base_ref = oracle_lib.static(ogt, og)
    base = dp.static_pagerank(gt, g)
    assert_same_result(base, base_ref)
    size = oracle_lib.batch_size_from_fraction(frac, og.m)
    dels, ins = oracle_lib.generate_random_batch(og, size, 0.8, oracle_lib.derive_seed(5, 1))
    og2, _, _ = oracle_lib.apply_batch(og, dels, ins)
    ogt2 = oracle_lib.transpose(og2)
    dp.prepare(gt, g)
    g2, gt2 = dp.apply_batch_pair(g, gt, dp.BatchUpdate(dels, ins))
    ref = oracle_lib.dynamic_frontier(og2, ogt2, dels, ins, base_ref.ranks, pruning=True)
    assert_same_result(dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=True), ref)


# ---- dynamicTraversal / markReachable (engine.cpp:124-151, frontier.cpp:86-121) ----
@pytest.mark.parametrize("case", [(131, 400, 4000, 8, 0.8, 2024), (137, 300, 1200, 3, 1.0, 77),
                                  (139, 150, 2500, 6, 0.8, 5), (3, 20000, 200000, 200, 0.8, 9)])
def test_dynamic_traversal_bitwise_vs_reference(dp, oracle_lib, case):
    og2, ogt2, dels, ins, prev = batch_case(oracle_lib, *case)
    g, gt = dev_pair(dp, og2, ogt2)
    ref = oracle_lib.dynamic_traversal(og2, ogt2, dels, ins, prev)
    assert_same_result(dp.dynamic_traversal(g, gt, dels, ins, prev), ref)


def test_dynamic_traversal_on_rmat(dp, oracle_lib):
    O = oracle_lib
    src, dst = O.rmat_edges(14, 16 << 14)
    og = O.add_self_loops(O.build_csr((src, dst), 1 << 14))
    base = O.static(O.transpose(og), og)
    dels, ins = O.generate_random_batch(og, O.batch_size_from_fraction(1e-4, og.m), 0.8, 3)
    og2, _, _ = O.apply_batch(og, dels, ins)
    ogt2 = O.transpose(og2)
    g, gt = dev_pair(dp, og2, ogt2)
    ref = O.dynamic_traversal(og2, ogt2, dels, ins, base.ranks)
    assert_same_result(dp.dynamic_traversal(g, gt, dels, ins, base.ranks), ref)


def test_dynamic_traversal_errors_and_empty_batch(dp, oracle_lib):
    og, ogt = rand_pair(oracle_lib, 151, 50, 200)
    g, gt = dev_pair(dp, og, ogt)
    prev = np.full(50, 1.0 / 50)
    r = dp.dynamic_traversal(g, gt, [], [], prev)
    assert r.converged and r.iterations == 1 and r.affected_vertex_iterations == 0
    assert np.array_equal(r.ranks, prev)
    with pytest.raises(ValueError, match="dynamicTraversal: previousRanks length mismatch"):
        dp.dynamic_traversal(g, gt, [], [], [1.0])
    with pytest.raises(ValueError, match="markReachable: seed out of range"):
        dp.dynamic_traversal(g, gt, [], [(70, 1)], prev)


@pytest.mark.parametrize("seed,n,pairs,nseeds", [(157, 300, 900, 1), (163, 2000, 5000, 7), (167, 5000, 60000, 40)])
def test_mark_reachable_vs_reference(dp, oracle_lib, seed, n, pairs, nseeds):
    og, _ = rand_pair(oracle_lib, seed, n, pairs)
    g = to_dev(dp, og)
    seeds = np.random.default_rng(seed).integers(0, n, nseeds).astype(np.uint32)
    assert np.array_equal(dp.mark_reachable(g, seeds), oracle_lib.mark_reachable(og, seeds))
    assert not dp.mark_reachable(g, []).any()
    with pytest.raises(ValueError, match="markReachable: seed out of range"):
        dp.mark_reachable(g, [n])
