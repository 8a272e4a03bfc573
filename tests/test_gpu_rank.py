"""Rank update, norms, partition and frontier primitives on the device.

Known answers restate proj/tests/unit/test_rank.cpp, test_partition.cpp and
test_frontier.cpp; random cases are compared bit for bit with the oracle.
"""
import numpy as np
import pytest

import oracle
from helpers import rand_pair, to_dev

pytestmark = pytest.mark.gpu


def pair(dp, edges, n):
    g = dp.add_self_loops(dp.build_csr(edges, n))
    return g, dp.transpose(g)


def test_single_self_looped_vertex_is_a_fixed_point(dp):  # test_rank.cpp:37-44
    g, gt = pair(dp, [], 1)
    cur, _, _ = dp.update_ranks(gt, g, [1.0])
    assert abs(cur[0] - 1.0) <= 1e-15


def test_two_cycle_converges_to_equal_ranks(dp):  # test_rank.cpp:46-53
    g, gt = pair(dp, [(0, 1), (1, 0)], 2)
    r = dp.static_pagerank(gt, g)
    assert r.converged
    assert np.allclose(r.ranks, [0.5, 0.5], atol=1e-12)


def test_closed_loop_evaluation_at_the_fixed_point_is_identity(dp):  # test_rank.cpp:55-69
    g, gt = pair(dp, [(1, 0), (2, 0), (3, 0)], 4)
    fixed = oracle.dense_pagerank(g.offsets, g.targets, 4, 0.85, 1e-14, 10000)
    cur, _, _ = dp.update_ranks(gt, g, fixed, vertex_affected=np.ones(4, np.uint8),
                                neighbors_pending=np.zeros(4, np.uint8), mode=dp.RankMode.CLOSED_LOOP_PRUNE)
    assert np.max(np.abs(cur - fixed)) <= 1e-10


def test_unaffected_vertices_copy_through_bitwise(dp, oracle_lib):  # test_rank.cpp:71-83
    rng = oracle_lib.rng(31)
    og = oracle_lib.random_graph(rng, 20, 60)
    g = to_dev(dp, og)
    gt = dp.transpose(g)
    prev = np.full(20, 1.0 / 20)
    for i in range(20):
        prev[i] *= 1.0 + 0.1 * rng.next_double()
    va = np.zeros(20, np.uint8)
    va[::2] = 1
    cur, _, _ = dp.update_ranks(gt, g, prev, vertex_affected=va, neighbors_pending=np.zeros(20, np.uint8))
    assert np.array_equal(cur[1::2], prev[1::2])


@pytest.mark.parametrize("tf,tp,mode,r1,np1,va1", [
    (0.29, 1e-6, 0, 0.7125, 1, 1),
    (0.30, 1e-6, 0, None, 0, None),
    (10.0, 10.0, 1, None, 0, 0),
    (1e-9, 1e-9, 1, None, 1, 1),
])
def test_frontier_and_prune_flags_follow_the_relative_delta(dp, tf, tp, mode, r1, np1, va1):
    # test_rank.cpp:85-126
    g, gt = pair(dp, [(0, 1)], 2)
    cfg = dp.EngineConfig(frontier_tolerance=tf, prune_tolerance=tp)
    cur, va, np_ = dp.update_ranks(gt, g, [0.5, 0.5], vertex_affected=np.ones(2, np.uint8),
                                   neighbors_pending=np.zeros(2, np.uint8), config=cfg, mode=mode)
    if r1 is not None:
        assert abs(cur[1] - r1) <= 1e-12 * r1
    assert np_[1] == np1
    if va1 is not None:
        assert va[1] == va1


def test_linf_norm_delta(dp, port):  # test_rank.cpp:128-146
    assert abs(dp.linf_norm_delta([0.1, 0.4], [0.2, 0.25]) - 0.15) <= 1e-15
    assert dp.linf_norm_delta([0.3, 0.7], [0.3, 0.7]) == 0.0
    rng = port.rng(41)
    a = np.array([rng.next_double() for _ in range(10000)])
    b = np.array([rng.next_double() for _ in range(10000)])
    assert dp.linf_norm_delta(a, b) == np.max(np.abs(a - b))
    with pytest.raises(ValueError):
        dp.linf_norm_delta(a, [1.0])


def test_l1_norm_delta_is_bit_exact(dp, oracle_lib, port):  # test_rank.cpp:148-165
    assert abs(dp.l1_norm_delta([0.1, 0.4], [0.2, 0.25]) - 0.25) <= 1e-15
    rng = port.rng(43)
    a = np.array([rng.next_double() for _ in range(10000)])
    b = np.array([rng.next_double() for _ in range(10000)])
    assert dp.l1_norm_delta(a, b) == oracle_lib.l1(a, b)
    big = np.random.default_rng(0).random(300001)
    assert dp.l1_norm_delta(big, big[::-1].copy()) == oracle_lib.l1(big, big[::-1].copy())


def test_full_plain_sweeps_conserve_the_rank_sum(dp, oracle_lib):  # test_rank.cpp:167-180
    g, gt = rand_pair(oracle_lib, 47, 200, 900)
    dg, dgt = to_dev(dp, g), to_dev(dp, gt)
    prev = np.full(200, 1.0 / 200)
    for _ in range(30):
        cur, _, _ = dp.update_ranks(dgt, dg, prev)
        assert abs(cur.sum() - 1.0) <= 1e-9
        prev = cur


@pytest.mark.parametrize("threshold", [0, 4, 32, 300])
@pytest.mark.parametrize("mode", [0, 1])
def test_update_ranks_bitwise_vs_reference(dp, oracle_lib, threshold, mode):
    """Every flat / chunked accumulation path, with and without flags."""
    rng = np.random.default_rng(threshold * 7 + mode)
    n = 3000
    # a hub-heavy graph so in-degrees cross 32, 256 and 512
    src = np.concatenate([rng.integers(0, n, 20000), rng.integers(0, n, 4000)]).astype(np.uint32)
    dst = np.concatenate([rng.integers(0, n, 20000), rng.integers(0, 6, 4000)]).astype(np.uint32)
    og = oracle_lib.add_self_loops(oracle_lib.build_csr((src, dst), n))
    ogt = oracle_lib.transpose(og)
    assert ogt.degrees().max() > 512
    g, gt = to_dev(dp, og), to_dev(dp, ogt)
    prev = rng.random(n) / n
    cfg = oracle.default_config(low_degree_threshold=threshold, frontier_tolerance=0.05, prune_tolerance=0.01)
    dcfg = dp.EngineConfig(low_degree_threshold=threshold, frontier_tolerance=0.05, prune_tolerance=0.01)
    # full sweep
    ref, _, _ = oracle_lib.update_ranks(ogt, og, None, None, prev, np.zeros(n), cfg, mode)
    cur, _, _ = dp.update_ranks(gt, g, prev, config=dcfg, mode=mode)
    assert np.array_equal(cur, ref)
    # flagged sweep
    va0 = (rng.random(n) < 0.5).astype(np.uint8)
    np0 = (rng.random(n) < 0.1).astype(np.uint8)
    ref, rva, rnp = oracle_lib.update_ranks(ogt, og, va0, np0, prev, np.zeros(n), cfg, mode)
    cur, va, np_ = dp.update_ranks(gt, g, prev, vertex_affected=va0, neighbors_pending=np0, config=dcfg,
                                   mode=mode)
    assert np.array_equal(cur, ref)
    assert np.array_equal(va, rva) and np.array_equal(np_, rnp)


def test_partition_known_answer(dp):  # test_partition.cpp:23-39
    edges = [(v, t) for v, d in enumerate([1, 40, 2, 33, 3]) for t in range(d)]
    g = dp.build_csr(edges, 41)
    p = dp.partition_by_degree(g, 32)
    assert p.low_count == 39
    assert p.order[:4].tolist() == [0, 2, 4, 5]
    assert p.order[39:].tolist() == [1, 3]


def test_partition_identity_and_empty(dp):  # test_partition.cpp:41-61
    g = dp.build_csr([(v, t) for v, d in enumerate([1, 2, 1, 2]) for t in range(d)], 4)
    p = dp.partition_by_degree(g, 32)
    assert p.low_count == 4 and p.order.tolist() == [0, 1, 2, 3]
    p = dp.partition_by_degree(dp.build_csr([], 0), 32)
    assert p.low_count == 0 and len(p.order) == 0


def test_partition_matches_reference(dp, oracle_lib):  # test_partition.cpp:63-92
    rng = oracle_lib.rng(17)
    for _ in range(50):
        n = 1 + rng.bounded(200)
        og = oracle_lib.random_graph(rng, n, 4 * n)
        thr = rng.bounded(12)
        order, low = oracle_lib.partition(og, thr)
        p = dp.partition_by_degree(to_dev(dp, og), thr)
        assert p.low_count == low and np.array_equal(p.order, order)
    og = oracle_lib.random_graph(oracle_lib.rng(23), 200000, 1200000)
    for thr in (0, 8, 32):
        order, low = oracle_lib.partition(og, thr)
        p = dp.partition_by_degree(to_dev(dp, og), thr)
        assert p.low_count == low and np.array_equal(p.order, order)


def test_initial_affected(dp):  # test_frontier.cpp:23-47
    g, _ = pair(dp, [], 6)
    va, np_ = dp.initial_affected(g, [(1, 2)], [(3, 4)])
    assert np.flatnonzero(np_).tolist() == [1, 3] and np.flatnonzero(va).tolist() == [2]
    g4, _ = pair(dp, [], 4)
    va, np_ = dp.initial_affected(g4, [], [])
    assert not va.any() and not np_.any()
    va, np_ = dp.initial_affected(g4, [(0, 1), (0, 2)], [])
    assert np.flatnonzero(np_).tolist() == [0] and np.flatnonzero(va).tolist() == [1, 2]
    g3, _ = pair(dp, [], 3)
    with pytest.raises(ValueError, match="initialAffected deletions: vertex id out of range"):
        dp.initial_affected(g3, [(0, 9)], [])


def test_expand_affected_known_answers(dp):  # test_frontier.cpp:49-65
    g, _ = pair(dp, [(1, 2), (1, 5)], 6)
    np_ = np.zeros(6, np.uint8)
    np_[1] = 1
    va = dp.expand_affected(g, np.zeros(6, np.uint8), np_)
    assert np.flatnonzero(va).tolist() == [1, 2, 5]
    g2, _ = pair(dp, [(0, 1)], 2)
    va = dp.expand_affected(g2, np.array([1, 0], np.uint8), np.zeros(2, np.uint8))
    assert np.flatnonzero(va).tolist() == [0]


def test_expand_affected_matches_reference(dp, oracle_lib):  # test_frontier.cpp:67-101
    rng = oracle_lib.rng(7)
    for _ in range(30):
        n = 2 + rng.bounded(60)
        og = oracle_lib.random_graph(rng, n, 4 * n)
        va0 = np.array([rng.bounded(4) == 0 for _ in range(n)], np.uint8)
        np0 = np.array([rng.bounded(4) == 0 for _ in range(n)], np.uint8)
        ref = oracle_lib.expand_affected(og, va0, np0)
        g = to_dev(dp, og)
        for thr in (0, 4, 32):
            assert np.array_equal(dp.expand_affected(g, va0, np0, thr), ref)
