"""In-sweep pull (sweep.cuh SweepArgs::pull_fused): with either sweep kernel
(split or fused latency mode) the device loop folds a pull-mode
expandAffected (frontier.cpp:55-84) into the next sweep -- pending flags ride in the contributions' sign bits,
unaffected vertices gather their in-lists and become affected when one
source is pending.  Compared bit for bit with the separate pull kernels
(DYNPR_PULL_FUSED=0), the host-driven loop and the reference library, on
RMAT graphs whose hubs exercise the multi-chunk path (partials carrying the
sign bit, warp-combined vertices above 32 chunks) and on batches large
enough that the loop picks pull."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.iterations == b.iterations
    assert a.converged == b.converged
    assert a.affected_vertex_iterations == b.affected_vertex_iterations
    assert a.final_delta == b.final_delta
    assert np.array_equal(a.ranks, b.ranks)


@pytest.fixture(scope="module")
def rmat16(dp, oracle_lib):
    O = oracle_lib
    src, dst = O.rmat_edges(16, 16 << 16)
    og = O.add_self_loops(O.build_csr((src, dst), 1 << 16))
    ogt = O.transpose(og)
    g = dp.rmat_graph(16)
    gt = dp.transpose(g)
    return og, ogt, g, gt, O.static(ogt, og)


@pytest.mark.parametrize("sweep", ["split", "fused"])
@pytest.mark.parametrize("frac", [1e-4, 1e-3, 1e-2, 0.1])
@pytest.mark.parametrize("pruning", [True, False])
def test_in_sweep_pull_matches_reference(dp, oracle_lib, monkeypatch, rmat16, frac, pruning, sweep):
    O = oracle_lib
    og, ogt, g, gt, base = rmat16
    size = O.batch_size_from_fraction(frac, og.m)
    dels, ins = O.generate_random_batch(og, size, 0.8, O.derive_seed(7, int(frac * 1e6)))
    og2, _, _ = O.apply_batch(og, dels, ins)
    ogt2 = O.transpose(og2)
    g2, gt2 = dp.apply_batch_pair(g, gt, dp.BatchUpdate(dels, ins))
    ref = O.dynamic_frontier(og2, ogt2, dels, ins, base.ranks, pruning=pruning)
    monkeypatch.setenv("DYNPR_SWEEP", sweep)
    runs = {}
    # DYNPR_LAZY_LISTS=0: pull sweeps append the push lists anyway (default:
    # they are collected from the sign bits when a push follows a pull)
    for mode, env in (("fused", {"DYNPR_HOST_LOOP": "0", "DYNPR_PULL_FUSED": "1"}),
                      ("fused-eager-lists", {"DYNPR_HOST_LOOP": "0", "DYNPR_LAZY_LISTS": "0"}),
                      ("separate", {"DYNPR_HOST_LOOP": "0", "DYNPR_PULL_FUSED": "0"}),
                      ("host", {"DYNPR_HOST_LOOP": "1"})):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        runs[mode] = dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=pruning)
        monkeypatch.delenv("DYNPR_PULL_FUSED", raising=False)
        monkeypatch.delenv("DYNPR_LAZY_LISTS", raising=False)
    for r in runs.values():
        _same(r, ref)
    # a second solve on the same context (stale sign bits in the reused
    # contribution buffers must not leak into the next solve)
    monkeypatch.setenv("DYNPR_HOST_LOOP", "0")
    _same(dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=pruning), ref)
    _same(dp.static_pagerank(gt2, g2), O.static(ogt2, og2))


@pytest.mark.parametrize("sweep", ["split", "fused"])
@pytest.mark.parametrize("threshold", [0, 40, 1000])
def test_in_sweep_pull_thresholds(dp, oracle_lib, monkeypatch, rmat16, threshold, sweep):
    """lowDegreeThreshold moves vertices between the flat single slices and
    the 256-chunk multi path (and the push lists between low / high)."""
    import oracle
    O = oracle_lib
    og, ogt, g, gt, _ = rmat16
    ocfg = oracle.default_config(low_degree_threshold=threshold)
    cfg = dp.EngineConfig(low_degree_threshold=threshold)
    base = O.static(ogt, og, ocfg)
    size = O.batch_size_from_fraction(3e-3, og.m)
    dels, ins = O.generate_random_batch(og, size, 0.8, 99)
    og2, _, _ = O.apply_batch(og, dels, ins)
    ogt2 = O.transpose(og2)
    g2, gt2 = dp.apply_batch_pair(g, gt, dp.BatchUpdate(dels, ins))
    monkeypatch.setenv("DYNPR_SWEEP", sweep)
    monkeypatch.setenv("DYNPR_HOST_LOOP", "0")
    for pruning in (True, False):
        ref = O.dynamic_frontier(og2, ogt2, dels, ins, base.ranks, ocfg, pruning=pruning)
        _same(dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, cfg, pruning), ref)
