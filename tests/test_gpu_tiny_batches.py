"""Tiny batches (1-200 edges) on an RMAT-16 graph -- the 1e-7..1e-5 |E| end
of BASELINE configs[1] at a size the reference solves in milliseconds: the
first sweeps touch a handful of vertices and the frontier reaches the hubs
after a few pushes.  DF and DF-P through the device loop (twice: the cached
loop graph) and the host-driven loop, both sweep kernels, the from-flags
entry point and a stream of single-edge batches, each equal to the
reference bit for bit (iterations, affected-vertex counts, final delta,
ranks)."""
import numpy as np
import pytest

from helpers import to_dev

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.iterations == b.iterations
    assert a.converged == b.converged
    assert a.affected_vertex_iterations == b.affected_vertex_iterations
    assert a.final_delta == b.final_delta
    assert np.array_equal(a.ranks, b.ranks)


def _rmat_pair(O, scale, seed):
    src, dst = O.rmat_edges(scale, 16 << scale, seed=seed)
    g = O.add_self_loops(O.build_csr((src, dst), 1 << scale))
    return g, O.transpose(g)


@pytest.fixture(scope="module")
def rmat16(oracle_lib):
    O = oracle_lib
    og, ogt = _rmat_pair(O, 16, 42)
    return og, ogt, O.static(ogt, og)


@pytest.mark.parametrize("sweep", ["fused", "split"])
@pytest.mark.parametrize("size,insf,bseed", [(1, 1.0, 3), (1, 0.0, 4), (2, 0.5, 5), (5, 0.8, 6), (20, 0.8, 7),
                                             (200, 0.8, 8)])
def test_tiny_batches_bitwise(dp, oracle_lib, monkeypatch, rmat16, sweep, size, insf, bseed):
    O = oracle_lib
    og, ogt, base = rmat16
    monkeypatch.setenv("DYNPR_SWEEP", sweep)
    dels, ins = O.generate_random_batch(og, size, insf, bseed)
    og2, _, _ = O.apply_batch(og, dels, ins)
    ogt2 = O.transpose(og2)
    g, gt = to_dev(dp, og2), to_dev(dp, ogt2)
    for pruning in (True, False):
        ref = O.dynamic_frontier(og2, ogt2, dels, ins, base.ranks, pruning=pruning)
        dev = dp.dynamic_frontier(g, gt, dels, ins, base.ranks, pruning=pruning)
        dev2 = dp.dynamic_frontier(g, gt, dels, ins, base.ranks, pruning=pruning)  # cached loop graph
        monkeypatch.setenv("DYNPR_HOST_LOOP", "1")
        host = dp.dynamic_frontier(g, gt, dels, ins, base.ranks, pruning=pruning)
        monkeypatch.delenv("DYNPR_HOST_LOOP")
        for r in (dev, dev2, host):
            _same(r, ref)


@pytest.mark.parametrize("sweep", ["fused", "split"])
def test_tiny_frontier_from_flags(dp, oracle_lib, monkeypatch, rmat16, sweep):
    """dynamicFrontierFromFlags with 1, 3 and 40 affected / pending vertices."""
    O = oracle_lib
    og, ogt, base = rmat16
    monkeypatch.setenv("DYNPR_SWEEP", sweep)
    n = og.n
    rng = np.random.default_rng(9)
    for k in (1, 3, 40):
        va = np.zeros(n, np.uint8)
        va[rng.choice(n, k, replace=False)] = 1
        pend = np.zeros(n, np.uint8)
        pend[rng.choice(n, k, replace=False)] = 1
        ref = O.dynamic_frontier_from_flags(og, ogt, va, pend, base.ranks, pruning=True)
        got = dp.dynamic_frontier_from_flags(dp_g(dp, og), dp_g(dp, ogt), va, pend, base.ranks, pruning=True)
        monkeypatch.setenv("DYNPR_HOST_LOOP", "1")
        host = dp.dynamic_frontier_from_flags(dp_g(dp, og), dp_g(dp, ogt), va, pend, base.ranks, pruning=True)
        monkeypatch.delenv("DYNPR_HOST_LOOP")
        _same(got, ref)
        _same(host, ref)


_cache = {}


def dp_g(dp, og):
    key = id(og)
    if key not in _cache:
        _cache[key] = to_dev(dp, og)
    return _cache[key]


def test_tiny_batch_stream(dp, oracle_lib, rmat16):
    """A stream of single-edge batches, each solved from the previous ranks
    (the temporal pattern): every solve equal to the reference."""
    O = oracle_lib
    og, ogt, base = rmat16
    ranks = base.ranks
    for k in range(6):
        dels, ins = O.generate_random_batch(og, 1 + (k % 3), 0.8, 100 + k)
        og2, _, _ = O.apply_batch(og, dels, ins)
        ogt2 = O.transpose(og2)
        ref = O.dynamic_frontier(og2, ogt2, dels, ins, ranks, pruning=True)
        got = dp.dynamic_frontier(to_dev(dp, og2), to_dev(dp, ogt2), dels, ins, ranks, pruning=True)
        _same(got, ref)
        og, ogt, ranks = og2, ogt2, ref.ranks
