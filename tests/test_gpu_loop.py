"""The device-driven convergence loop (cached CUDA graph with a WHILE node,
engine.cu run_device_loop) against the host-driven loop and the reference:
same iterations, affected-vertex counts, converged flag, final delta and
ranks, bit for bit, for every engine, both sweep kernels (fused latency
mode / split throughput mode), odd and even iteration counts and the
max-iterations / check-disabled exits."""
import numpy as np
import pytest

from helpers import rand_pair, to_dev

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.iterations == b.iterations
    assert a.converged == b.converged
    assert a.affected_vertex_iterations == b.affected_vertex_iterations
    assert a.final_delta == b.final_delta
    assert np.array_equal(a.ranks, b.ranks)


def _both(monkeypatch, fn):
    monkeypatch.setenv("DYNPR_HOST_LOOP", "1")
    host = fn()
    monkeypatch.setenv("DYNPR_HOST_LOOP", "0")
    dev = fn()
    dev2 = fn()  # cached graph reused
    _same(dev, host)
    _same(dev2, host)
    return dev


@pytest.mark.parametrize("sweep", ["fused", "split"])
@pytest.mark.parametrize("case", [(5, 3000, 40000, 60, 0.8, 3), (17, 20000, 300000, 2000, 0.8, 4),
                                  (23, 800, 9000, 5, 1.0, 8)])
def test_device_loop_all_engines(dp, oracle_lib, monkeypatch, sweep, case):
    monkeypatch.setenv("DYNPR_SWEEP", sweep)
    O = oracle_lib
    seed, n, pairs, size, insf, bseed = case
    og, ogt = rand_pair(O, seed, n, pairs)
    base = O.static(ogt, og)
    dels, ins = O.generate_random_batch(og, size, insf, bseed)
    og2, _, _ = O.apply_batch(og, dels, ins)
    ogt2 = O.transpose(og2)
    g, gt = to_dev(dp, og2), to_dev(dp, ogt2)
    _same(_both(monkeypatch, lambda: dp.static_pagerank(gt, g)), O.static(ogt2, og2))
    _same(_both(monkeypatch, lambda: dp.naive_dynamic(gt, g, base.ranks)), O.naive_dynamic(ogt2, og2, base.ranks))
    for pruning in (False, True):
        _same(_both(monkeypatch, lambda: dp.dynamic_frontier(g, gt, dels, ins, base.ranks, pruning=pruning)),
              O.dynamic_frontier(og2, ogt2, dels, ins, base.ranks, pruning=pruning))
    _same(_both(monkeypatch, lambda: dp.dynamic_traversal(g, gt, dels, ins, base.ranks)),
          O.dynamic_traversal(og2, ogt2, dels, ins, base.ranks))


@pytest.mark.parametrize("max_it", [1, 2, 3, 7, 8])
@pytest.mark.parametrize("check_disabled", [False, True])
def test_device_loop_iteration_limits(dp, oracle_lib, monkeypatch, max_it, check_disabled):
    O = oracle_lib
    og, ogt = rand_pair(O, 41, 2000, 20000)
    g, gt = to_dev(dp, og), to_dev(dp, ogt)
    cfg = dp.EngineConfig(max_iterations=max_it, convergence_check_disabled=check_disabled)
    import oracle
    ocfg = oracle.default_config(max_iterations=max_it, convergence_check_disabled=int(check_disabled))
    r = _both(monkeypatch, lambda: dp.static_pagerank(gt, g, cfg))
    assert r.iterations == max_it and not r.converged
    _same(r, O.static(ogt, og, ocfg))
    dels, ins = O.generate_random_batch(og, 40, 0.8, 6)
    og2, _, _ = O.apply_batch(og, dels, ins)
    ogt2 = O.transpose(og2)
    g2, gt2 = to_dev(dp, og2), to_dev(dp, ogt2)
    prev = O.static(ogt, og).ranks
    d = _both(monkeypatch, lambda: dp.dynamic_frontier(g2, gt2, dels, ins, prev, cfg, True))
    _same(d, O.dynamic_frontier(og2, ogt2, dels, ins, prev, ocfg, pruning=True))


def test_device_loop_converges_on_odd_and_even_iterations(dp, oracle_lib, monkeypatch):
    """Tolerances chosen so the solve stops in the even and in the odd half
    of the two-iteration graph body."""
    O = oracle_lib
    og, ogt = rand_pair(O, 43, 1500, 15000)
    g, gt = to_dev(dp, og), to_dev(dp, ogt)
    seen = set()
    import oracle
    for tol in (1e-4, 3e-5, 1e-5, 3e-6, 1e-6, 1e-8):
        r = _both(monkeypatch, lambda: dp.static_pagerank(gt, g, dp.EngineConfig(iteration_tolerance=tol)))
        _same(r, O.static(ogt, og, oracle.default_config(iteration_tolerance=tol)))
        seen.add(r.iterations % 2)
    assert seen == {0, 1}


def test_device_resident_arrays(dp, oracle_lib):
    """previous_ranks / out as CUDA tensors (__cuda_array_interface__):
    same results as host arrays, no host round trip of the rank vectors."""
    import torch
    O = oracle_lib
    og, ogt = rand_pair(O, 51, 3000, 30000)
    dels, ins = O.generate_random_batch(og, 30, 0.8, 2)
    og2, _, _ = O.apply_batch(og, dels, ins)
    g, gt = to_dev(dp, og), to_dev(dp, ogt)
    g2, gt2 = to_dev(dp, og2), to_dev(dp, O.transpose(og2))
    base = dp.static_pagerank(gt, g)
    out = torch.empty(3000, dtype=torch.float64, device="cuda")
    b2 = dp.static_pagerank(gt, g, out=out)
    assert b2.ranks.data_ptr() == out.data_ptr() and np.array_equal(out.cpu().numpy(), base.ranks)
    host = dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, pruning=True)
    out2 = torch.empty_like(out)
    dev = dp.dynamic_frontier(g2, gt2, dels, ins, out, pruning=True, out=out2)
    _same(type(host)(out2.cpu().numpy(), dev.iterations, dev.affected_vertex_iterations, dev.converged,
                     dev.final_delta), host)
    nd = dp.naive_dynamic(gt2, g2, out, out=out2)
    assert np.array_equal(out2.cpu().numpy(), dp.naive_dynamic(gt2, g2, base.ranks).ranks)
    with pytest.raises(ValueError, match="dtype float64"):
        dp.naive_dynamic(gt2, g2, out.float())
    with pytest.raises(ValueError, match="exactly vertex_count"):
        dp.static_pagerank(gt, g, out=out[:10])


@pytest.mark.parametrize("threshold", [0, 1, 300, 1000])
@pytest.mark.parametrize("sweep", ["fused", "split"])
def test_engines_any_low_degree_threshold(dp, oracle_lib, monkeypatch, threshold, sweep):
    """lowDegreeThreshold moves the flat / 256-chunk accumulation boundary
    (rank.cpp:42-75: flat when in-degree <= T) and the expansion split; every
    value must stay bitwise, including T > 256 (single segments longer than a
    chunk) on an RMAT graph whose hubs exceed T."""
    import oracle
    monkeypatch.setenv("DYNPR_SWEEP", sweep)
    O = oracle_lib
    src, dst = O.rmat_edges(13, 16 << 13)
    og = O.add_self_loops(O.build_csr((src, dst), 1 << 13))
    ogt = O.transpose(og)
    ocfg = oracle.default_config(low_degree_threshold=threshold)
    cfg = dp.EngineConfig(low_degree_threshold=threshold)
    base = O.static(ogt, og, ocfg)
    dels, ins = O.generate_random_batch(og, 120, 0.8, 3)
    og2, _, _ = O.apply_batch(og, dels, ins)
    ogt2 = O.transpose(og2)
    g2, gt2 = to_dev(dp, og2), to_dev(dp, ogt2)
    _same(dp.static_pagerank(gt2, g2, cfg), O.static(ogt2, og2, ocfg))
    _same(dp.dynamic_frontier(g2, gt2, dels, ins, base.ranks, cfg, True),
          O.dynamic_frontier(og2, ogt2, dels, ins, base.ranks, ocfg, pruning=True))


def test_concurrent_contexts_device_loops(dp, oracle_lib):
    """Independent contexts solving on separate host threads (reference
    SPEC: distinct instances on distinct graphs may run concurrently): the
    device loop's constant-bank argument slots are serialised per device, and
    every result stays bitwise."""
    import threading
    O = oracle_lib
    cases = []
    for seed in (61, 62, 63, 64):
        og, ogt = rand_pair(O, seed, 3000, 30000)
        cases.append((og, ogt, O.static(ogt, og)))
    out = [None] * len(cases)
    errors = []

    def work(i):
        try:
            ctx = dp.Context(0)
            og, ogt, _ = cases[i]
            g = dp.CsrGraph.from_csr(og.n, *og.csr(), ctx=ctx)
            gt = dp.CsrGraph.from_csr(ogt.n, *ogt.csr(), ctx=ctx)
            out[i] = [dp.static_pagerank(gt, g) for _ in range(3)]
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (og, ogt, ref), res in zip(cases, out):
        for r in res:
            _same(r, ref)


def _loop_trace(n_it):
    import ctypes as C
    from paper_2404_08299_b200 import _native as N
    cnt = C.c_uint64()
    N.lib().dynpr_debug_loop_trace(None, 0, C.byref(cnt))
    buf = np.zeros(cnt.value, np.uint64)
    N.lib().dynpr_debug_loop_trace(buf.ctypes.data, cnt.value, None)
    return buf.reshape(-1, 4)[:n_it]


def test_dfp_end_game_accounts_the_empty_iteration(dp, oracle_lib, monkeypatch):
    """DF-P on a split plan: when a sweep leaves nothing pending and nothing
    affected, the device loop accounts the next (empty) iteration without
    its sweep (engine.cu end_check).  Same counts, delta and ranks as the
    host loop, which runs that sweep, and as the reference; also with
    max_iterations cutting the loop right before and at that iteration."""
    import oracle
    O = oracle_lib
    monkeypatch.setenv("DYNPR_SWEEP", "split")
    src, dst = O.rmat_edges(16, 16 << 16)
    og = O.add_self_loops(O.build_csr((src, dst), 1 << 16))
    ogt = O.transpose(og)
    g0 = dp.rmat_graph(16)
    gt0 = dp.transpose(g0)
    base = O.static(ogt, og)
    empty_ends = 0
    for k, frac in enumerate((1e-5, 1e-4, 1e-3, 1e-4, 1e-5, 1e-3)):
        size = O.batch_size_from_fraction(frac, og.m)
        dels, ins = O.generate_random_batch(og, size, 0.8, O.derive_seed(5, k))
        og2, _, _ = O.apply_batch(og, dels, ins)
        ogt2 = O.transpose(og2)
        g, gt = dp.apply_batch_pair(g0, gt0, dp.BatchUpdate(dels, ins))
        ref = O.dynamic_frontier(og2, ogt2, dels, ins, base.ranks, pruning=True)
        dev = _both(monkeypatch, lambda: dp.dynamic_frontier(g, gt, dels, ins, base.ranks, pruning=True))
        _same(dev, ref)
        t = _loop_trace(dev.iterations)
        if dev.iterations > 1 and t[-1][1] == 0 and t[-1][2] == 0:
            empty_ends += 1
            for cut in (dev.iterations - 1, dev.iterations):
                ocfg = oracle.default_config(max_iterations=cut)
                cfg = dp.EngineConfig(max_iterations=cut)
                r = O.dynamic_frontier(og2, ogt2, dels, ins, base.ranks, ocfg, pruning=True)
                _same(_both(monkeypatch, lambda: dp.dynamic_frontier(g, gt, dels, ins, base.ranks, cfg, True)), r)
    assert empty_ends > 0, "no case ended with an empty iteration"
