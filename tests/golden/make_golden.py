"""Generate the golden vectors in this directory FROM THE REFERENCE ITSELF.

Runs the unmodified reference library (oracle/_ref/libdynpr_ref.so, built by
oracle/Makefile from /root/reference/proj/src) on seeded inputs and stores
inputs + outputs in reference_vectors.npz.  Only this container can run it
(/root/reference does not exist on the GPU box); the fixtures are committed.

    python tests/golden/make_golden.py

Inputs are drawn with the reference's own SplitMix64 / randomGraph
(oracles.hpp:80-89) and generateRandomBatch (workload.cpp:183-243); the
cases mirror the reference unit tests (test_graph/partition/rank/engine.cpp).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def main():
    R = oracle.Oracle("ref")
    R.set_threads(8)
    out = {}

    def put_graph(key, g):
        off, tgt = g.csr()
        out[key + "/n"] = np.array([g.n], np.uint64)
        out[key + "/off"] = off
        out[key + "/tgt"] = tgt

    # rng / seeds (rng.hpp)
    rng = R.rng(20240517)
    out["rng/bounded"] = np.array([rng.bounded(1000003) for _ in range(64)], np.uint64)
    out["rng/double"] = np.array([rng.next_double() for _ in range(64)])
    out["rng/derive"] = np.array([R.derive_seed(42, k) for k in range(16)], np.uint64)
    out["workload/batch_size"] = np.array(
        [R.batch_size_from_fraction(f, t) for f, t in [(1e-7, 17135093), (1e-4, 17135093), (1e-3, 4201682),
                                                       (0.5, 3), (1e-9, 10)]], np.uint64)

    # graphs: randomGraph, transpose, applyBatch (test_graph.cpp:99-121 shape)
    rng = R.rng(99)
    for i in range(8):
        g = R.random_graph(rng, 30 + 10 * i, 150 + 40 * i)
        put_graph(f"graph{i}/g", g)
        put_graph(f"graph{i}/gt", R.transpose(g))
        dels, ins = R.generate_random_batch(g, 12, 0.75, R.derive_seed(7, i))
        # add an absent deletion and repeated entries to exercise the tallies
        dels = (np.append(dels[0], [dels[0][0]]), np.append(dels[1], [dels[1][0]]))
        g2, miss, dup = R.apply_batch(g, dels, (np.append(ins[0], ins[0][:1]), np.append(ins[1], ins[1][:1])))
        out[f"graph{i}/dels"] = np.stack(dels).astype(np.uint32)
        out[f"graph{i}/ins"] = np.stack((np.append(ins[0], ins[0][:1]), np.append(ins[1], ins[1][:1]))).astype(
            np.uint32)
        put_graph(f"graph{i}/applied", g2)
        out[f"graph{i}/stats"] = np.array([miss, dup], np.uint64)
        order, low = R.partition(g, 3 + i)
        out[f"graph{i}/partition_order"] = order
        out[f"graph{i}/partition_low"] = np.array([low, 3 + i], np.uint64)

    # buildCsr + addSelfLoops from a raw edge list (rmat generator edges)
    src, dst = R.rmat_edges(10, 16 << 10)
    out["rmat10/src"], out["rmat10/dst"] = src, dst
    gr = R.build_csr((src, dst), 1 << 10)
    put_graph("rmat10/raw", gr)
    g = R.add_self_loops(gr)
    gt = R.transpose(g)
    put_graph("rmat10/g", g)
    st = R.static(gt, g)
    out["rmat10/static_ranks"] = st.ranks
    out["rmat10/static_meta"] = np.array([st.iterations, st.affected_vertex_iterations, st.converged])
    out["rmat10/static_delta"] = np.array([st.final_delta])
    dels, ins = R.generate_random_batch(g, R.batch_size_from_fraction(1e-3, g.m), 0.8, R.derive_seed(42, 0))
    out["rmat10/dels"] = np.stack(dels)
    out["rmat10/ins"] = np.stack(ins)
    g2, _, _ = R.apply_batch(g, dels, ins)
    gt2 = R.transpose(g2)
    put_graph("rmat10/g2", g2)
    for pruning in (0, 1):
        trace = []
        d = R.dynamic_frontier(g2, gt2, dels, ins, st.ranks, pruning=bool(pruning), trace=trace)
        d2 = R.dynamic_frontier(g2, gt2, dels, ins, st.ranks, pruning=bool(pruning))
        assert np.array_equal(d.ranks, d2.ranks) and d.iterations == d2.iterations  # replay == library
        out[f"rmat10/df{pruning}_ranks"] = d.ranks
        out[f"rmat10/df{pruning}_meta"] = np.array([d.iterations, d.affected_vertex_iterations, d.converged])
        out[f"rmat10/df{pruning}_processed"] = np.stack([f for _, _, f in trace]).astype(np.uint8)

    # updateRanks single sweeps on a hub-heavy graph (every accumulation path)
    nrng = np.random.default_rng(5)
    n = 1500
    s = np.concatenate([nrng.integers(0, n, 9000), nrng.integers(0, n, 1500)]).astype(np.uint32)
    d_ = np.concatenate([nrng.integers(0, n, 9000), nrng.integers(0, 3, 1500)]).astype(np.uint32)
    g = R.add_self_loops(R.build_csr((s, d_), n))
    gt = R.transpose(g)
    put_graph("sweep/g", g)
    prev = nrng.random(n) / n
    va = (nrng.random(n) < 0.6).astype(np.uint8)
    npd = (nrng.random(n) < 0.1).astype(np.uint8)
    out["sweep/prev"], out["sweep/va"], out["sweep/np"] = prev, va, npd
    for thr in (4, 32, 300):
        for mode in (0, 1):
            cfg = oracle.default_config(low_degree_threshold=thr, frontier_tolerance=0.05, prune_tolerance=0.02)
            cur, v2, n2 = R.update_ranks(gt, g, va, npd, prev, np.zeros(n), cfg, mode)
            out[f"sweep/t{thr}m{mode}_cur"], out[f"sweep/t{thr}m{mode}_va"], out[f"sweep/t{thr}m{mode}_np"] = cur, v2, n2
            full, _, _ = R.update_ranks(gt, g, None, None, prev, np.zeros(n), cfg, mode)
            out[f"sweep/t{thr}m{mode}_full"] = full
    # norms
    a, b = nrng.random(10007), nrng.random(10007)
    out["norm/a"], out["norm/b"] = a, b
    out["norm/linf_l1"] = np.array([R.linf(a, b), R.l1(a, b)])

    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
