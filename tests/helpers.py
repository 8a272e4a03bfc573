"""Shared test helpers: move oracle graphs to the device and compare."""
import numpy as np


def to_dev(dp, g, ctx=None):
    """Upload an oracle-side CSR graph to the device (CsrGraph(n, off, tgt))."""
    off, tgt = g.csr()
    return dp.CsrGraph.from_csr(g.n, off, tgt, ctx=ctx)


def same_csr(dev_graph, oracle_graph) -> bool:
    off, tgt = oracle_graph.csr()
    return (dev_graph.vertex_count == oracle_graph.n and dev_graph.edge_count == oracle_graph.m
            and np.array_equal(dev_graph.offsets, off) and np.array_equal(dev_graph.targets, tgt))


def rand_pair(O, seed, n, pairs):
    rng = O.rng(seed)
    g = O.random_graph(rng, n, pairs)
    return g, O.transpose(g)


def dev_cfg(dp, oc):
    """oracle Config -> product EngineConfig."""
    return dp.EngineConfig(oc.damping_factor, oc.iteration_tolerance, oc.frontier_tolerance,
                           oc.prune_tolerance, oc.max_iterations, oc.low_degree_threshold,
                           dp.PartitionStrategy(oc.partition_strategy), bool(oc.convergence_check_disabled))
