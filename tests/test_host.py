"""CPU tests of the boundary: the C-ABI library loads and exports every
symbol include/dynpr_cuda.h declares, and the host-side mirror of the
reference interface behaves like module.cpp without touching a GPU."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2404_08299_b200 as dp
from paper_2404_08299_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_every_header_symbol():
    L = N.lib()
    syms = N.header_symbols()
    assert len(syms) >= 29
    missing = [s for s in syms if not hasattr(L, s)]
    assert missing == []
    # the ctypes prototype table covers the header exactly
    assert sorted(N.PROTOTYPES) == syms


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_and_validation_without_gpu():
    c = N.Config()
    N.lib().dynpr_config_default(C.byref(c))
    assert (c.damping_factor, c.iteration_tolerance, c.frontier_tolerance, c.prune_tolerance,
            c.max_iterations, c.low_degree_threshold, c.partition_strategy) == (0.85, 1e-10, 1e-6, 1e-6, 500,
                                                                                 32, 2)
    cfg = dp.EngineConfig()
    assert cfg._c().damping_factor == c.damping_factor
    cfg.validate()
    for bad, msg in [(dict(damping_factor=1.0), "dampingFactor"), (dict(iteration_tolerance=0.0), "iterationTol"),
                     (dict(frontier_tolerance=-1.0), "tolerances"), (dict(max_iterations=0), "maxIterations")]:
        with pytest.raises(ValueError, match=msg):
            dp.EngineConfig(**bad).validate()


def test_edge_list_parsing():
    s, d = dp._edges([(0, 1), (2, 3)])
    assert s.tolist() == [0, 2] and d.tolist() == [1, 3] and s.dtype == np.uint32
    s, d = dp._edges(np.array([[4, 5]]))
    assert s.tolist() == [4] and d.tolist() == [5]
    s, d = dp._edges((np.array([1, 2]), np.array([3, 4])))
    assert s.tolist() == [1, 2]
    assert len(dp._edges([])[0]) == 0
    with pytest.raises(ValueError):
        dp._edges([(-1, 0)])


def test_no_cpu_fallback_without_a_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        dp.Context(0)


def test_compat_library_exports_the_reference_api():
    """libdynpr_compat.so defines the reference's out-of-line dynpr:: symbols
    (graph/partition/rank/frontier/engine/workload/harness .hpp), so code
    compiled against the reference headers links against it unchanged."""
    import shutil
    import subprocess
    lib = os.path.join(ROOT, "paper_2404_08299_b200", "libdynpr_compat.so")
    if not os.path.exists(lib) or not shutil.which("nm"):
        pytest.skip("compat library not built here")
    syms = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True).stdout
    for name in ["dynpr::CsrGraph::CsrGraph(", "dynpr::CsrGraph::hasEdge(", "dynpr::buildCsr(", "dynpr::transpose(",
                 "dynpr::addSelfLoops(", "dynpr::applyBatch(", "dynpr::partitionByDegree(",
                 "dynpr::EngineConfig::validate(", "dynpr::initRanksUniform(", "dynpr::initRanksFrom(",
                 "dynpr::updateRanks(", "dynpr::linfNormDelta(", "dynpr::l1NormDelta(", "dynpr::initialAffected(",
                 "dynpr::expandAffected(", "dynpr::markReachable(", "dynpr::staticPageRank(",
                 "dynpr::naiveDynamic(", "dynpr::dynamicTraversal(", "dynpr::dynamicFrontier(",
                 "dynpr::dynamicFrontierFromFlags(", "dynpr::loadMatrixMarket(", "dynpr::loadTemporalEdgeList(",
                 "dynpr::splitTemporal(", "dynpr::generateRandomBatch(", "dynpr::batchSizeFromFraction(",
                 "dynpr::ParseError::ParseError(", "dynpr::approachName(", "dynpr::approachFromName(",
                 "dynpr::computeReferenceRanks(", "dynpr::runExperiment(", "dynpr::summarizeRows(",
                 "dynpr::emitReport("]:
        assert name in syms, name
