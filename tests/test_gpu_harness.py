"""GPU parity of the experiment harness: runExperiment
driven through the device engines must write the SAME report bytes as the
reference's runExperiment + emitReport (oracle/_ref) with timing disabled --
every iteration count, affected-vertex count, convergence flag and L1 error
vs the 500-sweep reference (%.17g) identical.  This is the reference's
acceptance criterion 9/10 shape (temporal, 1e-3 batches, all five approaches,
seed 1, --no-timing) on a synthetic stream of the fixture's size."""
import ctypes as C

import numpy as np
import pytest

import oracle
from harness_data import write_matrix_market, write_temporal_stream
from helpers import to_dev

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.available("ref"), reason="reference library not built")]

ALL = ("static", "nd", "dt", "df", "dfp")


@pytest.fixture(scope="module")
def ref():
    return oracle.Oracle("ref")


def _spec(dp, path, mode, sizes, approaches=ALL, **kw):
    return dp.ExperimentSpec(graph_path=path, mode=mode, batch_size_specs=list(sizes),
                             approaches=[dp.approach_from_name(a) for a in approaches], record_timing=False, **kw)


def _ref_bytes(ref, dp, spec, fmt, out):
    from paper_2404_08299_b200 import _native as N
    c = N.ExperimentSpec()
    N.lib().dynpr_experiment_spec_default(C.byref(c))
    sizes = [s.encode() for s in spec.batch_size_specs]
    keep = [(C.c_char_p * max(len(sizes), 1))(*sizes),
            (C.c_int32 * len(spec.approaches))(*[int(a) for a in spec.approaches]),
            str(spec.graph_path).encode(), (spec.graph_name or "").encode()]
    c.batch_size_specs, c.approaches, c.graph_path, c.graph_name = keep
    c.n_batch_size_specs = len(sizes)
    c.n_approaches = len(spec.approaches)
    c.mode = int(spec.mode)
    c.seed = spec.seed
    c.repetitions = spec.repetitions
    c.base_fraction = spec.base_fraction
    c.batch_count = spec.batch_count
    c.insert_fraction = spec.insert_fraction
    c.chain_mode = int(spec.chain_mode)
    c.record_timing = int(spec.record_timing)
    c.config = (spec.config or dp.EngineConfig())._c()
    ref.run_experiment(c, int(fmt), str(out))
    return out.read_bytes()


def _ours_bytes(dp, spec, fmt, out):
    rows = dp.run_experiment(spec)
    dp.emit_report(rows, fmt, str(out))
    return rows, out.read_bytes()


def test_temporal_pipeline_report_identical(dp, ref, tmp_path):
    """Criterion-9 shape: 100 temporal 1e-3 batches, static,nd,dt,df,dfp."""
    p = write_temporal_stream(str(tmp_path / "temporal-10k.txt"))
    spec = _spec(dp, p, dp.ExperimentMode.TEMPORAL, ["1e-3"], seed=1)
    want = _ref_bytes(ref, dp, spec, dp.ReportFormat.CSV, tmp_path / "want.csv")
    rows, got = _ours_bytes(dp, spec, dp.ReportFormat.CSV, tmp_path / "got.csv")
    assert got == want
    data = [r for r in rows if r.batch_index >= 0]
    assert len(data) == 500 and sum(r.batch_index == -1 for r in rows) == 5
    assert all(r.converged for r in rows)


def test_temporal_shared_reference_json_identical(dp, ref, tmp_path):
    p = write_temporal_stream(str(tmp_path / "t.txt"), n_vertices=900, entries=6000, seed=9, unsorted=True)
    spec = _spec(dp, p, dp.ExperimentMode.TEMPORAL, ["2e-3", "5e-4"], ("nd", "df", "dfp"), batch_count=20,
                 base_fraction=0.8, chain_mode=dp.ChainMode.SHARED_REFERENCE, graph_name="shared")
    want = _ref_bytes(ref, dp, spec, dp.ReportFormat.JSON, tmp_path / "want.json")
    _, got = _ours_bytes(dp, spec, dp.ReportFormat.JSON, tmp_path / "got.json")
    assert got == want


@pytest.mark.parametrize("sym", ["general", "symmetric"])
def test_random_batch_report_identical(dp, ref, tmp_path, sym):
    p = write_matrix_market(str(tmp_path / f"rb-{sym}.mtx"), 2000, 16000, symmetry=sym, seed=13)
    spec = _spec(dp, p, dp.ExperimentMode.RANDOM_BATCH, ["1e-3", "1e-2"], repetitions=2, seed=7)
    want = _ref_bytes(ref, dp, spec, dp.ReportFormat.CSV, tmp_path / "want.csv")
    rows, got = _ours_bytes(dp, spec, dp.ReportFormat.CSV, tmp_path / "got.csv")
    assert got == want
    assert len(rows) == 2 * 2 * 5 + 2 * 5


def test_static_report_identical(dp, ref, tmp_path):
    p = write_matrix_market(str(tmp_path / "st.mtx"), 3000, 30000, seed=17)
    cfg = dp.EngineConfig(iteration_tolerance=1e-12, max_iterations=300)
    spec = _spec(dp, p, dp.ExperimentMode.STATIC, [], ("static",), repetitions=3, config=cfg)
    want = _ref_bytes(ref, dp, spec, dp.ReportFormat.CSV, tmp_path / "want.csv")
    _, got = _ours_bytes(dp, spec, dp.ReportFormat.CSV, tmp_path / "got.csv")
    assert got == want


def test_timed_rows_and_errors(dp, tmp_path):
    p = write_temporal_stream(str(tmp_path / "t.txt"), n_vertices=400, entries=3000, seed=2)
    spec = _spec(dp, p, dp.ExperimentMode.TEMPORAL, ["1e-2"], ("static", "dfp"), batch_count=5)
    spec.record_timing = True
    rows = dp.run_experiment(spec)
    assert all(r.runtime_millis > 0 for r in rows) and rows[0].graph_name == "t"
    with pytest.raises(ValueError, match="runExperiment: no approaches requested"):
        dp.run_experiment(_spec(dp, p, dp.ExperimentMode.TEMPORAL, ["1e-2"], ()))
    with pytest.raises(ValueError, match="runExperiment: no batch sizes requested"):
        dp.run_experiment(_spec(dp, p, dp.ExperimentMode.TEMPORAL, []))
    with pytest.raises(ValueError, match="repetitions must be >= 1"):
        dp.run_experiment(_spec(dp, p, dp.ExperimentMode.TEMPORAL, ["1e-2"], repetitions=0))
    with pytest.raises(ValueError, match="dampingFactor"):
        dp.run_experiment(_spec(dp, p, dp.ExperimentMode.TEMPORAL, ["1e-2"],
                                config=dp.EngineConfig(damping_factor=1.5)))
    with pytest.raises(dp.SizingError, match="splitTemporal: stream has 3000 entries"):
        dp.run_experiment(_spec(dp, p, dp.ExperimentMode.TEMPORAL, ["1e-1"]))
    with pytest.raises(dp.ParseError, match="missing %%MatrixMarket banner"):
        dp.run_experiment(_spec(dp, p, dp.ExperimentMode.STATIC, [], ("static",)))
    with pytest.raises(RuntimeError, match="cannot open"):
        dp.run_experiment(_spec(dp, str(tmp_path / "missing.mtx"), dp.ExperimentMode.STATIC, [], ("static",)))


def test_compute_reference_ranks_bitwise(dp, ref, tmp_path):
    g, gt = None, None
    O = ref
    rng = O.rng(5)
    og = O.random_graph(rng, 800, 6000)
    ogt = O.transpose(og)
    cfg = oracle.default_config(max_iterations=120)
    want = O.compute_reference_ranks(ogt, og, cfg)
    got = dp.compute_reference_ranks(to_dev(dp, ogt), to_dev(dp, og), dp.EngineConfig(max_iterations=120))
    assert np.array_equal(got, want)


def test_loaded_graph_feeds_device_build(dp, ref, tmp_path):
    """loadMatrixMarket -> device buildCsr + addSelfLoops: same CSR bytes as
    the reference's buildCsr + addSelfLoops of its own load."""
    p = write_matrix_market(str(tmp_path / "b.mtx"), 1500, 12000, symmetry="symmetric", seed=21)
    s, d, n = ref.load_matrix_market(p)
    og = ref.add_self_loops(ref.build_csr((s, d), n))
    ds, dd, dn = dp.load_matrix_market_arrays(p)
    g = dp.add_self_loops(dp.build_csr((ds, dd), dn))
    off, tgt = og.csr()
    assert np.array_equal(g.offsets, off) and np.array_equal(g.targets, tgt)
