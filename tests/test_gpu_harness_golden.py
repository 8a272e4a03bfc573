"""Device harness report bytes against digests of the reference's own
reports (tests/golden/harness_golden.json, made by
tests/golden/make_harness_golden.py from the unmodified library): runs where
oracle/_ref is not available too."""
import hashlib
import json
import os

import pytest

from harness_data import write_matrix_market, write_temporal_stream

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "harness_golden.json")))


def _digest(dp, spec, out):
    rows = dp.run_experiment(spec)
    dp.emit_report(rows, dp.ReportFormat.CSV, str(out))
    data = out.read_bytes()
    return hashlib.md5(data).hexdigest(), len(data)


def test_temporal_criterion9_digest(dp, tmp_path):
    p = write_temporal_stream(str(tmp_path / "temporal-10k.txt"))
    spec = dp.ExperimentSpec(graph_path=p, mode=dp.ExperimentMode.TEMPORAL, batch_size_specs=["1e-3"],
                             approaches=list(dp.Approach), seed=1, record_timing=False)
    md5, n = _digest(dp, spec, tmp_path / "r.csv")
    assert (md5, n) == (GOLDEN["temporal_criterion9"]["md5"], GOLDEN["temporal_criterion9"]["bytes"])


def test_random_batch_digest(dp, tmp_path):
    p = write_matrix_market(str(tmp_path / "rb-general.mtx"), 2000, 16000, symmetry="general", seed=13)
    spec = dp.ExperimentSpec(graph_path=p, mode=dp.ExperimentMode.RANDOM_BATCH, batch_size_specs=["1e-3", "1e-2"],
                             approaches=list(dp.Approach), seed=7, repetitions=2, record_timing=False)
    md5, n = _digest(dp, spec, tmp_path / "r.csv")
    assert (md5, n) == (GOLDEN["random_general"]["md5"], GOLDEN["random_general"]["bytes"])
