"""CPU tests of the input formats and the report writer (SURVEY 8f rows 1
and 3): libdynpr_cuda.so's MatrixMarket / SNAP-temporal loaders,
splitTemporal, summarizeRows and emitReport against the reference library
(oracle/_ref) -- same arrays, same error class and message, same report
bytes.  These entry points are host code, so no GPU is needed."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle
import paper_2404_08299_b200 as dp
from harness_data import write_matrix_market, write_temporal_stream

pytestmark = pytest.mark.skipif(not oracle.available("ref"), reason="reference library not built")


@pytest.fixture(scope="module")
def ref():
    return oracle.Oracle("ref")


@pytest.fixture(autouse=True, params=["1", "3", "7"], ids=["seq", "par3", "par7"])
def parse_threads(request, monkeypatch):
    """Run every loader test on the sequential path and on the parallel
    chunked parser (forced on small files)."""
    monkeypatch.setenv("DYNPR_PARSE_THREADS", request.param)
    return request.param


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


def _same_mm(ref, path):
    try:
        want = ref.load_matrix_market(path)
    except oracle.OracleError as e:
        exc = dp.ParseError if e.code == 6 else (RuntimeError if e.code == 7 else ValueError)
        with pytest.raises(exc) as got:
            dp.load_matrix_market_arrays(path)
        assert str(got.value) == e.msg, (str(got.value), e.msg)
        return None
    s, d, n = dp.load_matrix_market_arrays(path)
    assert n == want[2]
    assert np.array_equal(s, want[0]) and np.array_equal(d, want[1])
    return s, d, n


MM_CASES = {
    "general": "%%MatrixMarket matrix coordinate pattern general\n% c\n3 4 3\n1 2\n3 4\n2 2\n",
    "symmetric_weights": "%%MatrixMarket matrix coordinate real symmetric\n4 4 3\n1 2 0.5\n3 3 1\n4 1 2\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 -1\n3 2 4\n",
    "hermitian_upper": "%%MATRIXMARKET Matrix COORDINATE complex HERMITIAN\n2 2 1\n2 1 1 0\n",
    "crlf_blank_comments": "%%MatrixMarket matrix coordinate pattern general\r\n\r\n%x\r\n3 3 2\r\n\r\n% mid\r\n1 3\r\n3 1\r\n",
    "no_final_newline": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1",
    "trailing_ignored": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2\ngarbage here\n",
    "tabs_extra_tokens": "%%MatrixMarket\tmatrix\tcoordinate pattern general\n2\t2\t1\t9\n 1\t2 x y\n",
    "empty": "",
    "only_newline": "\n",
    "bad_banner": "%MatrixMarket matrix coordinate pattern general\n1 1 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "missing_size": "%%MatrixMarket matrix coordinate pattern general\n% only comments\n",
    "bad_size": "%%MatrixMarket matrix coordinate pattern general\n2 x 1\n1 1\n",
    "size_two_tokens": "%%MatrixMarket matrix coordinate pattern general\n2 2\n",
    "truncated": "%%MatrixMarket matrix coordinate pattern general\n3 3 3\n1 2\n2 3\n",
    "out_of_bounds": "%%MatrixMarket matrix coordinate pattern general\n3 2 2\n1 2\n1 3\n",
    "zero_index": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n0 1\n",
    "malformed_entry": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 b\n",
    "plus_sign": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n+1 2\n",
    "negative": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n-1 2\n",
    "space_before_comment": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n  % not a comment\n1 2\n",
    "whitespace_line": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n   \n1 2\n",
    "zero_entries": "%%MatrixMarket matrix coordinate pattern general\n5 2 0\n",
    "late_garbage_ignored": "%%MatrixMarket matrix coordinate pattern general\n4 4 3\n1 2\n2 3\n3 4\n"
                            + "".join(f"{i % 4 + 1} {i % 3 + 1}\n" for i in range(40)) + "bad line\n",
    "late_error_counts": "%%MatrixMarket matrix coordinate pattern general\n4 4 40\n"
                         + "".join(f"{i % 4 + 1} {i % 3 + 1}\n" for i in range(30)) + "x y\n",
    "short_many": "%%MatrixMarket matrix coordinate pattern symmetric\n9 9 50\n"
                  + "".join(f"{i % 9 + 1} {(i * 7) % 9 + 1}\n" for i in range(45)),
}


@pytest.mark.parametrize("case", sorted(MM_CASES))
def test_matrix_market_matches_reference(ref, tmp_path, case):
    _same_mm(ref, _write(tmp_path, case + ".mtx", MM_CASES[case]))


def test_matrix_market_missing_file(ref, tmp_path):
    _same_mm(ref, str(tmp_path / "nope.mtx"))


@pytest.mark.parametrize("sym,weights", [("general", False), ("symmetric", True)])
def test_matrix_market_generated(ref, tmp_path, sym, weights):
    p = write_matrix_market(str(tmp_path / "g.mtx"), 700, 9000, symmetry=sym, weights=weights)
    s, d, n = _same_mm(ref, p)
    edges, n2 = dp.load_matrix_market(p)  # module.cpp:138-143 shape
    assert n2 == n and edges[:5] == list(zip(s[:5].tolist(), d[:5].tolist()))


def _same_temporal(ref, path):
    try:
        want = ref.load_temporal(path)
    except oracle.OracleError as e:
        exc = dp.ParseError if e.code == 6 else RuntimeError
        with pytest.raises(exc) as got:
            dp.load_temporal_edge_list_arrays(path)
        assert str(got.value) == e.msg
        return None
    got = dp.load_temporal_edge_list_arrays(path)
    assert got[3] == want[3]
    for a, b in zip(got[:3], want[:3]):
        assert np.array_equal(a, b)
    return got


T_CASES = {
    "basic": "# c\n10 20 5\n20 30 3\n10 30 3\n",
    "crlf_blank": "# c\r\n\r\n7 8 1\r\n8 7 0\r\n",
    "negative_ts": "1 2 -5\n2 3 -7\n3 1 0\n",
    "duplicates_stable": "1 2 4\n1 2 4\n2 1 4\n5 6 1\n1 2 1\n",
    "extra_tokens": "1 2 3 extra\n2 3 4\n",
    "huge_ids": "18446744073709551615 0 1\n0 18446744073709551615 2\n",
    "malformed": "1 2 3\n1 x 3\n",
    "missing_ts": "1 2\n",
    "plus_ts": "1 2 +3\n",
    "space_hash": "1 2 3\n # comment?\n",
    "no_final_newline": "1 2 3\n3 4 1",
    "empty": "",
    "many_lines_late_error": "".join(f"{i * 31 % 97} {i * 17 % 89} {1000 - i}\n" for i in range(200)) + "1 2\n",
    "many_lines_unsorted": "# x\n" + "".join(f"{i * 31 % 97} {i * 17 % 89} {(i * 7919) % 13}\n"
                                            for i in range(300)),
}


@pytest.mark.parametrize("case", sorted(T_CASES))
def test_temporal_matches_reference(ref, tmp_path, case):
    _same_temporal(ref, _write(tmp_path, case + ".txt", T_CASES[case]))


@pytest.mark.parametrize("unsorted", [False, True])
def test_temporal_generated(ref, tmp_path, unsorted):
    p = write_temporal_stream(str(tmp_path / "t.txt"), unsorted=unsorted)
    got = _same_temporal(ref, p)
    entries, n = dp.load_temporal_edge_list(p)
    assert n == got[3] and entries[0] == (int(got[0][0]), int(got[1][0]), int(got[2][0]))


@pytest.mark.parametrize("frac,count,size", [(0.9, 30, 10), (0.5, 3, 7), (0.999, 1, 1)])
def test_split_temporal_matches_reference(ref, tmp_path, frac, count, size):
    p = write_temporal_stream(str(tmp_path / "t.txt"), entries=3000)
    (bs, bd), (s, d) = ref.split_temporal(p, frac, count, size)
    (cs, cd), batches = dp.split_temporal(p, frac, count, size)
    assert np.array_equal(bs, cs) and np.array_equal(bd, cd)
    assert np.array_equal(s, np.concatenate([b[0] for b in batches]))
    assert np.array_equal(d, np.concatenate([b[1] for b in batches]))


@pytest.mark.parametrize("frac,count,size,exc", [(0.9, 100, 100, dp.SizingError), (1.0, 1, 1, ValueError),
                                                 (0.0, 1, 1, ValueError), (0.5, 0, 1, ValueError),
                                                 (0.5, 1, 0, ValueError)])
def test_split_temporal_errors_match_reference(ref, tmp_path, frac, count, size, exc):
    p = write_temporal_stream(str(tmp_path / "t.txt"), entries=3000)
    with pytest.raises(oracle.OracleError) as want:
        ref.split_temporal(p, frac, count, size)
    with pytest.raises(exc) as got:
        dp.split_temporal(p, frac, count, size)
    assert str(got.value) == want.value.msg


def _rows(seed):
    rng = np.random.default_rng(seed)
    rows = []
    for a in ("static", "nd", "dfp"):
        for spec in ("1e-3", "1e-4"):
            for i in range(4):
                l1 = float(rng.random() * 1e-9) if i != 2 else (math.nan if a == "nd" else 0.0)
                rows.append(dp.ExperimentRow('g"r\\aph', a, spec, i, float(rng.random() * 10) if i else 0.0,
                                             int(rng.integers(1, 80)), int(rng.integers(0, 10**12)), l1,
                                             bool(rng.random() < 0.9)))
    return rows


def _ctypes_rows(rows):
    from paper_2404_08299_b200 import _native as N
    arr = (N.ExperimentRow * len(rows))()
    keep = []
    for k, r in enumerate(rows):
        enc = [r.graph_name.encode(), r.approach.encode(), r.batch_size_spec.encode()]
        keep.append(enc)
        arr[k] = N.ExperimentRow(*enc, r.batch_index, r.runtime_millis, r.iterations,
                                 r.affected_vertex_iterations, r.l1_error_vs_reference, int(r.converged))
    return arr, keep


@pytest.mark.parametrize("fmt", [dp.ReportFormat.CSV, dp.ReportFormat.JSON])
@pytest.mark.parametrize("summarize", [False, True])
def test_report_bytes_match_reference(ref, tmp_path, fmt, summarize):
    rows = _rows(11)
    arr, keep = _ctypes_rows(rows)
    ref.summarize_emit(arr, len(rows), summarize, int(fmt), str(tmp_path / "want"))
    out = dp.summarize_rows(rows) if summarize else rows
    dp.emit_report(out, fmt, str(tmp_path / "got"))
    assert (tmp_path / "got").read_bytes() == (tmp_path / "want").read_bytes()


def test_report_errors():
    with pytest.raises(ValueError, match="emitReport: no rows"):
        dp.emit_report([], dp.ReportFormat.CSV, "-")
    with pytest.raises(RuntimeError, match="emitReport: cannot open"):
        dp.emit_report(_rows(1), dp.ReportFormat.CSV, "/nonexistent-dir/x.csv")
    assert dp.approach_from_name("dfp") == dp.Approach.DYNAMIC_FRONTIER_PRUNE
    assert [dp.approach_name(a) for a in dp.Approach] == ["static", "nd", "dt", "df", "dfp"]
    with pytest.raises(ValueError, match="unknown approach 'x'"):
        dp.approach_from_name("x")
