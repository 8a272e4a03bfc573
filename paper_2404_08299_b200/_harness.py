"""Input formats and the experiment harness -- the
Python mirror of module.cpp:138-160 (load_matrix_market,
load_temporal_edge_list, compute_reference_ranks) plus the C++ harness API of
harness.hpp:12-79 (run_experiment, summarize_rows, emit_report) and
workload.hpp:58-64 (split_temporal).

Files are parsed by libdynpr_cuda.so (memory-mapped, same token rules and
ParseError texts as workload.cpp:43-136); experiments run the device engines
through dynpr_run_experiment, with graphs, batch ingest, the 500-sweep
reference ranks and the chained warm-start ranks all on the GPU.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N


class ParseError(ValueError):
    """dynpr::ParseError (workload.hpp:12-15); a ValueError like module.cpp:164."""


class Approach(enum.IntEnum):  # harness.hpp:12
    STATIC = 0
    NAIVE_DYNAMIC = 1
    DYNAMIC_TRAVERSAL = 2
    DYNAMIC_FRONTIER = 3
    DYNAMIC_FRONTIER_PRUNE = 4


_APPROACH_NAMES = ("static", "nd", "dt", "df", "dfp")


def approach_name(a: Approach) -> str:  # harness.cpp:318-327
    return _APPROACH_NAMES[int(a)]


def approach_from_name(name: str) -> Approach:  # harness.cpp:329-336
    try:
        return Approach(_APPROACH_NAMES.index(name))
    except ValueError:
        raise ValueError(f"unknown approach '{name}'") from None


class ExperimentMode(enum.IntEnum):  # harness.hpp:16
    STATIC = 0
    TEMPORAL = 1
    RANDOM_BATCH = 2


class ChainMode(enum.IntEnum):  # harness.hpp:20-23
    PER_APPROACH = 0
    SHARED_REFERENCE = 1


class ReportFormat(enum.IntEnum):  # harness.hpp:55
    CSV = 0
    JSON = 1


@dataclass
class ExperimentRow:  # harness.hpp:29-39
    graph_name: str = ""
    approach: str = ""
    batch_size_spec: str = ""
    batch_index: int = 0
    runtime_millis: float = 0.0
    iterations: int = 0
    affected_vertex_iterations: int = 0
    l1_error_vs_reference: float = 0.0
    converged: bool = False


@dataclass
class ExperimentSpec:  # harness.hpp:41-53
    graph_path: str = ""
    graph_name: str = ""
    mode: ExperimentMode = ExperimentMode.STATIC
    batch_size_specs: Sequence[str] = field(default_factory=list)
    approaches: Sequence[Approach] = field(default_factory=list)
    seed: int = 1
    repetitions: int = 1
    base_fraction: float = 0.9
    batch_count: int = 100
    insert_fraction: float = 0.8
    chain_mode: ChainMode = ChainMode.PER_APPROACH
    threads: int = 0
    record_timing: bool = True
    config: object = None  # EngineConfig (default when None)


def _check(rc: int) -> None:
    if rc == N.DYNPR_PARSE_ERROR:
        raise ParseError(N.last_error())
    from . import _check as base_check
    base_check(rc)


class _EdgeList:
    def __init__(self, handle: int):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            N.lib().dynpr_edge_list_destroy(C.c_void_p(self.h))
            self.h = None

    def info(self):
        n, cnt, ts = C.c_uint32(), C.c_uint64(), C.c_int()
        _check(N.lib().dynpr_edge_list_info(C.c_void_p(self.h), C.byref(n), C.byref(cnt), C.byref(ts)))
        return n.value, cnt.value, bool(ts.value)

    def arrays(self, first: int = 0, count: Optional[int] = None):
        n, total, has_ts = self.info()
        count = total - first if count is None else count
        s = np.empty(max(count, 1), np.uint32)
        d = np.empty(max(count, 1), np.uint32)
        t = np.empty(max(count, 1), np.int64) if has_ts else None
        _check(N.lib().dynpr_edge_list_copy(C.c_void_p(self.h), first, count, s.ctypes.data, d.ctypes.data,
                                            t.ctypes.data if t is not None else None))
        return s[:count], d[:count], (t[:count] if t is not None else None)


def _load(fn, path: str) -> _EdgeList:
    h = C.c_void_p()
    _check(fn(str(path).encode(), C.byref(h)))
    return _EdgeList(h.value)


def load_matrix_market_arrays(path: str):
    """loadMatrixMarket as numpy arrays: (src uint32, dst uint32, vertex_count)."""
    el = _load(N.lib().dynpr_load_matrix_market, path)
    n, _, _ = el.info()
    s, d, _ = el.arrays()
    return s, d, n


def load_matrix_market(path: str):
    """loadMatrixMarket (workload.cpp:43-107) -> (edges, vertex_count), the
    shape module.cpp:138-143 returns: edges is a list of (u, v) tuples."""
    s, d, n = load_matrix_market_arrays(path)
    return list(zip(s.tolist(), d.tolist())), n


def load_temporal_edge_list_arrays(path: str):
    """loadTemporalEdgeList as numpy arrays: (src, dst, timestamps, vertex_count)."""
    el = _load(N.lib().dynpr_load_temporal_edge_list, path)
    n, _, _ = el.info()
    s, d, t = el.arrays()
    return s, d, t, n


def load_temporal_edge_list(path: str):
    """loadTemporalEdgeList (workload.cpp:109-136) -> (entries, vertex_count)
    with entries a list of (source, target, timestamp) tuples
    (module.cpp:144-153)."""
    s, d, t, n = load_temporal_edge_list_arrays(path)
    return list(zip(s.tolist(), d.tolist(), t.tolist())), n


def split_temporal(path_or_entries, base_fraction: float, batch_count: int, batch_size: int):
    """splitTemporal (workload.cpp:138-181) of a temporal file -> (base_edges,
    [insertion batches]) as (src, dst) uint32 array pairs."""
    el = _load(N.lib().dynpr_load_temporal_edge_list, path_or_entries)
    base = C.c_void_p()
    base_count = C.c_uint64()
    _check(N.lib().dynpr_split_temporal(C.c_void_p(el.h), float(base_fraction), int(batch_count),
                                        int(batch_size), C.byref(base), C.byref(base_count)))
    b = _EdgeList(base.value)
    bs, bd, _ = b.arrays()
    batches = []
    for i in range(batch_count):
        s, d, _ = el.arrays(base_count.value + i * batch_size, batch_size)
        batches.append((s, d))
    return (bs, bd), batches


def compute_reference_ranks(g_transpose, g_forward, config=None) -> np.ndarray:
    """computeReferenceRanks (harness.cpp:340-349): Static for exactly
    max_iterations sweeps with the convergence check disabled, on the GPU."""
    from . import EngineConfig, _p
    cfg = (config or EngineConfig())._c()
    ranks = np.empty(max(g_transpose.vertex_count, 1), np.float64)
    _check(N.lib().dynpr_compute_reference_ranks(C.c_void_p(g_transpose.ctx.h), C.c_void_p(g_transpose.h),
                                                 C.c_void_p(g_forward.h), C.byref(cfg), _p(ranks)))
    return ranks[: g_transpose.vertex_count]


class _Report:
    def __init__(self, handle: int):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            N.lib().dynpr_report_destroy(C.c_void_p(self.h))
            self.h = None

    @classmethod
    def from_rows(cls, rows: Sequence[ExperimentRow]) -> "_Report":
        h = C.c_void_p()
        _check(N.lib().dynpr_report_create(C.byref(h)))
        r = cls(h.value)
        for x in rows:
            c = N.ExperimentRow(x.graph_name.encode(), x.approach.encode(), x.batch_size_spec.encode(),
                                int(x.batch_index), float(x.runtime_millis), int(x.iterations),
                                int(x.affected_vertex_iterations), float(x.l1_error_vs_reference),
                                int(bool(x.converged)))
            _check(N.lib().dynpr_report_append(C.c_void_p(r.h), C.byref(c)))
        return r

    def rows(self) -> List[ExperimentRow]:
        cnt = C.c_uint64()
        _check(N.lib().dynpr_report_size(C.c_void_p(self.h), C.byref(cnt)))
        out = []
        for i in range(cnt.value):
            c = N.ExperimentRow()
            _check(N.lib().dynpr_report_row(C.c_void_p(self.h), i, C.byref(c)))
            out.append(ExperimentRow(c.graph_name.decode(), c.approach.decode(), c.batch_size_spec.decode(),
                                     c.batch_index, c.runtime_millis, c.iterations,
                                     c.affected_vertex_iterations, c.l1_error_vs_reference, bool(c.converged)))
        return out


def run_experiment(spec: ExperimentSpec, ctx=None) -> List[ExperimentRow]:
    """runExperiment (harness.cpp:351-381) on the device engines: per-batch
    rows, then one summary row (batch_index -1) per (approach, batch size)."""
    from . import EngineConfig, _ctx
    cx = _ctx(ctx)
    c = N.ExperimentSpec()
    N.lib().dynpr_experiment_spec_default(C.byref(c))
    specs = [s.encode() for s in spec.batch_size_specs]
    spec_arr = (C.c_char_p * max(len(specs), 1))(*specs)
    appr = (C.c_int32 * max(len(spec.approaches), 1))(*[int(a) for a in spec.approaches])
    path = str(spec.graph_path).encode()
    name = (spec.graph_name or "").encode()
    c.graph_path = path
    c.graph_name = name
    c.mode = int(spec.mode)
    c.batch_size_specs = spec_arr
    c.n_batch_size_specs = len(specs)
    c.approaches = appr
    c.n_approaches = len(spec.approaches)
    c.seed = int(spec.seed)
    c.repetitions = int(spec.repetitions)
    c.base_fraction = float(spec.base_fraction)
    c.batch_count = int(spec.batch_count)
    c.insert_fraction = float(spec.insert_fraction)
    c.chain_mode = int(spec.chain_mode)
    c.threads = int(spec.threads)
    c.record_timing = int(bool(spec.record_timing))
    c.config = (spec.config or EngineConfig())._c()
    h = C.c_void_p()
    _check(N.lib().dynpr_run_experiment(C.c_void_p(cx.h), C.byref(c), C.byref(h)))
    return _Report(h.value).rows()


def summarize_rows(rows: Sequence[ExperimentRow]) -> List[ExperimentRow]:
    """summarizeRows (harness.cpp:68-113)."""
    r = _Report.from_rows(rows)
    h = C.c_void_p()
    _check(N.lib().dynpr_report_summarize(C.c_void_p(r.h), C.byref(h)))
    return _Report(h.value).rows()


def emit_report(rows: Sequence[ExperimentRow], format: ReportFormat, path: str) -> None:
    """emitReport (harness.cpp:380-396): CSV or JSON, %.17g floats; "-" = stdout."""
    r = _Report.from_rows(rows)
    _check(N.lib().dynpr_report_emit(C.c_void_p(r.h), int(format), str(path).encode()))
