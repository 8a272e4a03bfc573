"""ORACLE / TEST INFRASTRUCTURE -- the checker, never the product.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
reference arm may import this package.  It exposes two CPU implementations of
the reference hot path behind one numpy-facing API:

* ``Oracle("port")`` -- the plain-C restatement ``oracle/dynpr_oracle.c``
  (built into ``oracle/_build/libdynpr_oracle.so``), sequential, each function
  citing the reference file:line it restates.
* ``Oracle("ref")`` -- the unmodified reference library compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` into
  ``oracle/_ref/libdynpr_ref.so`` (OpenMP, the reference's own code).

The restatement is pinned against golden vectors generated from the
reference (tests/golden/) and, where ``_ref`` is present, against the
reference directly (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libdynpr_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libdynpr_ref.so")


class Config(C.Structure):
    """dynpr_config (include/dynpr_cuda.h) == EngineConfig (rank.hpp:25-39)."""

    _fields_ = [
        ("damping_factor", C.c_double),
        ("iteration_tolerance", C.c_double),
        ("frontier_tolerance", C.c_double),
        ("prune_tolerance", C.c_double),
        ("max_iterations", C.c_int32),
        ("low_degree_threshold", C.c_uint32),
        ("partition_strategy", C.c_int32),
        ("convergence_check_disabled", C.c_int32),
    ]


def default_config(**kw) -> Config:
    c = Config(0.85, 1e-10, 1e-6, 1e-6, 500, 32, 2, 0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class Stats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("affected_vertex_iterations", C.c_uint64),
        ("final_delta", C.c_double),
        ("processed_edges", C.c_uint64),
        ("device_ms", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


OBSERVER = C.CFUNCTYPE(None, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                       C.c_uint64, C.c_void_p)

_vp = C.c_void_p
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32).reshape(-1))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8).reshape(-1))


def split_edges(edges):
    """list of (u, v) | (src, dst) arrays | object with .src/.dst -> (src uint32, dst uint32)."""
    if hasattr(edges, "src") and hasattr(edges, "dst"):
        return _u32(edges.src), _u32(edges.dst)
    if isinstance(edges, tuple) and len(edges) == 2 and isinstance(edges[0], np.ndarray):
        return _u32(edges[0]), _u32(edges[1])
    arr = np.asarray(list(edges), dtype=np.uint64).reshape(-1, 2)
    return _u32(arr[:, 0]), _u32(arr[:, 1])


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.msg = msg


@dataclass
class Result:
    ranks: np.ndarray
    iterations: int
    affected_vertex_iterations: int
    converged: bool
    final_delta: float
    processed_edges: int = 0
    ms: float = 0.0
    trace: list = field(default_factory=list)


class Graph:
    """Owning handle of an oracle-side CSR graph."""

    def __init__(self, lib: "Oracle", handle):
        self._lib = lib
        self.h = handle
        n = C.c_uint32()
        m = C.c_uint64()
        lib._info(handle, C.byref(n), C.byref(m))
        self.n = n.value
        self.m = m.value

    def __del__(self):
        try:
            if self.h:
                self._lib._free(self.h)
        except Exception:
            pass

    def csr(self):
        off = np.zeros(self.n + 1, dtype=np.uint64)
        tgt = np.zeros(max(self.m, 1), dtype=np.uint32)
        self._lib._download(self.h, _ptr(off, _u64p), _ptr(tgt, _u32p))
        return off, tgt[: self.m]

    def degrees(self):
        off, _ = self.csr()
        return np.diff(off).astype(np.uint32)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        p = "orc_" if kind == "port" else "ref_"
        self.p = p
        getattr(L, p + "last_error").restype = C.c_char_p
        if kind == "port":
            self._info = L.orc_graph_info
            self._free = L.orc_graph_free
            self._download = L.orc_graph_download
            for name in ("orc_transpose", "orc_add_self_loops", "orc_random_graph"):
                getattr(L, name).restype = _vp
            L.orc_linf.restype = C.c_double
            L.orc_l1.restype = C.c_double
            L.orc_derive_seed.restype = C.c_uint64
            L.orc_batch_size_from_fraction.restype = C.c_uint64
            L.orc_batch_size_from_fraction.argtypes = [C.c_double, C.c_uint64]
            L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
            L.orc_random_graph.argtypes = [_u64p, C.c_uint32, C.c_uint64]
            L.orc_rng_next.restype = C.c_uint64
            L.orc_rng_bounded.restype = C.c_uint64
            L.orc_rng_bounded.argtypes = [_u64p, C.c_uint64]
            L.orc_rng_double.restype = C.c_double
            L.orc_linf.argtypes = [_dp, _dp, C.c_uint64]
            L.orc_l1.argtypes = [_dp, _dp, C.c_uint64]
            L.orc_kronecker_edges.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, _u32p, _u32p]
            L.orc_rmat_edges.argtypes = [C.c_uint32, C.c_uint64, C.c_double, C.c_double,
                                         C.c_double, C.c_uint64, _u32p, _u32p]
        else:
            self._info = L.ref_graph_info
            self._free = L.ref_graph_free
            self._download = L.ref_graph_download
            L.ref_rng_new.restype = _vp
            L.ref_rng_new.argtypes = [C.c_uint64]
            L.ref_rng_free.argtypes = [_vp]
            for nm in ("ref_rng_next", "ref_rng_bounded", "ref_derive_seed",
                       "ref_batch_size_from_fraction"):
                getattr(L, nm).restype = C.c_uint64
            L.ref_rng_next.argtypes = [_vp]
            L.ref_rng_bounded.argtypes = [_vp, C.c_uint64]
            L.ref_rng_next_double.restype = C.c_double
            L.ref_rng_next_double.argtypes = [_vp]
            L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
            L.ref_batch_size_from_fraction.argtypes = [C.c_double, C.c_uint64]
            L.ref_random_graph.argtypes = [_vp, C.c_uint32, C.c_uint64, C.POINTER(_vp)]
            L.ref_set_threads.argtypes = [C.c_int]
        self._info.argtypes = [_vp, _u32p, _u64p]
        self._free.argtypes = [_vp]
        self._download.argtypes = [_vp, _u64p, _u32p]

    # ---- helpers ------------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, getattr(self.L, self.p + "last_error")().decode())

    def _graph_out(self, fn, *args):
        out = _vp()
        self._check(fn(*args, C.byref(out)))
        return Graph(self, out.value)

    def set_threads(self, t: int):
        if self.kind == "ref":
            self.L.ref_set_threads(int(t))

    def max_threads(self) -> int:
        return self.L.ref_max_threads() if self.kind == "ref" else 1

    # ---- rng / workload ----------------------------------------------------
    def derive_seed(self, seed: int, stream: int) -> int:
        return int(getattr(self.L, self.p + "derive_seed")(C.c_uint64(seed), C.c_uint64(stream)))

    def batch_size_from_fraction(self, f: float, total: int) -> int:
        return int(getattr(self.L, self.p + "batch_size_from_fraction")(f, total))

    def generate_random_batch(self, g: Graph, total: int, ins_frac: float, seed: int):
        cap = max(int(total), 1)
        is_, id_ = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        ds, dd = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        ni, nd = C.c_uint64(), C.c_uint64()
        self._check(getattr(self.L, self.p + "generate_random_batch")(
            C.c_void_p(g.h), C.c_uint64(total), C.c_double(ins_frac), C.c_uint64(seed),
            _ptr(is_, _u32p), _ptr(id_, _u32p), C.byref(ni),
            _ptr(ds, _u32p), _ptr(dd, _u32p), C.byref(nd)))
        return (ds[: nd.value].copy(), dd[: nd.value].copy()), (is_[: ni.value].copy(), id_[: ni.value].copy())

    # ---- graphs --------------------------------------------------------------
    def graph_from_csr(self, n: int, off, tgt) -> Graph:
        off = np.ascontiguousarray(np.asarray(off, dtype=np.uint64))
        m = len(tgt)  # targets.size(), checked against offsets.back() (graph.cpp:35-37)
        tgt = _u32(tgt) if len(tgt) else np.zeros(1, np.uint32)
        return self._graph_out(getattr(self.L, self.p + "graph_from_csr"), C.c_uint32(n),
                               _ptr(off, _u64p), _ptr(tgt, _u32p), C.c_uint64(m))

    def build_csr(self, edges, n: int) -> Graph:
        s, d = split_edges(edges)
        if len(s) == 0:
            s = d = np.zeros(1, np.uint32)
            cnt = 0
        else:
            cnt = len(s)
        fn = self.L.orc_build_csr if self.kind == "port" else self.L.ref_build_csr
        return self._graph_out(fn, C.c_uint32(n), _ptr(s, _u32p), _ptr(d, _u32p), C.c_uint64(cnt))

    def add_self_loops(self, g: Graph) -> Graph:
        if self.kind == "port":
            return Graph(self, self.L.orc_add_self_loops(C.c_void_p(g.h)))
        return self._graph_out(self.L.ref_add_self_loops, C.c_void_p(g.h))

    def transpose(self, g: Graph) -> Graph:
        if self.kind == "port":
            return Graph(self, self.L.orc_transpose(C.c_void_p(g.h)))
        return self._graph_out(self.L.ref_transpose, C.c_void_p(g.h))

    def apply_batch(self, g: Graph, dels, ins):
        ds, dd = split_edges(dels)
        is_, id_ = split_edges(ins)
        nd, ni = len(ds), len(is_)
        z = np.zeros(1, np.uint32)
        ds, dd = (ds, dd) if nd else (z, z)
        is_, id_ = (is_, id_) if ni else (z, z)
        miss, dup = C.c_uint64(0), C.c_uint64(0)
        out = _vp()
        self._check(getattr(self.L, self.p + "apply_batch")(
            C.c_void_p(g.h), _ptr(ds, _u32p), _ptr(dd, _u32p), C.c_uint64(nd),
            _ptr(is_, _u32p), _ptr(id_, _u32p), C.c_uint64(ni), C.byref(out),
            C.byref(miss), C.byref(dup)))
        return Graph(self, out.value), miss.value, dup.value

    def has_edge(self, g: Graph, s: int, t: int) -> bool:
        return bool(getattr(self.L, self.p + "has_edge")(C.c_void_p(g.h), C.c_uint32(s), C.c_uint32(t)))

    def random_graph(self, rng, n: int, pairs: int) -> Graph:
        """oracles.hpp:80-89; `rng` is an Rng of this backend."""
        if self.kind == "port":
            st = C.c_uint64(rng.state)
            h = self.L.orc_random_graph(C.byref(st), C.c_uint32(n), C.c_uint64(pairs))
            rng.state = st.value
            return Graph(self, h)
        out = _vp()
        self._check(self.L.ref_random_graph(C.c_void_p(rng.h), C.c_uint32(n),
                                            C.c_uint64(pairs), C.byref(out)))
        return Graph(self, out.value)

    def rng(self, seed: int):
        return PortRng(self, seed) if self.kind == "port" else RefRng(self, seed)

    def kronecker_edges(self, scale: int, count: int, seed=42):
        """Graph500-style Kronecker edges: RMAT draws + the seeded id bijection
        of the device generator (dynpr_graph_kronecker)."""
        src = np.zeros(max(count, 1), np.uint32)
        dst = np.zeros(max(count, 1), np.uint32)
        port = self if self.kind == "port" else Oracle("port")
        port.L.orc_kronecker_edges(scale, count, seed, _ptr(src, _u32p), _ptr(dst, _u32p))
        return src[:count], dst[:count]

    def rmat_edges(self, scale: int, count: int, a=0.57, b=0.19, c=0.19, seed=42):
        src = np.zeros(max(count, 1), np.uint32)
        dst = np.zeros(max(count, 1), np.uint32)
        port = self if self.kind == "port" else Oracle("port")
        port.L.orc_rmat_edges(scale, count, a, b, c, seed, _ptr(src, _u32p), _ptr(dst, _u32p))
        return src[:count], dst[:count]

    # ---- primitives --------------------------------------------------------
    def partition(self, g: Graph, threshold: int):
        order = np.zeros(max(g.n, 1), np.uint32)
        low = C.c_uint32()
        if self.kind == "port":
            self.L.orc_partition(C.c_void_p(g.h), C.c_uint32(threshold), _ptr(order, _u32p), C.byref(low))
        else:
            self._check(self.L.ref_partition(C.c_void_p(g.h), C.c_uint32(threshold),
                                             _ptr(order, _u32p), C.byref(low)))
        return order[: g.n], low.value

    def update_ranks(self, gT: Graph, gF: Graph, va, np_, prev, cur, cfg: Config, mode: int,
                     use_partition: bool = True):
        prev = _f64(prev)
        cur = _f64(cur).copy()
        if va is not None:
            va = _u8(va).copy()
            np_ = _u8(np_).copy()
            vap, npp = _ptr(va, _u8p), _ptr(np_, _u8p)
        else:
            vap = npp = None
        if self.kind == "port":
            self.L.orc_update_ranks(C.c_void_p(gT.h), C.c_void_p(gF.h), vap, npp,
                                    _ptr(prev, _dp), _ptr(cur, _dp), C.byref(cfg), C.c_int(mode))
        else:
            self._check(self.L.ref_update_ranks(C.c_void_p(gT.h), C.c_void_p(gF.h), vap, npp,
                                                _ptr(prev, _dp), _ptr(cur, _dp), C.byref(cfg),
                                                C.c_int(mode), C.c_int(int(use_partition))))
        return cur, va, np_

    def linf(self, a, b) -> float:
        a, b = _f64(a), _f64(b)
        if self.kind == "port":
            if len(a) != len(b):
                raise OracleError(1, "linfNormDelta: length mismatch")
            return float(self.L.orc_linf(_ptr(a, _dp), _ptr(b, _dp), len(a)))
        if len(a) != len(b):
            raise OracleError(1, "linfNormDelta: length mismatch")
        out = C.c_double()
        self._check(self.L.ref_linf(_ptr(a, _dp), _ptr(b, _dp), C.c_uint64(len(a)), C.byref(out)))
        return out.value

    def l1(self, a, b) -> float:
        a, b = _f64(a), _f64(b)
        if len(a) != len(b):
            raise OracleError(1, "l1NormDelta: length mismatch")
        if self.kind == "port":
            return float(self.L.orc_l1(_ptr(a, _dp), _ptr(b, _dp), len(a)))
        out = C.c_double()
        self._check(self.L.ref_l1(_ptr(a, _dp), _ptr(b, _dp), C.c_uint64(len(a)), C.byref(out)))
        return out.value

    def initial_affected(self, g: Graph, dels, ins):
        ds, dd = split_edges(dels)
        is_, id_ = split_edges(ins)
        nd, ni = len(ds), len(is_)
        z = np.zeros(1, np.uint32)
        ds, dd = (ds, dd) if nd else (z, z)
        is_, id_ = (is_, id_) if ni else (z, z)
        va = np.zeros(max(g.n, 1), np.uint8)
        np_ = np.zeros(max(g.n, 1), np.uint8)
        if self.kind == "port":
            self._check(self.L.orc_initial_affected(
                C.c_uint32(g.n), _ptr(ds, _u32p), _ptr(dd, _u32p), C.c_uint64(nd),
                _ptr(is_, _u32p), _ptr(id_, _u32p), C.c_uint64(ni), _ptr(va, _u8p), _ptr(np_, _u8p)))
        else:
            self._check(self.L.ref_initial_affected(
                C.c_void_p(g.h), _ptr(ds, _u32p), _ptr(dd, _u32p), C.c_uint64(nd),
                _ptr(is_, _u32p), _ptr(id_, _u32p), C.c_uint64(ni), _ptr(va, _u8p), _ptr(np_, _u8p)))
        return va[: g.n], np_[: g.n]

    def expand_affected(self, g: Graph, va, np_, use_partition=False, threshold=32):
        va = _u8(va).copy()
        np_ = _u8(np_)
        if self.kind == "port":
            self.L.orc_expand_affected(C.c_void_p(g.h), _ptr(va, _u8p), _ptr(np_, _u8p))
        else:
            self._check(self.L.ref_expand_affected(C.c_void_p(g.h), _ptr(va, _u8p), _ptr(np_, _u8p),
                                                   C.c_int(int(use_partition)), C.c_uint32(threshold)))
        return va

    def validate_config(self, cfg: Config):
        self._check(getattr(self.L, self.p + "validate_config")(C.byref(cfg)))

    # ---- engines -------------------------------------------------------------
    @staticmethod
    def _observer(trace: Optional[list], want_flags: bool, cb: Optional[Callable] = None):
        if trace is None and cb is None:
            return None, None

        def obs(it, ranks, processed, n, user):
            r = np.ctypeslib.as_array(ranks, shape=(n,)).copy()
            f = np.ctypeslib.as_array(processed, shape=(n,)).copy() if processed else None
            if trace is not None:
                trace.append((it, r, f))
            if cb is not None:
                cb(it, r)

        fn = OBSERVER(obs)
        return fn, fn

    def _result(self, ranks, st: Stats, trace) -> Result:
        return Result(ranks, st.iterations, st.affected_vertex_iterations, bool(st.converged),
                      st.final_delta, st.processed_edges, st.device_ms, trace or [])

    def static(self, gT: Graph, gF: Graph, cfg: Config = None, trace: Optional[list] = None) -> Result:
        cfg = cfg or default_config()
        ranks = np.zeros(max(gT.n, 1), np.float64)
        st = Stats()
        obs, keep = self._observer(trace, False)
        self._check(getattr(self.L, self.p + "static")(C.c_void_p(gT.h), C.c_void_p(gF.h), C.byref(cfg),
                                              _ptr(ranks, _dp), C.byref(st), obs, None))
        return self._result(ranks[: gT.n], st, trace)

    def naive_dynamic(self, gT: Graph, gF: Graph, prev, cfg: Config = None,
                      trace: Optional[list] = None) -> Result:
        cfg = cfg or default_config()
        prev = _f64(prev)
        ranks = np.zeros(max(gT.n, 1), np.float64)
        st = Stats()
        obs, keep = self._observer(trace, False)
        self._check(getattr(self.L, self.p + "naive_dynamic")(
            C.c_void_p(gT.h), C.c_void_p(gF.h), _ptr(prev, _dp), C.c_uint64(len(prev)),
            C.byref(cfg), _ptr(ranks, _dp), C.byref(st), obs, None))
        return self._result(ranks[: gT.n], st, trace)

    def dynamic_frontier(self, gF: Graph, gT: Graph, dels, ins, prev, cfg: Config = None,
                         pruning: bool = True, trace: Optional[list] = None) -> Result:
        """DF / DF-P.  With ``trace`` given the processed set of every sweep
        is recorded (port: natively; ref: through ref_frontier_trace, the
        public-call replay of convergeLoop)."""
        cfg = cfg or default_config()
        ds, dd = split_edges(dels)
        is_, id_ = split_edges(ins)
        nd, ni = len(ds), len(is_)
        z = np.zeros(1, np.uint32)
        ds, dd = (ds, dd) if nd else (z, z)
        is_, id_ = (is_, id_) if ni else (z, z)
        prev = _f64(prev)
        ranks = np.zeros(max(gT.n, 1), np.float64)
        st = Stats()
        obs, keep = self._observer(trace, True)
        if self.kind == "ref" and trace is not None:
            self._check(self.L.ref_frontier_trace(
                C.c_void_p(gF.h), C.c_void_p(gT.h), _ptr(ds, _u32p), _ptr(dd, _u32p), C.c_uint64(nd),
                _ptr(is_, _u32p), _ptr(id_, _u32p), C.c_uint64(ni), _ptr(prev, _dp), C.byref(cfg),
                C.c_int(int(pruning)), _ptr(ranks, _dp), C.byref(st), obs, None))
        else:
            self._check(getattr(self.L, self.p + "dynamic_frontier")(
                C.c_void_p(gF.h), C.c_void_p(gT.h), _ptr(ds, _u32p), _ptr(dd, _u32p), C.c_uint64(nd),
                _ptr(is_, _u32p), _ptr(id_, _u32p), C.c_uint64(ni), _ptr(prev, _dp),
                C.c_uint64(len(prev)), C.byref(cfg), C.c_int(int(pruning)), _ptr(ranks, _dp),
                C.byref(st), obs, None))
        return self._result(ranks[: gT.n], st, trace)

    def dynamic_frontier_from_flags(self, gF: Graph, gT: Graph, va, np_, prev, cfg: Config = None,
                                    pruning: bool = False, trace: Optional[list] = None) -> Result:
        cfg = cfg or default_config()
        va, np_, prev = _u8(va), _u8(np_), _f64(prev)
        ranks = np.zeros(max(gT.n, 1), np.float64)
        st = Stats()
        obs, keep = self._observer(trace, True)
        self._check(getattr(self.L, self.p + "dynamic_frontier_from_flags")(
            C.c_void_p(gF.h), C.c_void_p(gT.h), _ptr(va, _u8p), _ptr(np_, _u8p), C.c_uint64(len(va)),
            _ptr(prev, _dp), C.c_uint64(len(prev)), C.byref(cfg), C.c_int(int(pruning)),
            _ptr(ranks, _dp), C.byref(st), obs, None))
        return self._result(ranks[: gT.n], st, trace)

    def dynamic_traversal(self, gF: Graph, gT: Graph, dels, ins, prev, cfg: Config = None,
                          trace: Optional[list] = None) -> Result:
        """dynamicTraversal (engine.cpp:124-151)."""
        cfg = cfg or default_config()
        ds, dd = split_edges(dels)
        is_, id_ = split_edges(ins)
        nd, ni = len(ds), len(is_)
        z = np.zeros(1, np.uint32)
        ds, dd = (ds, dd) if nd else (z, z)
        is_, id_ = (is_, id_) if ni else (z, z)
        prev = _f64(prev)
        ranks = np.zeros(max(gT.n, 1), np.float64)
        st = Stats()
        obs, keep = self._observer(trace, False)
        self._check(getattr(self.L, self.p + "dynamic_traversal")(
            C.c_void_p(gF.h), C.c_void_p(gT.h), _ptr(ds, _u32p), _ptr(dd, _u32p), C.c_uint64(nd),
            _ptr(is_, _u32p), _ptr(id_, _u32p), C.c_uint64(ni), _ptr(prev, _dp), C.c_uint64(len(prev)),
            C.byref(cfg), _ptr(ranks, _dp), C.byref(st), obs, None))
        return self._result(ranks[: gT.n], st, trace)

    def mark_reachable(self, g: Graph, seeds) -> np.ndarray:
        """markReachable (frontier.cpp:86-121): vertexAffected bytes."""
        sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint32).reshape(-1))
        z = sd if len(sd) else np.zeros(1, np.uint32)
        va = np.zeros(max(g.n, 1), np.uint8)
        self._check(getattr(self.L, self.p + "mark_reachable")(
            C.c_void_p(g.h), _ptr(z, _u32p), C.c_uint64(len(sd)), _ptr(va, _u8p)))
        return va[: g.n]

    def compute_reference_ranks(self, gT: Graph, gF: Graph, cfg: Config = None):
        cfg = cfg or default_config()
        ranks = np.zeros(max(gT.n, 1), np.float64)
        self._check(getattr(self.L, self.p + "compute_reference_ranks")(
            C.c_void_p(gT.h), C.c_void_p(gF.h), C.byref(cfg), _ptr(ranks, _dp)))
        return ranks[: gT.n]

    # ---- input formats + harness (reference library only) ------------------
    def _edges_out(self, h):
        L = self.L
        L.ref_edges_count.restype = C.c_uint64
        L.ref_edges_vertex_count.restype = C.c_uint32
        for nm in ("ref_edges_count", "ref_edges_vertex_count", "ref_edges_free"):
            getattr(L, nm).argtypes = [_vp]
        L.ref_edges_copy.argtypes = [_vp, _vp, _vp, _vp]
        cnt = L.ref_edges_count(h)
        n = L.ref_edges_vertex_count(h)
        s = np.empty(max(cnt, 1), np.uint32)
        d = np.empty(max(cnt, 1), np.uint32)
        t = np.empty(max(cnt, 1), np.int64)
        L.ref_edges_copy(h, s.ctypes.data, d.ctypes.data, t.ctypes.data)
        L.ref_edges_free(h)
        return s[:cnt], d[:cnt], t[:cnt], n

    def _load(self, fn, path):
        fn.argtypes = [C.c_char_p, C.POINTER(_vp)]
        h = _vp()
        self._check(fn(str(path).encode(), C.byref(h)))
        return h.value

    def load_matrix_market(self, path):
        """loadMatrixMarket -> (src, dst, vertex_count)."""
        s, d, _, n = self._edges_out(self._load(self.L.ref_load_matrix_market, path))
        return s, d, n

    def load_temporal(self, path):
        """loadTemporalEdgeList -> (src, dst, timestamps, vertex_count)."""
        return self._edges_out(self._load(self.L.ref_load_temporal, path))

    def split_temporal(self, path, base_fraction, batch_count, batch_size):
        """splitTemporal -> ((base_src, base_dst), (batch_src, batch_dst) concatenated)."""
        h = self._load(self.L.ref_load_temporal, path)
        base, batches = _vp(), _vp()
        self.L.ref_split_temporal.argtypes = [_vp, C.c_double, C.c_int, C.c_uint64, C.POINTER(_vp),
                                              C.POINTER(_vp)]
        try:
            self._check(self.L.ref_split_temporal(h, base_fraction, batch_count, batch_size, C.byref(base),
                                                  C.byref(batches)))
        finally:
            self.L.ref_edges_free(h)
        bs, bd, _, _ = self._edges_out(base.value)
        s, d, _, _ = self._edges_out(batches.value)
        return (bs, bd), (s, d)

    def run_experiment(self, spec_struct, fmt: int, out_path: str):
        """runExperiment + emitReport; spec_struct is a dynpr_experiment_spec
        ctypes structure (paper_2404_08299_b200._native.ExperimentSpec)."""
        self.L.ref_run_experiment.argtypes = [_vp, C.c_int, C.c_char_p]
        self._check(self.L.ref_run_experiment(C.addressof(spec_struct), fmt, str(out_path).encode()))

    def summarize_emit(self, rows_array, count: int, summarize: bool, fmt: int, out_path: str):
        """summarizeRows (optional) + emitReport over a ctypes array of
        dynpr_experiment_row."""
        self.L.ref_summarize_emit.argtypes = [_vp, C.c_uint64, C.c_int, C.c_int, C.c_char_p]
        self._check(self.L.ref_summarize_emit(C.addressof(rows_array), count, int(summarize), fmt,
                                              str(out_path).encode()))


class PortRng:
    def __init__(self, lib: Oracle, seed: int):
        self.lib = lib
        self.state = seed

    def bounded(self, b: int) -> int:
        st = C.c_uint64(self.state)
        x = self.lib.L.orc_rng_bounded(C.byref(st), C.c_uint64(b))
        self.state = st.value
        return int(x)

    def next_double(self) -> float:
        st = C.c_uint64(self.state)
        x = self.lib.L.orc_rng_double(C.byref(st))
        self.state = st.value
        return float(x)


class RefRng:
    def __init__(self, lib: Oracle, seed: int):
        self.lib = lib
        self.h = lib.L.ref_rng_new(C.c_uint64(seed))

    def __del__(self):
        try:
            self.lib.L.ref_rng_free(C.c_void_p(self.h))
        except Exception:
            pass

    def bounded(self, b: int) -> int:
        return int(self.lib.L.ref_rng_bounded(C.c_void_p(self.h), C.c_uint64(b)))

    def next_double(self) -> float:
        return float(self.lib.L.ref_rng_next_double(C.c_void_p(self.h)))


# ---- bench input for the CPU arms (oracle/bench_input.c, OpenMP) ------------------
def _port_lib():
    L = C.CDLL(PORT_LIB)
    L.orc_par_rmat_edges.argtypes = [C.c_uint32, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                     _u32p, _u32p]
    L.orc_par_build_csr.argtypes = [C.c_uint32, _u32p, _u32p, C.c_uint64, C.c_int, _u64p, _u32p]
    L.orc_par_build_csr.restype = C.c_uint64
    L.orc_par_transpose.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, _u32p]
    return L


def par_rmat_csr(scale: int, edge_factor: int = 16, seed: int = 42, a=0.57, b=0.19, c=0.19):
    """RMAT forward CSR (buildCsr + addSelfLoops of edge_factor << scale
    pairs) built on all host cores: the bytes of Oracle("port").rmat_edges ->
    build_csr -> add_self_loops (and of the device generator), without the
    product library.  Returns (n, offsets u64[n+1], targets u32[m])."""
    L = _port_lib()
    n = 1 << scale
    count = edge_factor << scale
    src = np.empty(count, np.uint32)
    dst = np.empty(count, np.uint32)
    L.orc_par_rmat_edges(scale, count, a, b, c, seed, _ptr(src, _u32p), _ptr(dst, _u32p))
    off = np.empty(n + 1, np.uint64)
    tgt = np.empty(count + n, np.uint32)
    m = L.orc_par_build_csr(n, _ptr(src, _u32p), _ptr(dst, _u32p), count, 1, _ptr(off, _u64p), _ptr(tgt, _u32p))
    del src, dst
    return n, off, np.ascontiguousarray(tgt[:m])


def par_transpose(n: int, off, tgt):
    """transpose (graph.cpp:70-83) of a sorted, deduplicated CSR on all host cores."""
    L = _port_lib()
    off = np.ascontiguousarray(off, dtype=np.uint64)
    tgt = np.ascontiguousarray(tgt, dtype=np.uint32)
    toff = np.empty(n + 1, np.uint64)
    ttgt = np.empty(max(len(tgt), 1), np.uint32)
    L.orc_par_transpose(n, _ptr(off, _u64p), _ptr(tgt, _u32p), _ptr(toff, _u64p), _ptr(ttgt, _u32p))
    return toff, ttgt[: len(tgt)]


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


def dense_pagerank(off: np.ndarray, tgt: np.ndarray, n: int, alpha=0.85, tol=1e-14, max_iter=10000):
    """Restatement of tests/common/oracles.hpp:40-76 (dense power iteration)
    with numpy; used only as an independent ground truth in tests."""
    outdeg = np.diff(off).astype(np.float64)
    if np.any(outdeg == 0):
        raise ValueError("densePageRank: dangling vertex")
    M = np.zeros((n, n))
    src = np.repeat(np.arange(n), np.diff(off).astype(np.int64))
    M[tgt.astype(np.int64), src] = 1.0 / outdeg[src]
    r = np.full(n, 1.0 / n)
    tele = (1.0 - alpha) / n
    for _ in range(max_iter):
        nxt = tele + alpha * (M @ r)
        d = np.max(np.abs(nxt - r))
        r = nxt
        if d <= tol:
            break
    return r
