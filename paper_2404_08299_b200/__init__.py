"""B200-native Static and DF-P PageRank -- Python mirror of the reference's
``dynpr`` module (proj/python/dynpr/__init__.py, bindings/module.cpp).

Same names, argument order and meaning, and error behaviour as the
reference's pybind11 bindings (module.cpp:22-166): invalid arguments raise
``ValueError`` with the reference's message text.  Every graph is an
immutable device-resident CSR snapshot (``CsrGraph``); ranks come back as
numpy float64 arrays.  All compute runs in libdynpr_cuda.so's hand-written
sm_100a kernels through the C-ABI of include/dynpr_cuda.h; there is no CPU
fallback -- without the library or a GPU every call raises.

Argument-order note (reference engine.hpp:33-62): ``static_pagerank`` and
``naive_dynamic`` take ``(g_transpose, g_forward, ...)``; ``dynamic_frontier``
takes ``(g_forward, g_transpose, ...)``.
"""
from __future__ import annotations

import ctypes as C
import enum
import weakref
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import NativeUnavailable

__all__ = [
    "BatchUpdate", "BatchApplyStats", "EdgeArray", "Context", "CsrGraph", "DegreePartition", "EngineConfig",
    "PartitionStrategy", "RankMode", "RankResult", "SizingError", "NativeUnavailable",
    "add_self_loops", "apply_batch", "apply_batch_pair", "build_csr", "default_context",
    "dynamic_frontier", "dynamic_frontier_from_flags", "expand_affected", "initial_affected",
    "l1_norm_delta", "linf_norm_delta", "naive_dynamic", "partition_by_degree", "rmat_graph",
    "static_pagerank", "transpose", "update_ranks", "generate_random_batch", "batch_size_from_fraction",
    "derive_seed", "prepare", "LocalTeam", "nccl_unique_id", "share_nccl_unique_id",
    "context_from_process_group", "attach_symmetric_exchange", "TorchDistTransport", "IpcExchange", "layout_info", "dynamic_traversal", "mark_reachable",
    "ParseError", "Approach", "ExperimentMode", "ChainMode", "ReportFormat", "ExperimentRow", "ExperimentSpec",
    "approach_name", "approach_from_name", "load_matrix_market", "load_matrix_market_arrays",
    "load_temporal_edge_list", "load_temporal_edge_list_arrays", "split_temporal", "compute_reference_ranks",
    "run_experiment", "summarize_rows", "emit_report",
]


class SizingError(ValueError):
    """dynpr::SizingError (workload.hpp:17-19); a ValueError like in module.cpp:165."""


class PartitionStrategy(enum.IntEnum):  # rank.hpp:14-18
    DONT_PARTITION = 0
    PARTITION_TRANSPOSE = 1
    PARTITION_BOTH = 2


class RankMode(enum.IntEnum):  # rank.hpp:23
    PLAIN = 0
    CLOSED_LOOP_PRUNE = 1


@dataclass
class EngineConfig:  # rank.hpp:25-39, defaults
    damping_factor: float = 0.85
    iteration_tolerance: float = 1e-10
    frontier_tolerance: float = 1e-6
    prune_tolerance: float = 1e-6
    max_iterations: int = 500
    low_degree_threshold: int = 32
    partition_strategy: PartitionStrategy = PartitionStrategy.PARTITION_BOTH
    convergence_check_disabled: bool = False

    def _c(self) -> N.Config:
        return N.Config(float(self.damping_factor), float(self.iteration_tolerance),
                        float(self.frontier_tolerance), float(self.prune_tolerance),
                        int(self.max_iterations), int(self.low_degree_threshold),
                        int(self.partition_strategy), int(bool(self.convergence_check_disabled)))

    def validate(self) -> None:
        """EngineConfig::validate (rank.cpp:11-20); raises ValueError."""
        c = self._c()
        _check(N.lib().dynpr_config_validate(C.byref(c)))


@dataclass
class RankResult:  # engine.hpp:16-22
    ranks: np.ndarray
    iterations: int
    affected_vertex_iterations: int
    converged: bool
    final_delta: float
    processed_edges: int = 0
    device_ms: float = 0.0


@dataclass
class DegreePartition:  # partition.hpp:12-15
    order: np.ndarray
    low_count: int


class EdgeArray:
    """An EdgeList (graph.hpp:10, a list of (source, target) pairs in the
    reference's Python binding) held as two uint32 arrays: it compares,
    indexes and iterates like the reference's list of tuples, while the
    engines take `src` / `dst` without a conversion."""

    __slots__ = ("src", "dst")

    def __init__(self, src, dst):
        self.src = np.ascontiguousarray(np.asarray(src, dtype=np.uint32).reshape(-1))
        self.dst = np.ascontiguousarray(np.asarray(dst, dtype=np.uint32).reshape(-1))
        if len(self.src) != len(self.dst):
            raise ValueError("EdgeArray: src and dst lengths differ")

    def __len__(self):
        return len(self.src)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return EdgeArray(self.src[i], self.dst[i])
        return (int(self.src[i]), int(self.dst[i]))

    def __iter__(self):
        return iter(zip(self.src.tolist(), self.dst.tolist()))

    def tolist(self):
        return list(zip(self.src.tolist(), self.dst.tolist()))

    def __eq__(self, other):
        if isinstance(other, EdgeArray):
            return np.array_equal(self.src, other.src) and np.array_equal(self.dst, other.dst)
        try:
            return self.tolist() == [tuple(x) for x in other]
        except TypeError:
            return NotImplemented

    __hash__ = None

    def __repr__(self):
        head = ", ".join(f"({u}, {v})" for u, v in zip(self.src[:4].tolist(), self.dst[:4].tolist()))
        return f"EdgeArray([{head}{', ...' if len(self) > 4 else ''}], len={len(self)})"


@dataclass
class BatchUpdate:  # graph.hpp:54-57
    deletions: object = field(default_factory=list)
    insertions: object = field(default_factory=list)


@dataclass
class BatchApplyStats:  # graph.hpp:61-64
    missing_deletions: int = 0
    duplicate_insertions: int = 0


def _check(rc: int) -> None:
    if rc == N.DYNPR_OK:
        return
    msg = N.last_error()
    if rc == N.DYNPR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == N.DYNPR_SIZING_ERROR:
        raise SizingError(msg)
    if rc == N.DYNPR_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(msg)


class Context:
    """One CUDA device + stream + workspace (dynpr_context).

    A plain context solves on its own GPU.  `Context.nccl(...)` (one process
    per GPU) and `LocalTeam(world).context(...)` (virtual ranks on host
    threads of one process) create contexts of a range-partitioned team: the
    engines are then called SPMD with the same graphs and inputs on every
    rank, each rank sweeps its edge-balanced vertex range, and the
    contributions / pending flags are all-gathered after every sweep
    (SURVEY 8e).  Every rank returns the full result."""

    def __init__(self, device: int = 0, _handle: Optional[int] = None, _keep=None):
        if _handle is None:
            h = C.c_void_p()
            _check(N.lib().dynpr_context_create(int(device), C.byref(h)))
            _handle = h.value
        self.h = _handle
        self.device = device
        self._keep = _keep  # a LocalTeam must outlive its contexts
        self._fin = weakref.finalize(self, N.lib().dynpr_context_destroy, C.c_void_p(self.h))

    @classmethod
    def nccl(cls, device: int, rank: int, world: int, unique_id: bytes) -> "Context":
        """Rank `rank` of a `world`-GPU team joined through NCCL (unique_id
        from nccl_unique_id() on rank 0, shared out of band)."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(N.lib().dynpr_context_create_nccl(int(device), int(rank), int(world), buf, C.byref(h)))
        return cls(device, _handle=h.value)

    @classmethod
    def hostcomm(cls, device: int, transport: "TorchDistTransport") -> "Context":
        """Rank `transport.rank` of a team whose collectives go through a host
        transport (dynpr_context_create_hostcomm) -- any number of processes,
        several per GPU allowed."""
        h = C.c_void_p()
        _check(N.lib().dynpr_context_create_hostcomm(int(device), int(transport.rank), int(transport.world),
                                                     C.byref(transport.ops), None, C.byref(h)))
        return cls(device, _handle=h.value, _keep=transport)

    def attach_peers(self, ptrs0: Sequence[int], ptrs1: Sequence[int], capacity: int) -> None:
        """Fused exchange: every rank's two contribution buffers (device
        addresses valid in this process, `capacity` doubles each); [] detaches.
        See dynpr_context_attach_peers."""
        world = len(ptrs0)
        a0 = (C.c_uint64 * max(world, 1))(*[int(p) for p in ptrs0])
        a1 = (C.c_uint64 * max(world, 1))(*[int(p) for p in ptrs1])
        _check(N.lib().dynpr_context_attach_peers(C.c_void_p(self.h), world, a0, a1, int(capacity)))

    @property
    def rank(self) -> int:
        r, w = C.c_int(), C.c_int()
        _check(N.lib().dynpr_context_rank(C.c_void_p(self.h), C.byref(r), C.byref(w)))
        return r.value

    @property
    def world(self) -> int:
        r, w = C.c_int(), C.c_int()
        _check(N.lib().dynpr_context_rank(C.c_void_p(self.h), C.byref(r), C.byref(w)))
        return w.value

    @property
    def launches(self) -> int:
        return int(N.lib().dynpr_context_launches(C.c_void_p(self.h)))

    def set_profiling(self, enable: bool) -> None:
        _check(N.lib().dynpr_context_set_profiling(C.c_void_p(self.h), int(enable)))

    def sweep_times(self):
        ms, sw, by = C.c_double(), C.c_uint64(), C.c_uint64()
        _check(N.lib().dynpr_context_sweep_times(C.c_void_p(self.h), C.byref(ms), C.byref(sw), C.byref(by)))
        return ms.value, sw.value, by.value


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId on this process (rank 0 of an NCCL team)."""
    buf = (C.c_uint8 * 128)()
    _check(N.lib().dynpr_nccl_get_unique_id(buf))
    return bytes(buf)


def share_nccl_unique_id(group=None) -> bytes:
    """Rank 0 of a torch.distributed process group (any backend) creates the
    NCCL unique id and broadcasts it; every rank returns the same 128 bytes."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def attach_symmetric_exchange(ctx: Context, n: int, group=None):
    """Allocates the two n-double contribution buffers of every rank in
    torch symmetric memory (CUDA IPC handles exchanged over the process
    group), maps all peers' buffers and attaches them to `ctx` (fused
    NVLink exchange).  Returns the tensors/handles, which must stay alive
    while the context solves."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    group = group or dist.group.WORLD
    keep = []
    ptrs = []
    for _ in range(2):
        t = symm_mem.empty(max(n, 1), dtype=torch.float64, device=f"cuda:{ctx.device}")
        h = symm_mem.rendezvous(t, group)
        keep.append((t, h))
        ptrs.append([int(p) for p in h.buffer_ptrs])
    ctx.attach_peers(ptrs[0], ptrs[1], max(n, 1))
    return keep


def context_from_process_group(device: int, group=None, transport: str = "nccl") -> Context:
    """One process per GPU (torchrun): this process's rank of a team spanning
    the torch.distributed process group -- over NCCL (default), or with
    transport="host" over the group itself (TorchDistTransport: gloo/MPI,
    several processes per GPU allowed)."""
    import torch.distributed as dist
    if transport == "host":
        return Context.hostcomm(device, TorchDistTransport(group))
    if transport != "nccl":
        raise ValueError(f"unknown transport {transport!r}")
    uid = share_nccl_unique_id(group)
    return Context.nccl(device, dist.get_rank(group), dist.get_world_size(group), uid)


class TorchDistTransport:
    """dynpr_comm_ops over a torch.distributed process group whose backend
    takes CPU tensors (gloo, or MPI): the host transport of
    `Context.hostcomm`.  Collectives run on the thread that called the engine,
    in the same order on every rank.  The callbacks must not raise into C: a
    failure is recorded in `error` and returned as a nonzero status, which
    the engine turns into a RuntimeError."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.error: Optional[str] = None
        self.calls = 0
        self.ops = N.CommOps(N.ALLREDUCE_U64(self._allreduce), N.ALLGATHERV(self._allgatherv),
                             N.BARRIER(self._barrier))

    def _guard(self, fn) -> int:
        try:
            self.calls += 1
            fn()
            return 0
        except Exception:  # noqa: BLE001 -- reported through the engine's status
            import traceback
            self.error = traceback.format_exc()
            return 1

    def _allreduce(self, data, count, op, _user):
        def run():
            import torch
            import torch.distributed as dist
            view = np.ctypeslib.as_array(data, shape=(int(count),))
            mine = torch.from_numpy(view.copy().view(np.int64))
            parts = [torch.empty_like(mine) for _ in range(self.world)]
            dist.all_gather(parts, mine, group=self.group)
            st = np.stack([p.numpy().view(np.uint64) for p in parts])
            view[:] = st.max(axis=0) if op == 1 else st.sum(axis=0, dtype=np.uint64)  # mod 2^64
        return self._guard(run)

    def _allgatherv(self, buf, offsets, world, _user):
        def run():
            import torch
            import torch.distributed as dist
            off = [int(offsets[i]) for i in range(world + 1)]
            host = np.ctypeslib.as_array((C.c_uint8 * max(off[-1], 1)).from_address(buf))
            sizes = [off[r + 1] - off[r] for r in range(world)]
            width = max(max(sizes), 1)
            send = torch.zeros(width, dtype=torch.uint8)
            me = self.rank
            send[:sizes[me]] = torch.from_numpy(host[off[me]:off[me + 1]].copy())
            parts = [torch.empty(width, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, send, group=self.group)
            for r in range(world):
                if r != me and sizes[r]:
                    host[off[r]:off[r + 1]] = parts[r].numpy()[:sizes[r]]
        return self._guard(run)

    def _barrier(self, _user):
        def run():
            import torch.distributed as dist
            dist.barrier(group=self.group)
        return self._guard(run)


class IpcExchange:
    """The fused exchange across processes without torch symmetric memory:
    each rank's two contribution buffers are CUDA IPC allocations of this
    library, their handles all-gathered over the process group and mapped by
    every rank (peers on the same or another GPU), then attached to the
    context.  Keep the object alive while the context solves; close() (or
    garbage collection) detaches, unmaps and frees in that order."""

    def __init__(self, ctx: "Context", n: int, group=None):
        import torch.distributed as dist
        self.ctx = ctx
        self.group = group
        self.own = []
        self.opened = []
        handles = []
        lib = N.lib()
        for _ in range(2):
            p = C.c_void_p()
            h = (C.c_uint8 * 64)()
            _check(lib.dynpr_ipc_alloc(C.c_void_p(ctx.h), 8 * max(n, 1), C.byref(p), h))
            self.own.append(p.value)
            handles.append(bytes(h))
        allh = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, handles, group=group)
        me = dist.get_rank(group)
        ptrs = [[], []]
        for r, hs in enumerate(allh):
            for k in range(2):
                if r == me:
                    ptrs[k].append(self.own[k])
                    continue
                p = C.c_void_p()
                _check(lib.dynpr_ipc_open(C.c_void_p(ctx.h), (C.c_uint8 * 64).from_buffer_copy(hs[k]), C.byref(p)))
                self.opened.append(p.value)
                ptrs[k].append(p.value)
        ctx.attach_peers(ptrs[0], ptrs[1], max(n, 1))

    def close(self) -> None:
        if self.ctx is None:
            return
        import torch.distributed as dist
        lib = N.lib()
        self.ctx.attach_peers([], [], 0)
        for p in self.opened:
            _check(lib.dynpr_ipc_close(C.c_void_p(self.ctx.h), C.c_void_p(p)))
        dist.barrier(group=self.group)  # every peer unmapped before the owners free
        for p in self.own:
            _check(lib.dynpr_ipc_free(C.c_void_p(self.ctx.h), C.c_void_p(p)))
        self.ctx = None


class LocalTeam:
    """`world` virtual ranks of the partitioned engine inside one process
    (any devices, typically one GPU): the single-GPU test harness of the
    multi-GPU path.  Each rank's engine call must run on its own host
    thread (the calls meet at barriers)."""

    def __init__(self, world: int):
        h = C.c_void_p()
        _check(N.lib().dynpr_team_create(int(world), C.byref(h)))
        self.h = h.value
        self.world = world
        self._fin = weakref.finalize(self, N.lib().dynpr_team_destroy, C.c_void_p(self.h))

    def context(self, device: int, rank: int) -> Context:
        h = C.c_void_p()
        _check(N.lib().dynpr_context_create_team(int(device), C.c_void_p(self.h), int(rank), C.byref(h)))
        return Context(device, _handle=h.value, _keep=self)


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else default_context()


# ---- array plumbing ------------------------------------------------------------
def _arr(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=dtype).reshape(-1))


def _edges(edges):
    """EdgeArray | [(u, v), ...] | (src, dst) arrays | (k, 2) array -> uint32 src, dst."""
    if isinstance(edges, EdgeArray):
        return edges.src, edges.dst
    if isinstance(edges, tuple) and len(edges) == 2 and not np.isscalar(edges[0]) and \
            isinstance(edges[0], np.ndarray):
        return _arr(edges[0], np.uint32), _arr(edges[1], np.uint32)
    if isinstance(edges, np.ndarray):
        a = edges.reshape(-1, 2)
    else:
        lst = list(edges)
        if not lst:
            return np.zeros(0, np.uint32), np.zeros(0, np.uint32)
        a = np.asarray(lst, dtype=np.int64).reshape(-1, 2)
    if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
        raise ValueError("vertex id out of uint32 range")
    return _arr(a[:, 0], np.uint32), _arr(a[:, 1], np.uint32)


def _p(a: Optional[np.ndarray]):
    if a is None or a.size == 0:
        return None
    return C.c_void_p(a.ctypes.data)


def _is_device_array(x) -> bool:
    return getattr(x, "__cuda_array_interface__", None) is not None


_TYPESTR = {np.float64: "<f8", np.uint8: "|u1", np.uint32: "<u4"}


def _in_array(x, dtype):
    """(pointer, length, keep-alive) of an input array.  Device arrays
    (anything exposing __cuda_array_interface__: torch CUDA tensors, CuPy)
    are passed to the C-ABI as device pointers -- no host round trip; the
    library detects device memory itself (dynpr_cuda.h conventions)."""
    cai = getattr(x, "__cuda_array_interface__", None)
    if cai is not None:
        if cai.get("typestr") != _TYPESTR[dtype]:
            raise ValueError(f"device array must have dtype {np.dtype(dtype).name}")
        if cai.get("strides") not in (None, ()):
            shape = cai["shape"]
            itemsize = np.dtype(dtype).itemsize
            if len(shape) != 1 or cai["strides"][0] != itemsize:
                raise ValueError("device array must be contiguous")
        n = int(np.prod(cai["shape"])) if cai["shape"] else 1
        return (C.c_void_p(cai["data"][0]) if n else None), n, x
    a = _arr(x, dtype)
    return _p(a), len(a), a


def _out_ranks(out, n: int):
    """(pointer, result array) for an engine's ranks: a fresh numpy array, or
    the caller's device array `out` (n float64) so chained solves never
    leave the GPU."""
    if out is None:
        r = np.empty(max(n, 1), np.float64)  # every entry is written
        return _p(r), r
    ptr, length, keep = _in_array(out, np.float64)
    if length != n:
        raise ValueError("out must hold exactly vertex_count float64 values")
    return ptr, keep


class CsrGraph:
    """Immutable device CSR snapshot (graph.hpp:17-49); host arrays are
    downloaded lazily and cached."""

    def __init__(self, handle: int, ctx: Context):
        self.h = handle
        self.ctx = ctx
        n, m = C.c_uint32(), C.c_uint64()
        _check(N.lib().dynpr_graph_info(C.c_void_p(handle), C.byref(n), C.byref(m)))
        self._n, self._m = n.value, m.value
        self._host = None
        self._fin = weakref.finalize(self, N.lib().dynpr_graph_destroy, C.c_void_p(handle))

    @classmethod
    def from_csr(cls, vertex_count: int, offsets, targets, ctx: Optional[Context] = None) -> "CsrGraph":
        """CsrGraph(vertexCount, offsets, targets) with full validation."""
        ctx = _ctx(ctx)
        off = _arr(offsets, np.uint64)
        tgt = _arr(targets, np.uint32)
        if len(off) != int(vertex_count) + 1:
            raise ValueError("CsrGraph: malformed offsets array")
        h = C.c_void_p()
        _check(N.lib().dynpr_graph_from_csr(C.c_void_p(ctx.h), int(vertex_count), _p(off), _p(tgt),
                                            len(tgt), C.byref(h)))
        return cls(h.value, ctx)

    @property
    def vertex_count(self) -> int:
        return self._n

    @property
    def edge_count(self) -> int:
        return self._m

    def _download(self):
        if self._host is None:
            off = np.zeros(self._n + 1, np.uint64)
            tgt = np.zeros(max(self._m, 1), np.uint32)
            _check(N.lib().dynpr_graph_download(C.c_void_p(self.ctx.h), C.c_void_p(self.h),
                                                _p(off), _p(tgt)))
            self._host = (off, tgt[: self._m])
        return self._host

    @property
    def offsets(self) -> np.ndarray:
        return self._download()[0]

    @property
    def targets(self) -> np.ndarray:
        return self._download()[1]

    def degree(self, v: int) -> int:
        off = self.offsets
        return int(off[v + 1] - off[v])

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets).astype(np.uint32)

    def out(self, v: int) -> list:
        off, tgt = self._download()
        return tgt[int(off[v]):int(off[v + 1])].tolist()

    def has_edge(self, source: int, target: int) -> bool:
        out = C.c_int()
        _check(N.lib().dynpr_graph_has_edge(C.c_void_p(self.ctx.h), C.c_void_p(self.h), int(source),
                                            int(target), C.byref(out)))
        return bool(out.value)

    def has_self_loop(self, v: int) -> bool:
        return self.has_edge(v, v)

    def __eq__(self, other) -> bool:  # bytewise (graph.hpp:43)
        if not isinstance(other, CsrGraph):
            return NotImplemented
        if self._n != other._n or self._m != other._m:
            return False
        return bool(np.array_equal(self.offsets, other.offsets) and np.array_equal(self.targets, other.targets))

    def __repr__(self) -> str:
        return f"<CsrGraph |V|={self._n} |E|={self._m}>"


def _new_graph(fn, ctx: Context, *args) -> CsrGraph:
    h = C.c_void_p()
    _check(fn(C.c_void_p(ctx.h), *args, C.byref(h)))
    return CsrGraph(h.value, ctx)


# ---- graph construction (graph.hpp:66-80) -------------------------------------
def build_csr(edges, vertex_count: int, ctx: Optional[Context] = None) -> CsrGraph:
    ctx = _ctx(ctx)
    s, d = _edges(edges)
    return _new_graph(N.lib().dynpr_graph_build, ctx, int(vertex_count), _p(s), _p(d), len(s))


def transpose(g: CsrGraph) -> CsrGraph:
    return _new_graph(N.lib().dynpr_graph_transpose, g.ctx, C.c_void_p(g.h))


def add_self_loops(g: CsrGraph) -> CsrGraph:
    return _new_graph(N.lib().dynpr_graph_add_self_loops, g.ctx, C.c_void_p(g.h))


def _batch_arrays(batch: BatchUpdate):
    ds, dd = _edges(batch.deletions)
    is_, id_ = _edges(batch.insertions)
    return ds, dd, is_, id_


def apply_batch(g: CsrGraph, batch: BatchUpdate, stats: Optional[BatchApplyStats] = None) -> CsrGraph:
    ds, dd, is_, id_ = _batch_arrays(batch)
    miss, dup = C.c_uint64(0), C.c_uint64(0)
    h = C.c_void_p()
    _check(N.lib().dynpr_graph_apply_batch(C.c_void_p(g.ctx.h), C.c_void_p(g.h), _p(ds), _p(dd), len(ds),
                                           _p(is_), _p(id_), len(is_), C.byref(h), C.byref(miss), C.byref(dup)))
    if stats is not None:
        stats.missing_deletions += miss.value
        stats.duplicate_insertions += dup.value
    return CsrGraph(h.value, g.ctx)


def apply_batch_pair(g: CsrGraph, gt: CsrGraph, batch: BatchUpdate,
                     stats: Optional[BatchApplyStats] = None):
    """Device batch ingest of a (forward, transpose) pair: returns
    (applyBatch(g), transpose(applyBatch(g))) without a re-transpose."""
    ds, dd, is_, id_ = _batch_arrays(batch)
    miss, dup = C.c_uint64(0), C.c_uint64(0)
    hf, ht = C.c_void_p(), C.c_void_p()
    _check(N.lib().dynpr_graph_apply_batch_pair(C.c_void_p(g.ctx.h), C.c_void_p(g.h), C.c_void_p(gt.h),
                                                _p(ds), _p(dd), len(ds), _p(is_), _p(id_), len(is_),
                                                C.byref(hf), C.byref(ht), C.byref(miss), C.byref(dup)))
    if stats is not None:
        stats.missing_deletions += miss.value
        stats.duplicate_insertions += dup.value
    return CsrGraph(hf.value, g.ctx), CsrGraph(ht.value, g.ctx)


def prepare(g_transpose: CsrGraph, g_forward: CsrGraph, config: Optional[EngineConfig] = None,
            frontier: bool = True) -> float:
    """Build (and cache on g_transpose) the engine layout of the pair: the
    device graph format the sweeps read (see include/dynpr_cuda.h).  Returns
    the build's device milliseconds.  Engines build it on demand otherwise."""
    cfg = config or EngineConfig()
    ms = C.c_double()
    _check(N.lib().dynpr_graph_prepare(C.c_void_p(g_transpose.ctx.h), C.c_void_p(g_transpose.h),
                                       C.c_void_p(g_forward.h), int(cfg.low_degree_threshold), int(frontier),
                                       C.byref(ms)))
    return ms.value


def layout_info(g_transpose: CsrGraph) -> dict:
    """The engine layout cached on a transpose graph (dynpr_graph_layout_info):
    SELL words held by its context, the owned vertex range in relabelled
    order, whether the relabelled forward CSR is built, and the generation
    (0 = built from scratch, k = derived incrementally k batches after)."""
    w, lo, hi, fw, gen = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_int(), C.c_int()
    _check(N.lib().dynpr_graph_layout_info(C.c_void_p(g_transpose.h), C.byref(w), C.byref(lo), C.byref(hi),
                                           C.byref(fw), C.byref(gen)))
    return {"sell_words": w.value, "v_lo": lo.value, "v_hi": hi.value, "has_forward": bool(fw.value),
            "generation": gen.value}


def rmat_graph(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
               seed: int = 42, ctx: Optional[Context] = None) -> CsrGraph:
    """Self-loop-augmented RMAT/Kronecker graph generated on the device
    (Graph500 parameters; counter-based SplitMix64 seeding)."""
    ctx = _ctx(ctx)
    return _new_graph(N.lib().dynpr_graph_rmat, ctx, int(scale), int(edge_factor), float(a), float(b),
                      float(c), int(seed))


def kronecker_graph(scale: int, edge_factor: int = 16, seed: int = 42, ctx: Optional[Context] = None) -> CsrGraph:
    """Graph500-style Kronecker graph generated on the device: the RMAT draws
    of rmat_graph with the Graph500 initiator, vertex ids scrambled by a
    seeded bijection (dynpr_graph_kronecker), self-loops added."""
    ctx = _ctx(ctx)
    return _new_graph(N.lib().dynpr_graph_kronecker, ctx, int(scale), int(edge_factor), int(seed))


# ---- workload (workload.hpp:189-197) --------------------------------------------
def batch_size_from_fraction(fraction: float, total: int) -> int:
    return int(N.lib().dynpr_batch_size_from_fraction(float(fraction), int(total)))


def derive_seed(seed: int, stream: int) -> int:
    return int(N.lib().dynpr_derive_seed(int(seed), int(stream)))


def generate_random_batch(g: CsrGraph, total_size: int, insert_fraction: float = 0.8,
                          seed: int = 1) -> BatchUpdate:
    """generateRandomBatch (workload.cpp:183-243): identical draws to the
    reference; deletions/insertions come back as (src, dst) uint32 arrays."""
    cap = max(int(total_size), 1)
    is_, id_ = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
    ds, dd = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
    ni, nd = C.c_uint64(), C.c_uint64()
    _check(N.lib().dynpr_generate_random_batch(C.c_void_p(g.ctx.h), C.c_void_p(g.h), int(total_size),
                                               float(insert_fraction), int(seed), _p(is_), _p(id_),
                                               C.byref(ni), _p(ds), _p(dd), C.byref(nd)))
    return BatchUpdate(deletions=EdgeArray(ds[: nd.value], dd[: nd.value]),
                       insertions=EdgeArray(is_[: ni.value], id_[: ni.value]))


# ---- primitives ------------------------------------------------------------------
def partition_by_degree(g: CsrGraph, threshold: int) -> DegreePartition:
    order = np.zeros(max(g.vertex_count, 1), np.uint32)
    low = C.c_uint32()
    _check(N.lib().dynpr_partition_by_degree(C.c_void_p(g.ctx.h), C.c_void_p(g.h), int(threshold),
                                             _p(order), C.byref(low)))
    return DegreePartition(order[: g.vertex_count], low.value)


def update_ranks(gt: CsrGraph, g: CsrGraph, previous, current=None, vertex_affected=None,
                 neighbors_pending=None, config: Optional[EngineConfig] = None,
                 mode: RankMode = RankMode.PLAIN):
    """One sweep of updateRanks (rank.cpp:79-140).  Returns
    (current, vertex_affected, neighbors_pending) (flags None when not given)."""
    cfg = (config or EngineConfig())._c()
    n = gt.vertex_count
    prev = _arr(previous, np.float64)
    cur = np.array(prev if current is None else _arr(current, np.float64), dtype=np.float64)
    va = np_ = None
    if vertex_affected is not None:
        va = _arr(vertex_affected, np.uint8).copy()
        np_ = _arr(neighbors_pending if neighbors_pending is not None else np.zeros(n, np.uint8),
                   np.uint8).copy()
    if len(prev) != n:
        raise ValueError("updateRanks: previous length mismatch")
    _check(N.lib().dynpr_update_ranks(C.c_void_p(gt.ctx.h), C.c_void_p(gt.h), C.c_void_p(g.h), _p(va), _p(np_),
                                      _p(prev), _p(cur), C.byref(cfg), int(mode)))
    return cur, va, np_


def linf_norm_delta(a, b, ctx: Optional[Context] = None) -> float:
    a, b = _arr(a, np.float64), _arr(b, np.float64)
    if len(a) != len(b):
        raise ValueError("linfNormDelta: length mismatch")
    out = C.c_double()
    _check(N.lib().dynpr_linf_norm_delta(C.c_void_p(_ctx(ctx).h), _p(a), _p(b), len(a), C.byref(out)))
    return out.value


def l1_norm_delta(a, b, ctx: Optional[Context] = None) -> float:
    a, b = _arr(a, np.float64), _arr(b, np.float64)
    if len(a) != len(b):
        raise ValueError("l1NormDelta: length mismatch")
    out = C.c_double()
    _check(N.lib().dynpr_l1_norm_delta(C.c_void_p(_ctx(ctx).h), _p(a), _p(b), len(a), C.byref(out)))
    return out.value


def initial_affected(g: CsrGraph, deletions, insertions):
    """initialAffected (frontier.cpp:33-53) -> (vertex_affected, neighbors_pending)."""
    ds, dd = _edges(deletions)
    is_, id_ = _edges(insertions)
    n = g.vertex_count
    va = np.zeros(max(n, 1), np.uint8)
    np_ = np.zeros(max(n, 1), np.uint8)
    _check(N.lib().dynpr_initial_affected(C.c_void_p(g.ctx.h), C.c_void_p(g.h), _p(ds), _p(dd), len(ds),
                                          _p(is_), _p(id_), len(is_), _p(va), _p(np_)))
    return va[:n], np_[:n]


def expand_affected(g: CsrGraph, vertex_affected, neighbors_pending, threshold: int = 32) -> np.ndarray:
    """expandAffected (frontier.cpp:55-84): returns the expanded vertexAffected."""
    va = _arr(vertex_affected, np.uint8).copy()
    np_ = _arr(neighbors_pending, np.uint8)
    if len(va) != g.vertex_count or len(np_) != g.vertex_count:
        raise ValueError("expandAffected: flags length mismatch")
    _check(N.lib().dynpr_expand_affected(C.c_void_p(g.ctx.h), C.c_void_p(g.h), _p(va), _p(np_),
                                         int(threshold)))
    return va


# ---- engines (engine.hpp:33-71) --------------------------------------------------
def _observer(cb: Optional[Callable]):
    if cb is None:
        return N.OBSERVER(0), None

    def obs(it, ranks, processed, n, user):
        r = np.ctypeslib.as_array(ranks, shape=(n,)).copy()
        if processed:
            cb(it, r, np.ctypeslib.as_array(processed, shape=(n,)).copy())
        else:
            cb(it, r)

    fn = N.OBSERVER(obs)
    return fn, fn


def _result(ranks: np.ndarray, st: N.Stats) -> RankResult:
    return RankResult(ranks, st.iterations, st.affected_vertex_iterations, bool(st.converged),
                      st.final_delta, st.processed_edges, st.device_ms)


def static_pagerank(g_transpose: CsrGraph, g_forward: CsrGraph, config: Optional[EngineConfig] = None,
                    observer: Optional[Callable] = None, out=None) -> RankResult:
    """staticPageRank(gTranspose, gForward, cfg) -- engine.cpp:99-108.
    `out`: optional device array (n float64) that receives the ranks."""
    cfg = (config or EngineConfig())._c()
    rp, ranks = _out_ranks(out, g_transpose.vertex_count)
    st = N.Stats()
    obs, keep = _observer(observer)
    _check(N.lib().dynpr_static_pagerank(C.c_void_p(g_transpose.ctx.h), C.c_void_p(g_transpose.h),
                                         C.c_void_p(g_forward.h), C.byref(cfg), rp, C.byref(st), obs,
                                         None))
    return _result(ranks[: g_transpose.vertex_count], st)


def naive_dynamic(g_transpose: CsrGraph, g_forward: CsrGraph, previous_ranks,
                  config: Optional[EngineConfig] = None, observer: Optional[Callable] = None,
                  out=None) -> RankResult:
    """naiveDynamic(gTranspose, gForward, previousRanks, cfg) -- engine.cpp:110-122.
    previous_ranks / out may be device arrays."""
    cfg = (config or EngineConfig())._c()
    pp, plen, pkeep = _in_array(previous_ranks, np.float64)
    rp, ranks = _out_ranks(out, g_transpose.vertex_count)
    st = N.Stats()
    obs, keep = _observer(observer)
    _check(N.lib().dynpr_naive_dynamic(C.c_void_p(g_transpose.ctx.h), C.c_void_p(g_transpose.h),
                                       C.c_void_p(g_forward.h), pp, plen, C.byref(cfg), rp,
                                       C.byref(st), obs, None))
    return _result(ranks[: g_transpose.vertex_count], st)


def dynamic_frontier(g_forward: CsrGraph, g_transpose: CsrGraph, deletions, insertions, previous_ranks,
                     config: Optional[EngineConfig] = None, pruning: bool = False,
                     observer: Optional[Callable] = None, out=None) -> RankResult:
    """dynamicFrontier(gForward, gTranspose, dels, ins, prev, cfg, pruning) --
    engine.cpp:192-203 (DF-P with pruning=True).  The observer, when given,
    receives (iteration, ranks, processed_flags)."""
    cfg = (config or EngineConfig())._c()
    ds, dd = _edges(deletions)
    is_, id_ = _edges(insertions)
    pp, plen, pkeep = _in_array(previous_ranks, np.float64)
    rp, ranks = _out_ranks(out, g_transpose.vertex_count)
    st = N.Stats()
    obs, keep = _observer(observer)
    _check(N.lib().dynpr_dynamic_frontier(C.c_void_p(g_forward.ctx.h), C.c_void_p(g_forward.h),
                                          C.c_void_p(g_transpose.h), _p(ds), _p(dd), len(ds), _p(is_), _p(id_),
                                          len(is_), pp, plen, C.byref(cfg), int(bool(pruning)),
                                          rp, C.byref(st), obs, None))
    return _result(ranks[: g_transpose.vertex_count], st)


def dynamic_traversal(g_forward: CsrGraph, g_transpose: CsrGraph, deletions, insertions, previous_ranks,
                      config: Optional[EngineConfig] = None, observer: Optional[Callable] = None,
                      out=None) -> RankResult:
    """dynamicTraversal(gForward, gTranspose, dels, ins, prev, cfg) --
    engine.cpp:124-151: every vertex reachable from an update endpoint
    (device BFS) is processed every sweep; no expansion, no pruning."""
    cfg = (config or EngineConfig())._c()
    ds, dd = _edges(deletions)
    is_, id_ = _edges(insertions)
    pp, plen, pkeep = _in_array(previous_ranks, np.float64)
    rp, ranks = _out_ranks(out, g_transpose.vertex_count)
    st = N.Stats()
    obs, keep = _observer(observer)
    _check(N.lib().dynpr_dynamic_traversal(C.c_void_p(g_forward.ctx.h), C.c_void_p(g_forward.h),
                                           C.c_void_p(g_transpose.h), _p(ds), _p(dd), len(ds), _p(is_), _p(id_),
                                           len(is_), pp, plen, C.byref(cfg), rp, C.byref(st),
                                           obs, None))
    return _result(ranks[: g_transpose.vertex_count], st)


def mark_reachable(g: CsrGraph, seeds) -> np.ndarray:
    """markReachable(g, seeds) -- frontier.cpp:86-121: the vertexAffected
    bytes of every vertex reachable from a seed (device BFS)."""
    sd = _arr(seeds, np.uint32)
    va = np.zeros(max(g.vertex_count, 1), np.uint8)
    _check(N.lib().dynpr_mark_reachable(C.c_void_p(g.ctx.h), C.c_void_p(g.h), _p(sd), len(sd), _p(va)))
    return va[: g.vertex_count]


def dynamic_frontier_from_flags(g_forward: CsrGraph, g_transpose: CsrGraph, vertex_affected,
                                neighbors_pending, previous_ranks, config: Optional[EngineConfig] = None,
                                pruning: bool = False, observer: Optional[Callable] = None) -> RankResult:
    """dynamicFrontierFromFlags -- engine.cpp:178-190."""
    cfg = (config or EngineConfig())._c()
    va = _arr(vertex_affected, np.uint8)
    np_ = _arr(neighbors_pending, np.uint8)
    prev = _arr(previous_ranks, np.float64)
    ranks = np.empty(max(g_transpose.vertex_count, 1), np.float64)
    st = N.Stats()
    obs, keep = _observer(observer)
    _check(N.lib().dynpr_dynamic_frontier_from_flags(C.c_void_p(g_forward.ctx.h), C.c_void_p(g_forward.h),
                                                     C.c_void_p(g_transpose.h), _p(va), _p(np_), len(va),
                                                     _p(prev), len(prev), C.byref(cfg), int(bool(pruning)),
                                                     _p(ranks), C.byref(st), obs, None))
    return _result(ranks[: g_transpose.vertex_count], st)


from ._harness import (  # noqa: E402  (input formats + experiment harness)
    Approach, ChainMode, ExperimentMode, ExperimentRow, ExperimentSpec, ParseError, ReportFormat,
    approach_from_name, approach_name, compute_reference_ranks, emit_report, load_matrix_market,
    load_matrix_market_arrays, load_temporal_edge_list, load_temporal_edge_list_arrays, run_experiment,
    split_temporal, summarize_rows,
)
