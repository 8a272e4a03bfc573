"""ctypes binding of libdynpr_cuda.so (the C-ABI in include/dynpr_cuda.h).

There is no CPU fallback: if the shared library is missing, or no CUDA device
is visible, every call that needs it raises.  The binding only declares
prototypes; all compute runs in the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdynpr_cuda.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "dynpr_cuda.h")

DYNPR_OK = 0
DYNPR_INVALID_ARGUMENT = 1
DYNPR_CUDA_ERROR = 2
DYNPR_NCCL_ERROR = 3
DYNPR_OUT_OF_MEMORY = 4
DYNPR_SIZING_ERROR = 5
DYNPR_PARSE_ERROR = 6
DYNPR_RUNTIME_ERROR = 7


class Config(C.Structure):
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


class Stats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("affected_vertex_iterations", C.c_uint64),
        ("final_delta", C.c_double),
        ("processed_edges", C.c_uint64),
        ("device_ms", C.c_double),
    ]


class ExperimentSpec(C.Structure):  # dynpr_experiment_spec
    _fields_ = [
        ("graph_path", C.c_char_p),
        ("graph_name", C.c_char_p),
        ("mode", C.c_int32),
        ("batch_size_specs", C.POINTER(C.c_char_p)),
        ("n_batch_size_specs", C.c_int32),
        ("approaches", C.POINTER(C.c_int32)),
        ("n_approaches", C.c_int32),
        ("seed", C.c_uint64),
        ("repetitions", C.c_int32),
        ("base_fraction", C.c_double),
        ("batch_count", C.c_int32),
        ("insert_fraction", C.c_double),
        ("chain_mode", C.c_int32),
        ("threads", C.c_int32),
        ("record_timing", C.c_int32),
        ("config", Config),
    ]


class ExperimentRow(C.Structure):  # dynpr_experiment_row
    _fields_ = [
        ("graph_name", C.c_char_p),
        ("approach", C.c_char_p),
        ("batch_size_spec", C.c_char_p),
        ("batch_index", C.c_int64),
        ("runtime_millis", C.c_double),
        ("iterations", C.c_int64),
        ("affected_vertex_iterations", C.c_uint64),
        ("l1_error_vs_reference", C.c_double),
        ("converged", C.c_int32),
    ]


OBSERVER = C.CFUNCTYPE(None, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                       C.c_uint64, C.c_void_p)

# dynpr_comm_ops (caller-supplied host transport)
ALLREDUCE_U64 = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_uint64), C.c_uint64, C.c_int, C.c_void_p)
ALLGATHERV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.c_void_p)
BARRIER = C.CFUNCTYPE(C.c_int, C.c_void_p)


class CommOps(C.Structure):
    _fields_ = [("allreduce_u64", ALLREDUCE_U64), ("allgatherv", ALLGATHERV), ("barrier", BARRIER)]


_vp = C.c_void_p
_pvp = C.POINTER(C.c_void_p)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_cfgp = C.POINTER(Config)
_stp = C.POINTER(Stats)
_i = C.c_int
_u32 = C.c_uint32
_u64 = C.c_uint64
_d = C.c_double

# name -> (restype, argtypes); mirrors include/dynpr_cuda.h
PROTOTYPES = {
    "dynpr_last_error": (C.c_char_p, []),
    "dynpr_version": (C.c_char_p, []),
    "dynpr_config_default": (None, [_cfgp]),
    "dynpr_config_validate": (_i, [_cfgp]),
    "dynpr_context_create": (_i, [_i, _pvp]),
    "dynpr_context_destroy": (_i, [_vp]),
    "dynpr_context_launches": (_u64, [_vp]),
    "dynpr_context_set_profiling": (_i, [_vp, _i]),
    "dynpr_context_sweep_times": (_i, [_vp, _dp, _u64p, _u64p]),
    "dynpr_nccl_get_unique_id": (_i, [_vp]),
    "dynpr_context_create_nccl": (_i, [_i, _i, _i, _vp, _pvp]),
    "dynpr_team_create": (_i, [_i, _pvp]),
    "dynpr_team_destroy": (_i, [_vp]),
    "dynpr_context_create_team": (_i, [_i, _vp, _i, _pvp]),
    "dynpr_context_rank": (_i, [_vp, _ip, _ip]),
    "dynpr_context_attach_peers": (_i, [_vp, _i, _vp, _vp, _u64]),
    "dynpr_context_create_hostcomm": (_i, [_i, _i, _i, C.POINTER(CommOps), _vp, _pvp]),
    "dynpr_graph_layout_info": (_i, [_vp, _u64p, _u32p, _u32p, _ip, _ip]),
    "dynpr_ipc_alloc": (_i, [_vp, _u64, _pvp, _vp]),
    "dynpr_ipc_open": (_i, [_vp, _vp, _pvp]),
    "dynpr_ipc_close": (_i, [_vp, _vp]),
    "dynpr_ipc_free": (_i, [_vp, _vp]),
    "dynpr_graph_from_csr": (_i, [_vp, _u32, _vp, _vp, _u64, _pvp]),
    "dynpr_graph_build": (_i, [_vp, _u32, _vp, _vp, _u64, _pvp]),
    "dynpr_graph_add_self_loops": (_i, [_vp, _vp, _pvp]),
    "dynpr_graph_transpose": (_i, [_vp, _vp, _pvp]),
    "dynpr_graph_apply_batch": (_i, [_vp, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _pvp, _u64p, _u64p]),
    "dynpr_graph_apply_batch_pair": (_i, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _pvp, _pvp,
                                          _u64p, _u64p]),
    "dynpr_graph_info": (_i, [_vp, _u32p, _u64p]),
    "dynpr_graph_download": (_i, [_vp, _vp, _vp, _vp]),
    "dynpr_graph_has_edge": (_i, [_vp, _vp, _u32, _u32, _ip]),
    "dynpr_graph_destroy": (_i, [_vp]),
    "dynpr_graph_rmat": (_i, [_vp, _u32, _u32, _d, _d, _d, _u64, _pvp]),
    "dynpr_graph_kronecker": (_i, [_vp, _u32, _u32, _u64, _pvp]),
    "dynpr_graph_prepare": (_i, [_vp, _vp, _vp, _u32, _i, _dp]),
    "dynpr_batch_size_from_fraction": (_u64, [_d, _u64]),
    "dynpr_derive_seed": (_u64, [_u64, _u64]),
    "dynpr_generate_random_batch": (_i, [_vp, _vp, _u64, _d, _u64, _vp, _vp, _u64p, _vp, _vp, _u64p]),
    "dynpr_partition_by_degree": (_i, [_vp, _vp, _u32, _vp, _u32p]),
    "dynpr_update_ranks": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _cfgp, _i]),
    "dynpr_linf_norm_delta": (_i, [_vp, _vp, _vp, _u64, _dp]),
    "dynpr_l1_norm_delta": (_i, [_vp, _vp, _vp, _u64, _dp]),
    "dynpr_initial_affected": (_i, [_vp, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp]),
    "dynpr_expand_affected": (_i, [_vp, _vp, _vp, _vp, _u32]),
    "dynpr_static_pagerank": (_i, [_vp, _vp, _vp, _cfgp, _vp, _stp, OBSERVER, _vp]),
    "dynpr_static_pagerank_csr": (_i, [_vp, _u32, _vp, _vp, _vp, _vp, _u64, _cfgp, _vp, _stp, OBSERVER, _vp]),
    "dynpr_naive_dynamic": (_i, [_vp, _vp, _vp, _vp, _u64, _cfgp, _vp, _stp, OBSERVER, _vp]),
    "dynpr_dynamic_frontier": (_i, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _u64, _cfgp, _i,
                                    _vp, _stp, OBSERVER, _vp]),
    "dynpr_dynamic_traversal": (_i, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _u64, _cfgp, _vp, _stp,
                                     OBSERVER, _vp]),
    "dynpr_mark_reachable": (_i, [_vp, _vp, _vp, _u64, _vp]),
    "dynpr_dynamic_frontier_from_flags": (_i, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _u64, _cfgp, _i, _vp,
                                               _stp, OBSERVER, _vp]),
    "dynpr_load_matrix_market": (_i, [C.c_char_p, _pvp]),
    "dynpr_load_temporal_edge_list": (_i, [C.c_char_p, _pvp]),
    "dynpr_split_temporal": (_i, [_vp, _d, C.c_int32, _u64, _pvp, _u64p]),
    "dynpr_edge_list_info": (_i, [_vp, _u32p, _u64p, _ip]),
    "dynpr_edge_list_copy": (_i, [_vp, _u64, _u64, _vp, _vp, _vp]),
    "dynpr_edge_list_destroy": (_i, [_vp]),
    "dynpr_edge_list_create": (_i, [_u32, _vp, _vp, _vp, _u64, _vp]),
    "dynpr_compute_reference_ranks": (_i, [_vp, _vp, _vp, _cfgp, _vp]),
    "dynpr_experiment_spec_default": (None, [C.POINTER(ExperimentSpec)]),
    "dynpr_run_experiment": (_i, [_vp, C.POINTER(ExperimentSpec), _pvp]),
    "dynpr_report_create": (_i, [_pvp]),
    "dynpr_report_append": (_i, [_vp, C.POINTER(ExperimentRow)]),
    "dynpr_report_size": (_i, [_vp, _u64p]),
    "dynpr_report_row": (_i, [_vp, _u64, C.POINTER(ExperimentRow)]),
    "dynpr_report_summarize": (_i, [_vp, _pvp]),
    "dynpr_report_emit": (_i, [_vp, C.c_int32, C.c_char_p]),
    "dynpr_report_destroy": (_i, [_vp]),
    "dynpr_debug_sweep_trace": (_i, [_vp, _u64, _u64p]),
    "dynpr_debug_loop_trace": (_i, [_vp, _u64, _u64p]),
    "dynpr_debug_prims": (_i, [_vp, C.c_int, _vp, _vp, _u64, C.c_int, _vp, _vp, _u64p]),
}

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    pass


def header_symbols():
    """Function names declared in include/dynpr_cuda.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(dynpr_[a-z0-9_]+)\s*\(", text)) - {"dynpr_observer"})


def lib():
    """The loaded library (raises NativeUnavailable when it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def last_error() -> str:
    return lib().dynpr_last_error().decode()
