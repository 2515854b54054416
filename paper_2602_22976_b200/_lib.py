"""ctypes binding of include/hlm_b200.h (libhlm_b200.so).  No compute happens in Python."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HLM_B200_LIB") or os.path.join(_HERE, "lib", "libhlm_b200.so")

OK, ERR_INPUT, ERR_ROUND_LIMIT, ERR_CUDA, ERR_NOMEM, ERR_UNSUPPORTED, ERR_NCCL = range(7)
UNIQUE_ID_BYTES = 128


class CsrView(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("num_edges", C.c_uint32),
                ("vertex_offsets", C.c_void_p), ("vertex_incidence", C.c_void_p),
                ("edge_offsets", C.c_void_p), ("edge_members", C.c_void_p),
                ("base_weights", C.c_void_p)]


class Stream(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("kind", C.c_int32), ("mode", C.c_int32),
                ("noise_low", C.c_double), ("noise_high", C.c_double)]


class Config(C.Structure):
    _fields_ = [("variant", C.c_int32), ("max_rounds", C.c_uint32), ("loop_mode", C.c_int32),
                ("tie_mode", C.c_int32), ("flags", C.c_uint32), ("num_gpus", C.c_uint32)]


class Result(C.Structure):
    _fields_ = [("matched_edges", C.POINTER(C.c_uint32)), ("matched_round", C.POINTER(C.c_uint16)),
                ("num_matched", C.c_uint64), ("total_weight", C.c_double), ("rounds", C.c_uint32),
                ("per_round_matched", C.POINTER(C.c_uint32)),
                ("per_round_deactivated", C.POINTER(C.c_uint32)),
                ("total_edge_visits", C.c_uint64), ("total_pin_visits", C.c_uint64),
                ("device_edge_visits", C.c_uint64), ("device_pin_visits", C.c_uint64),
                ("wall_time_ms", C.c_double), ("device_ms", C.c_double),
                ("tie_redo_rounds", C.c_uint32), ("kernel_launches", C.c_uint32),
                ("graph_launches", C.c_uint32), ("write_conflicts", C.c_uint32),
                ("round_filter_ms", C.POINTER(C.c_float)), ("round_check_ms", C.POINTER(C.c_float)),
                ("h2d_bytes", C.c_uint64), ("prefix_sum_invocations", C.c_uint32), ("compactions", C.c_uint32),
                ("engine", C.c_uint32), ("engine_switch_round", C.c_uint32)]


class GraphInfo(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("num_edges", C.c_uint32), ("num_pins", C.c_uint64),
                ("uniform_size", C.c_uint32), ("max_edge_size", C.c_uint32),
                ("num_large_edges", C.c_uint32), ("unit_weights", C.c_int32), ("device", C.c_int32),
                ("device_bytes", C.c_uint64)]


class SynSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("n", C.c_uint32), ("m", C.c_uint32), ("d", C.c_uint32),
                ("scale", C.c_uint32), ("seed", C.c_uint64), ("int_weights", C.c_int32),
                ("edge_begin", C.c_uint32), ("m_local", C.c_uint32)]


class ShardReport(C.Structure):
    _fields_ = [("rounds", C.c_uint32), ("num_local_shards", C.c_uint32), ("num_processes", C.c_uint32),
                ("tie_redo_rounds", C.c_uint32), ("host_syncs", C.c_uint32), ("kernel_launches", C.c_uint32),
                ("nccl_calls", C.c_uint32), ("num_edges_global", C.c_uint64), ("collective_bytes", C.c_uint64),
                ("collective_bytes_per_round", C.POINTER(C.c_uint64)),
                ("live_vertices_per_round", C.POINTER(C.c_uint32))]


class HostGraph(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("num_edges", C.c_uint32),
                ("vertex_offsets", C.POINTER(C.c_uint64)), ("vertex_incidence", C.POINTER(C.c_uint32)),
                ("edge_offsets", C.POINTER(C.c_uint64)), ("edge_members", C.POINTER(C.c_uint32)),
                ("base_weights", C.POINTER(C.c_double)), ("num_warnings", C.c_uint32)]


class CompactWork(C.Structure):
    _fields_ = [("total_edge_visits", C.c_uint64), ("total_pin_visits", C.c_uint64),
                ("prefix_sum_invocations", C.c_uint32), ("compactions", C.c_uint32)]


# every symbol include/hlm_b200.h declares: (restype, argtypes)
SYMBOLS = {
    "hlm_b200_abi_version": (C.c_int, []),
    "hlm_b200_last_error": (C.c_char_p, []),
    "hlm_b200_device_count": (C.c_int, []),
    "hlm_b200_graph_upload": (C.c_int, [C.POINTER(CsrView), C.c_int, C.POINTER(C.c_void_p)]),
    "hlm_b200_graph_upload_shard": (C.c_int, [C.POINTER(CsrView), C.c_uint32, C.c_int, C.POINTER(C.c_void_p)]),
    "hlm_b200_graph_generate": (C.c_int, [C.POINTER(SynSpec), C.c_int, C.POINTER(C.c_void_p)]),
    "hlm_b200_graph_info_get": (C.c_int, [C.c_void_p, C.POINTER(GraphInfo)]),
    "hlm_b200_graph_download": (C.c_int, [C.c_void_p] * 6),
    "hlm_b200_graph_release": (None, [C.c_void_p]),
    "hlm_b200_graph_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hlm_b200_match": (C.c_int, [C.c_void_p, C.POINTER(Stream), C.POINTER(Config), C.POINTER(Result)]),
    "hlm_b200_match_host": (C.c_int, [C.POINTER(CsrView), C.POINTER(Stream), C.POINTER(Config), C.c_int,
                                      C.POINTER(Result)]),
    "hlm_b200_result_free": (None, [C.POINTER(Result)]),
    "hlm_b200_verify": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_double)]),
    "hlm_b200_eval_stream": (C.c_int, [C.POINTER(Stream), C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                       C.c_void_p, C.c_void_p, C.c_int]),
    "hlm_b200_default_max_rounds": (C.c_uint32, [C.c_uint32]),
    "hlm_b200_comm_unique_id": (C.c_int, [C.c_void_p]),
    "hlm_b200_comm_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "hlm_b200_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]),
    "hlm_b200_comm_destroy": (None, [C.c_void_p]),
    "hlm_b200_match_sharded": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.POINTER(Stream),
                                         C.POINTER(Config), C.POINTER(Result), C.POINTER(ShardReport)]),
    "hlm_b200_shard_report_free": (None, [C.POINTER(ShardReport)]),
    "hlm_b200_parse_hgr": (C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(HostGraph)]),
    "hlm_b200_parse_metis_graph": (C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(HostGraph)]),
    "hlm_b200_generate_random": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                           C.POINTER(HostGraph)]),
    "hlm_b200_generate_tight_family": (C.c_int, [C.c_uint32, C.c_double, C.POINTER(HostGraph)]),
    "hlm_b200_random_weights_1_100": (C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p]),
    "hlm_b200_host_graph_free": (None, [C.POINTER(HostGraph)]),
    "hlm_b200_write_hgr": (C.c_int, [C.POINTER(CsrView), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "hlm_b200_write_matching": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double, C.c_uint32, C.POINTER(C.c_void_p),
                                          C.POINTER(C.c_size_t)]),
    "hlm_b200_parse_matching": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
    "hlm_b200_text_free": (None, [C.c_void_p]),
    "hlm_b200_compact": (C.c_int, [C.POINTER(CsrView), C.c_void_p, C.c_void_p, C.c_int, C.POINTER(HostGraph),
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(CompactWork)]),
}

_lib = None


def load_library():
    """Loads libhlm_b200.so (built in-tree by __graft_entry__.build()).  Fails loudly if it is
    missing: there is no Python or CPU fallback for the matching path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python __graft_entry__.py` (nvcc, sm_100a) first; "
            "paper_2602_22976_b200 has no fallback path")
    lib = C.CDLL(LIB_PATH)
    for name, (restype, argtypes) in SYMBOLS.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def last_error() -> str:
    return (load_library().hlm_b200_last_error() or b"").decode()
