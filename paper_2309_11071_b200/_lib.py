"""ctypes binding of the in-tree C ABI library (libstreamgnn.so).

The library is the product: every engine call goes to the sm_100a kernels
behind include/streamgnn.h. There is no Python or CPU fallback — if the shared
object is missing this module raises on import of the binding.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SGNN_B200_LIB selects another build of the same library (A/B measurements of build variants)
LIB_PATH = os.environ.get("SGNN_B200_LIB") or os.path.join(HERE, "libstreamgnn.so")

STATUS = {
    0: "SGNN_OK", 1: "SGNN_ERR_IO", 2: "SGNN_ERR_FORMAT", 3: "SGNN_ERR_DIMENSION", 4: "SGNN_ERR_DUPLICATE_EDGE",
    5: "SGNN_ERR_MISSING_EDGE", 6: "SGNN_ERR_UNSUPPORTED_MODEL", 7: "SGNN_ERR_INVALID_ARGUMENT",
    8: "SGNN_ERR_STALE_DELTA", 9: "SGNN_ERR_CONTRACT", 10: "SGNN_ERR_NAN_INPUT", 11: "SGNN_ERR_VERIFY_MISMATCH",
    12: "SGNN_ERR_UNKNOWN",
}

# Every symbol include/streamgnn.h and include/streamgnn_b200.h declare.
REFERENCE_SYMBOLS = [
    "sgnn_status_name", "sgnn_last_error", "sgnn_graph_create", "sgnn_graph_load", "sgnn_graph_destroy",
    "sgnn_graph_num_nodes", "sgnn_graph_num_edges", "sgnn_graph_add_edge", "sgnn_graph_out_neighbors",
    "sgnn_graph_in_neighbors", "sgnn_graph_save", "sgnn_model_load", "sgnn_model_destroy", "sgnn_model_num_layers",
    "sgnn_model_aggregator", "sgnn_engine_create", "sgnn_engine_open", "sgnn_engine_destroy",
    "sgnn_engine_save_checkpoints", "sgnn_engine_save_graph", "sgnn_engine_apply_update", "sgnn_engine_set_option",
    "sgnn_engine_stats_line", "sgnn_engine_embedding_dim", "sgnn_engine_read_embedding", "sgnn_engine_verify",
    "sgnn_stream_open", "sgnn_stream_next", "sgnn_stream_destroy", "sgnn_gen_synthetic", "sgnn_gen_model",
]
EXTENSION_SYMBOLS = [
    "sgnn_b200_device_available", "sgnn_b200_graph_from_edges", "sgnn_b200_engine_create_mem",
    "sgnn_b200_engine_apply_update_device", "sgnn_b200_engine_dirty_nodes", "sgnn_b200_engine_read_table",
    "sgnn_b200_engine_apply_update_device_async", "sgnn_b200_engine_read_rows",
    "sgnn_b200_engine_num_nodes", "sgnn_b200_engine_num_edges", "sgnn_b200_engine_kernel_times",
    "sgnn_b200_engine_flush_l2", "sgnn_b200_engine_stream", "sgnn_b200_engine_launches_per_round",
    "sgnn_b200_graph_load_binary", "sgnn_b200_graph_save_binary", "sgnn_b200_group_create", "sgnn_b200_engine_create_shm", "sgnn_b200_engine_memory",
    "sgnn_b200_shm_open", "sgnn_b200_shm_barrier", "sgnn_b200_shm_all_gather", "sgnn_b200_shm_allreduce",
    "sgnn_b200_shm_close", "sgnn_b200_group_apply_update", "sgnn_b200_engine_shard_range",
    "sgnn_b200_shard_bounds", "sgnn_b200_stats_report", "sgnn_b200_stats_canonical",
]


class GenConfig(C.Structure):
    _fields_ = [("num_nodes", C.c_uint32), ("avg_degree", C.c_double), ("feature_len", C.c_uint32),
                ("stream_len", C.c_uint32), ("seed", C.c_uint64), ("insert_fraction", C.c_double)]


_lib = None


def lib():
    """Loads and types the library once."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build()) first")
    L = C.CDLL(LIB_PATH)
    vp, pp = C.c_void_p, C.POINTER(C.c_void_p)
    u32p, sz = C.POINTER(C.c_uint32), C.POINTER(C.c_size_t)
    sig = {
        "sgnn_status_name": (C.c_char_p, [C.c_int]),
        "sgnn_last_error": (C.c_char_p, []),
        "sgnn_graph_create": (C.c_int, [C.c_uint32, pp]),
        "sgnn_graph_load": (C.c_int, [C.c_char_p, C.c_int, pp]),
        "sgnn_graph_destroy": (None, [vp]),
        "sgnn_graph_num_nodes": (C.c_uint32, [vp]),
        "sgnn_graph_num_edges": (C.c_uint64, [vp]),
        "sgnn_graph_add_edge": (C.c_int, [vp, C.c_uint32, C.c_uint32]),
        "sgnn_graph_out_neighbors": (C.c_int, [vp, C.c_uint32, vp, C.c_size_t, sz]),
        "sgnn_graph_in_neighbors": (C.c_int, [vp, C.c_uint32, vp, C.c_size_t, sz]),
        "sgnn_graph_save": (C.c_int, [vp, C.c_char_p]),
        "sgnn_model_load": (C.c_int, [C.c_char_p, C.c_char_p, pp]),
        "sgnn_model_destroy": (None, [vp]),
        "sgnn_model_num_layers": (C.c_int, [vp]),
        "sgnn_model_aggregator": (C.c_int, [vp]),
        "sgnn_engine_create": (C.c_int, [vp, vp, C.c_char_p, pp]),
        "sgnn_engine_open": (C.c_int, [vp, vp, C.c_char_p, C.c_char_p, pp]),
        "sgnn_engine_destroy": (None, [vp]),
        "sgnn_engine_save_checkpoints": (C.c_int, [vp, C.c_char_p]),
        "sgnn_engine_save_graph": (C.c_int, [vp, C.c_char_p]),
        "sgnn_engine_apply_update": (C.c_int, [vp, vp, vp, vp, C.c_size_t]),
        "sgnn_engine_set_option": (C.c_int, [vp, C.c_char_p, C.c_int64]),
        "sgnn_engine_stats_line": (C.c_int, [vp, C.c_char_p, C.c_size_t, sz]),
        "sgnn_engine_embedding_dim": (C.c_int, [vp, C.c_int, C.c_int, u32p]),
        "sgnn_engine_read_embedding": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint32, vp, C.c_size_t]),
        "sgnn_engine_verify": (C.c_int, [vp, u32p, u32p, u32p, u32p]),
        "sgnn_stream_open": (C.c_int, [C.c_char_p, pp]),
        "sgnn_stream_next": (C.c_int, [vp, C.c_char_p, u32p, u32p]),
        "sgnn_stream_destroy": (None, [vp]),
        "sgnn_gen_synthetic": (C.c_int, [C.POINTER(GenConfig), C.c_char_p]),
        "sgnn_gen_model": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_double,
                                     C.c_char_p]),
        "sgnn_b200_device_available": (C.c_int, [C.c_char_p, C.c_size_t]),
        "sgnn_b200_graph_from_edges": (C.c_int, [C.c_uint32, vp, vp, C.c_uint64, C.c_int, pp]),
        "sgnn_b200_engine_create_mem": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_uint32, pp]),
        "sgnn_b200_engine_apply_update_device": (C.c_int, [vp, vp, vp, vp, C.c_size_t]),
        "sgnn_b200_engine_dirty_nodes": (C.c_int, [vp, C.c_int, vp, C.c_size_t, sz]),
        "sgnn_b200_engine_read_table": (C.c_int, [vp, C.c_int, C.c_int, vp, C.c_size_t]),
        "sgnn_b200_engine_apply_update_device_async": (C.c_int, [vp, vp, vp, vp, C.c_size_t, vp]),
        "sgnn_b200_engine_read_rows": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint32, C.c_uint32, vp, C.c_size_t]),
        "sgnn_b200_engine_num_nodes": (C.c_uint32, [vp]),
        "sgnn_b200_engine_num_edges": (C.c_uint64, [vp]),
        "sgnn_b200_engine_kernel_times": (C.c_size_t, [vp, vp, C.c_size_t]),
        "sgnn_b200_engine_flush_l2": (C.c_int, [vp]),
        "sgnn_b200_engine_launches_per_round": (C.c_size_t, [vp]),
        "sgnn_b200_engine_stream": (C.c_void_p, [vp]),
        "sgnn_b200_graph_load_binary": (C.c_int, [C.c_char_p, C.c_int, pp]),
        "sgnn_b200_graph_save_binary": (C.c_int, [vp, C.c_char_p]),
        "sgnn_b200_group_create": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_uint32, C.c_int, pp]),
        "sgnn_b200_engine_create_shm": (C.c_int, [C.c_char_p, C.c_int, C.c_int, vp, vp, vp, C.c_uint32, C.c_uint32,
                                                  pp]),
        "sgnn_b200_engine_memory": (C.c_int, [vp, vp]),
        "sgnn_b200_shm_open": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_double, pp]),
        "sgnn_b200_shm_barrier": (C.c_int, [vp]),
        "sgnn_b200_shm_all_gather": (C.c_int, [vp, C.c_uint64, vp]),
        "sgnn_b200_shm_allreduce": (C.c_int, [vp, vp, C.c_size_t]),
        "sgnn_b200_shm_close": (None, [vp]),
        "sgnn_b200_group_apply_update": (C.c_int, [pp, C.c_int, vp, vp, vp, C.c_size_t]),
        "sgnn_b200_engine_shard_range": (C.c_int, [vp, u32p, u32p]),
        "sgnn_b200_shard_bounds": (C.c_int, [vp, C.c_uint32, C.c_int, vp]),
        "sgnn_b200_stats_report": (C.c_int, [vp, C.c_size_t, C.c_char_p, C.c_size_t, sz]),
        "sgnn_b200_stats_canonical": (C.c_int, [C.c_char_p, C.c_char_p, C.c_size_t, sz]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
