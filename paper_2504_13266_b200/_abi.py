"""ctypes mirror of include/pp_loader.h (struct layouts, enums, prototypes)."""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libppload.so")

PP_OK, PP_ERR_INVALID, PP_ERR_OOM, PP_ERR_CUDA, PP_ERR_NCCL, PP_ERR_STATE, PP_END_OF_EPOCH = range(7)
PP_F32, PP_BF16, PP_F16 = 0, 1, 2
PP_MEM_HOST, PP_MEM_DEVICE, PP_MEM_FILES = 0, 1, 2
PP_PEERS_NONE, PP_PEERS_IPC, PP_PEERS_LOOPBACK, PP_PEERS_NCCL = 0, 1, 2, 3
IPC_HANDLE_BYTES = 256  # PP_IPC_HANDLE_BYTES
NCCL_ID_BYTES = 128  # PP_NCCL_ID_BYTES

# every symbol include/pp_loader.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "pp_loader_create", "pp_loader_destroy", "pp_epoch_permute", "pp_epoch_prefetch", "pp_next_batch", "pp_next_batches", "pp_seek",
    "pp_set_stream", "pp_loader_query", "pp_last_error", "pp_abi_version", "pp_footprint_bytes",
    "pp_export_store", "pp_import_peer_stores", "pp_link_loopback", "pp_fill_synthetic", "pp_get_order",
    "pp_read_store", "pp_debug_set_sort_bits_delta", "pp_next_batches_linear", "pp_propagate",
    "pp_epoch_permute_local", "pp_propagate_store", "pp_next_batches_ev",
    "pp_set_grid_limit", "pp_nccl_unique_id",
]


class PPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class pp_hop_desc(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("where", ctypes.c_int),
        ("num_nodes", ctypes.c_int64),
        ("num_hops", ctypes.c_int32),
        ("feat_dim", ctypes.c_int32),
        ("hop_stride", ctypes.c_int64),
        ("row_stride", ctypes.c_int64),
        ("dtype", ctypes.c_int),
    ]


class pp_loader_desc(ctypes.Structure):
    _fields_ = [
        ("hops", pp_hop_desc),
        ("node_set", ctypes.POINTER(ctypes.c_int64)),
        ("num_set", ctypes.c_int64),
        ("labels", ctypes.POINTER(ctypes.c_int32)),
        ("batch_size", ctypes.c_int32),
        ("out_dtype", ctypes.c_int),
        ("drop_last", ctypes.c_int32),
        ("hbm_budget_bytes", ctypes.c_int64),
        ("world_size", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("peers", ctypes.c_int),
        ("device", ctypes.c_int32),
        ("store_set_only", ctypes.c_int32),
        ("borrow_device_data", ctypes.c_int32),
        ("nccl_unique_id", ctypes.c_void_p),
    ]


class pp_loader_info(ctypes.Structure):
    _fields_ = [
        ("num_positions", ctypes.c_int64),
        ("num_nodes_total", ctypes.c_int64),
        ("local_rows", ctypes.c_int64),
        ("rows_hbm", ctypes.c_int64),
        ("rows_spill", ctypes.c_int64),
        ("record_bytes_in", ctypes.c_int64),
        ("record_stride", ctypes.c_int64),
        ("record_bytes_out", ctypes.c_int64),
        ("steps_per_epoch", ctypes.c_int64),
        ("cursor", ctypes.c_int64),
        ("permuted", ctypes.c_int32),
        ("gather_path", ctypes.c_int32),
        ("local_epoch", ctypes.c_int32),
        ("epoch_positions", ctypes.c_int64),
        ("exchange_cast", ctypes.c_int32),
        ("storage_mode", ctypes.c_int32),
        ("storage_bytes_read", ctypes.c_int64),
        ("pdl_launches", ctypes.c_int64),
        ("all_to_all", ctypes.c_int32),
        ("spill_shared", ctypes.c_int32),
        ("hbm_store_bytes", ctypes.c_int64),
        ("hbm_exchange_bytes", ctypes.c_int64),
        ("hbm_scratch_bytes", ctypes.c_int64),
        ("host_spill_bytes", ctypes.c_int64),
    ]


_lock = threading.Lock()
_lib = None


def lib():
    """Load libppload.so.  Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:  # fast path: no lock once loaded
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            P, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
            st = ctypes.c_int
            sig = {
                "pp_loader_create": (st, [P, P]),
                "pp_loader_destroy": (st, [P]),
                "pp_epoch_permute": (st, [P, u64, i64, P]),
                "pp_epoch_prefetch": (st, [P, u64, i64]),
                "pp_next_batch": (st, [P, P, P, P, P, P]),
                "pp_next_batches": (st, [P, i32, P, i64, P, P, P, P, P]),
                "pp_seek": (st, [P, i64]),
                "pp_set_stream": (st, [P, P]),
                "pp_loader_query": (st, [P, P]),
                "pp_last_error": (ctypes.c_char_p, []),
                "pp_abi_version": (i32, []),
                "pp_footprint_bytes": (i64, [i64, i32, i32, i32, i32]),
                "pp_export_store": (st, [P, P]),
                "pp_import_peer_stores": (st, [P, P]),
                "pp_link_loopback": (st, [P, i32]),
                "pp_fill_synthetic": (st, [P, u64]),
                "pp_get_order": (st, [P, P]),
                "pp_read_store": (st, [P, i64, i64, P]),
                "pp_debug_set_sort_bits_delta": (st, [P, i32]),
                "pp_next_batches_linear": (st, [P, i32, P, i32, P, ctypes.c_int, i64, P, P, P]),
                "pp_propagate": (st, [i64, i32, P, P, P, i32, P, P]),
                "pp_epoch_permute_local": (st, [P, u64, i64, P]),
                "pp_propagate_store": (st, [P, i32, P, P, P, P]),
                "pp_next_batches_ev": (st, [P, i32, P, i64, P, P, P, P, P, P]),
                "pp_set_grid_limit": (st, [P, i32]),
                "pp_nccl_unique_id": (st, [P]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib
