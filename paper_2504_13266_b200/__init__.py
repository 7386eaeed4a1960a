"""B200-native PP-GNN mini-batch loader (arXiv 2504.13266), Python binding.

Argument marshalling over ``libppload.so`` (include/pp_loader.h) with the
same entry-point names; every step of the loading path runs in the library's
sm_100a kernels.  There is no CPU fallback: importing the binding without the
built library raises.

PyTorch is used only for device memory and streams (callers pass tensors /
``torch.cuda.Stream`` objects; we pass their raw pointers through).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._abi import (  # noqa: F401
    PP_OK, PP_ERR_INVALID, PP_ERR_OOM, PP_ERR_CUDA, PP_ERR_NCCL, PP_ERR_STATE, PP_END_OF_EPOCH,
    PP_F32, PP_BF16, PP_F16, PP_MEM_HOST, PP_MEM_DEVICE, PP_MEM_FILES, PP_PEERS_NONE, PP_PEERS_IPC, PP_PEERS_LOOPBACK,
    PP_PEERS_NCCL, IPC_HANDLE_BYTES, NCCL_ID_BYTES,
    pp_hop_desc, pp_loader_desc, pp_loader_info, PPError, lib, LIB_PATH,
)

__all__ = [
    "Loader", "PPError", "lib", "LIB_PATH",
    "pp_loader_create", "pp_loader_destroy", "pp_epoch_permute", "pp_epoch_prefetch", "pp_next_batch", "pp_next_batches",
    "pp_seek", "pp_set_stream", "pp_loader_query", "pp_last_error", "pp_abi_version", "pp_footprint_bytes",
    "pp_fill_synthetic", "pp_get_order", "pp_read_store", "pp_link_loopback", "pp_export_store",
    "pp_import_peer_stores", "pp_debug_set_sort_bits_delta", "pp_next_batches_linear", "pp_propagate",
    "pp_epoch_permute_local", "pp_propagate_store", "pp_next_batches_ev",
    "pp_set_grid_limit", "pp_nccl_unique_id",
]


def _check(rc: int, what: str, ok=(PP_OK,)) -> int:
    if rc not in ok:
        raise PPError(rc, f"{what}: {lib().pp_last_error().decode()}")
    return rc


def _ptr(x) -> int | None:
    """Raw address of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


_DT = {"f32": PP_F32, "float32": PP_F32, "bf16": PP_BF16, "bfloat16": PP_BF16, "f16": PP_F16, "float16": PP_F16}


def _dtype(d) -> int:
    if isinstance(d, int):
        return d
    return _DT[str(d).replace("torch.", "")]


# --------------------------------------------------------------------------- same-name entry points
def pp_abi_version() -> int:
    return lib().pp_abi_version()


def pp_last_error() -> str:
    return lib().pp_last_error().decode()


def pp_footprint_bytes(num_nodes, feat_dim, elem_bytes, num_ops, num_hops_R) -> int:
    return lib().pp_footprint_bytes(num_nodes, feat_dim, elem_bytes, num_ops, num_hops_R)


def pp_loader_create(*, data=None, where=PP_MEM_HOST, num_nodes, num_hops, feat_dim, hop_stride=0, row_stride=0,
                     dtype=PP_F32, node_set=None, labels=None, batch_size, out_dtype=PP_BF16, drop_last=False,
                     hbm_budget_bytes=0, world_size=1, rank=0, peers=PP_PEERS_NONE, device=0, files=None,
                     store_set_only=False, borrow_device_data=False, nccl_unique_id=None):
    """pp_loader_create(desc) -> handle.  ``data`` is a numpy array (host) or a torch CUDA tensor
    (device) of the hop matrices with the given element strides; None allocates the store only.
    ``files``: H hop file paths (raw [N][F] of dtype each) -> the storage tier (PP_MEM_FILES)."""
    d = pp_loader_desc()
    keep = []
    if files is not None:
        paths = (ctypes.c_char_p * len(files))(*[os.fsencode(f) for f in files])
        keep.append(paths)
        d.hops.data = ctypes.cast(paths, ctypes.c_void_p).value
        where = PP_MEM_FILES
    elif data is not None:
        if isinstance(data, np.ndarray):
            data = np.ascontiguousarray(data)
            keep.append(data)
            where = PP_MEM_HOST
        else:
            where = PP_MEM_DEVICE if data.is_cuda else PP_MEM_HOST
        d.hops.data = _ptr(data)
    d.hops.where = where
    d.hops.num_nodes = num_nodes
    d.hops.num_hops = num_hops
    d.hops.feat_dim = feat_dim
    d.hops.hop_stride = hop_stride
    d.hops.row_stride = row_stride
    d.hops.dtype = _dtype(dtype)
    if node_set is not None:
        ns = np.ascontiguousarray(node_set, dtype=np.int64)
        keep.append(ns)
        d.node_set = ctypes.cast(ns.ctypes.data, ctypes.POINTER(ctypes.c_int64))
        d.num_set = ns.shape[0]
    if labels is not None:
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        keep.append(lab)
        d.labels = ctypes.cast(lab.ctypes.data, ctypes.POINTER(ctypes.c_int32))
    d.batch_size = batch_size
    d.out_dtype = _dtype(out_dtype)
    d.drop_last = int(drop_last)
    d.hbm_budget_bytes = hbm_budget_bytes
    d.world_size = world_size
    d.rank = rank
    d.peers = peers
    d.device = device
    d.store_set_only = int(store_set_only)
    d.borrow_device_data = int(borrow_device_data)
    if nccl_unique_id is not None:
        uid = ctypes.create_string_buffer(bytes(nccl_unique_id), NCCL_ID_BYTES)
        keep.append(uid)
        d.nccl_unique_id = ctypes.cast(uid, ctypes.c_void_p).value
    h = ctypes.c_void_p()
    _check(lib().pp_loader_create(ctypes.byref(d), ctypes.byref(h)), "pp_loader_create")
    return h


def pp_loader_destroy(h) -> None:
    _check(lib().pp_loader_destroy(h), "pp_loader_destroy")


def pp_epoch_permute(h, seed: int, chunk: int = 1, stream=None) -> None:
    _check(lib().pp_epoch_permute(h, ctypes.c_uint64(seed & (2**64 - 1)), chunk, _stream(stream)), "pp_epoch_permute")


def pp_epoch_permute_local(h, seed: int, chunk: int = 1, stream=None) -> None:
    _check(lib().pp_epoch_permute_local(h, ctypes.c_uint64(seed & (2**64 - 1)), chunk, _stream(stream)),
           "pp_epoch_permute_local")


def pp_epoch_prefetch(h, seed: int, chunk: int = 1) -> None:
    _check(lib().pp_epoch_prefetch(h, ctypes.c_uint64(seed & (2**64 - 1)), chunk), "pp_epoch_prefetch")


def pp_next_batch(h, out, out_labels=None, out_nodes=None, consumer_stream=None) -> int:
    """Returns the rows written, or -1 at the end of the epoch (PP_END_OF_EPOCH)."""
    rows = ctypes.c_int32()
    rc = lib().pp_next_batch(h, _ptr(out), _ptr(out_labels), _ptr(out_nodes), ctypes.byref(rows),
                             _stream(consumer_stream))
    _check(rc, "pp_next_batch", ok=(PP_OK, PP_END_OF_EPOCH))
    return -1 if rc == PP_END_OF_EPOCH else rows.value


def pp_next_batches(h, n, out, out_stride_bytes, out_labels=None, out_nodes=None, consumer_stream=None):
    """Returns the list of rows per assembled step ([] at the end of the epoch)."""
    rows = (ctypes.c_int32 * n)()
    done = ctypes.c_int32()
    rc = lib().pp_next_batches(h, n, _ptr(out), out_stride_bytes, _ptr(out_labels), _ptr(out_nodes), rows,
                               ctypes.byref(done), _stream(consumer_stream))
    _check(rc, "pp_next_batches", ok=(PP_OK, PP_END_OF_EPOCH))
    return [] if rc == PP_END_OF_EPOCH else list(rows[: done.value])


def _event(e):
    if e is None:
        return None
    if isinstance(e, int):
        return e
    return e.cuda_event  # torch.cuda.Event


def pp_next_batches_ev(h, n, out, out_stride_bytes, out_labels=None, out_nodes=None, wait_event=None,
                       ready_event=None):
    """Event-ordered pp_next_batches (double buffer): waits for ``wait_event`` before writing,
    records ``ready_event`` when the slots are written (torch.cuda.Event or raw cudaEvent_t).
    Returns the list of rows per assembled step ([] at the end of the epoch)."""
    rows = (ctypes.c_int32 * n)()
    done = ctypes.c_int32()
    rc = lib().pp_next_batches_ev(h, n, _ptr(out), out_stride_bytes, _ptr(out_labels), _ptr(out_nodes), rows,
                                  ctypes.byref(done), _event(wait_event), _event(ready_event))
    _check(rc, "pp_next_batches_ev", ok=(PP_OK, PP_END_OF_EPOCH))
    return [] if rc == PP_END_OF_EPOCH else list(rows[: done.value])


def pp_next_batches_linear(h, n, W, D, Z, z_dtype, z_stride_bytes, consumer_stream=None):
    """Fused batch assembly + per-hop linear (tensor cores).  Returns rows per step ([] at epoch end)."""
    rows = (ctypes.c_int32 * n)()
    done = ctypes.c_int32()
    rc = lib().pp_next_batches_linear(h, n, _ptr(W), D, _ptr(Z), _dtype(z_dtype), z_stride_bytes, rows,
                                      ctypes.byref(done), _stream(consumer_stream))
    _check(rc, "pp_next_batches_linear", ok=(PP_OK, PP_END_OF_EPOCH))
    return [] if rc == PP_END_OF_EPOCH else list(rows[: done.value])


def pp_propagate(row_ptr, col_idx, X, K, hops, stream=None) -> None:
    """Eq. (2) on the GPU: hops[k] = B hops[k-1], hops[0] = X (device tensors: int64 CSR of I + A,
    fp32 X [n, F], fp32 hops [K+1, n, F])."""
    n, F = X.shape
    _check(lib().pp_propagate(n, F, _ptr(row_ptr), _ptr(col_idx), _ptr(X), K, _ptr(hops), _stream(stream)),
           "pp_propagate")


def pp_propagate_store(h, k: int, row_ptr, col_idx, deg, stream=None) -> None:
    """Hop slot k of this rank's store records = B (slot k-1 of every owner's records): device int64
    local CSR (global columns), device int32 global degrees d~."""
    _check(lib().pp_propagate_store(h, k, _ptr(row_ptr), _ptr(col_idx), _ptr(deg), _stream(stream)),
           "pp_propagate_store")


def pp_set_grid_limit(h, max_ctas: int) -> None:
    _check(lib().pp_set_grid_limit(h, max_ctas), "pp_set_grid_limit")


def pp_seek(h, step: int) -> None:
    _check(lib().pp_seek(h, step), "pp_seek")


def pp_set_stream(h, stream) -> None:
    _check(lib().pp_set_stream(h, _stream(stream)), "pp_set_stream")


def pp_loader_query(h) -> dict:
    info = pp_loader_info()
    _check(lib().pp_loader_query(h, ctypes.byref(info)), "pp_loader_query")
    return {name: getattr(info, name) for name, _ in pp_loader_info._fields_}


def pp_fill_synthetic(h, data_seed: int) -> None:
    _check(lib().pp_fill_synthetic(h, ctypes.c_uint64(data_seed)), "pp_fill_synthetic")


def pp_get_order(h) -> np.ndarray:
    n = pp_loader_query(h)["epoch_positions"]
    out = np.zeros(n, dtype=np.int64)
    _check(lib().pp_get_order(h, out.ctypes.data), "pp_get_order")
    return out


def pp_read_store(h, row0: int, n: int) -> np.ndarray:
    q = pp_loader_query(h)
    out = np.zeros((n, q["record_bytes_in"]), dtype=np.uint8)
    _check(lib().pp_read_store(h, row0, n, out.ctypes.data), "pp_read_store")
    return out


def pp_link_loopback(handles) -> None:
    arr = (ctypes.c_void_p * len(handles))(*[h.value for h in handles])
    _check(lib().pp_link_loopback(arr, len(handles)), "pp_link_loopback")


def pp_nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (PP_NCCL_ID_BYTES) for PP_PEERS_NCCL loaders; broadcast it to every rank."""
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    _check(lib().pp_nccl_unique_id(buf), "pp_nccl_unique_id")
    return buf.raw


def pp_export_store(h) -> bytes:
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(lib().pp_export_store(h, buf), "pp_export_store")
    return buf.raw


def pp_import_peer_stores(h, handles: bytes) -> None:
    _check(lib().pp_import_peer_stores(h, handles), "pp_import_peer_stores")


def pp_debug_set_sort_bits_delta(h, delta: int) -> None:
    _check(lib().pp_debug_set_sort_bits_delta(h, delta), "pp_debug_set_sort_bits_delta")


# --------------------------------------------------------------------------- convenience handle
class Loader:
    """Owning wrapper around a ``pp_loader*`` (marshalling only)."""

    def __init__(self, **desc):
        self.h = pp_loader_create(**desc)
        self.info = pp_loader_query(self.h)
        self.info_hops = (desc["num_hops"], desc["feat_dim"])
        self._batch_size = desc["batch_size"]
        self._out_dtype = _dtype(desc.get("out_dtype", PP_BF16))
        self._device = desc.get("device", 0)
        # per-batch hot path: the C entry point and the out-parameter bound once
        self._next = lib().pp_next_batch
        self._rows = ctypes.c_int32()
        self._rows_ref = ctypes.byref(self._rows)

    def close(self):
        if self.h is not None and self.h.value:
            pp_loader_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def epoch_permute(self, seed, chunk=1, stream=None):
        pp_epoch_permute(self.h, seed, chunk, stream)

    def epoch_permute_local(self, seed, chunk=1, stream=None):
        pp_epoch_permute_local(self.h, seed, chunk, stream)

    def epoch_prefetch(self, seed, chunk=1):
        pp_epoch_prefetch(self.h, seed, chunk)

    def next_batch(self, out, out_labels=None, out_nodes=None, consumer_stream=None):
        """pp_next_batch: rows written, or -1 at the end of the epoch."""
        rc = self._next(self.h, out.data_ptr() if hasattr(out, "data_ptr") else _ptr(out),
                        None if out_labels is None else _ptr(out_labels),
                        None if out_nodes is None else _ptr(out_nodes), self._rows_ref,
                        None if consumer_stream is None else _stream(consumer_stream))
        if rc == PP_OK:
            return self._rows.value
        if rc == PP_END_OF_EPOCH:
            return -1
        _check(rc, "pp_next_batch")

    def next_batches(self, n, out, out_stride_bytes, out_labels=None, out_nodes=None, consumer_stream=None):
        return pp_next_batches(self.h, n, out, out_stride_bytes, out_labels, out_nodes, consumer_stream)

    def next_batches_ev(self, n, out, out_stride_bytes, out_labels=None, out_nodes=None, wait_event=None,
                        ready_event=None):
        return pp_next_batches_ev(self.h, n, out, out_stride_bytes, out_labels, out_nodes, wait_event, ready_event)

    def next_batches_linear(self, n, W, D, Z, z_dtype, z_stride_bytes, consumer_stream=None):
        return pp_next_batches_linear(self.h, n, W, D, Z, z_dtype, z_stride_bytes, consumer_stream)

    def propagate_store(self, k, row_ptr, col_idx, deg, stream=None):
        pp_propagate_store(self.h, k, row_ptr, col_idx, deg, stream)

    def set_grid_limit(self, max_ctas):
        pp_set_grid_limit(self.h, max_ctas)

    def seek(self, step):
        pp_seek(self.h, step)

    def set_stream(self, stream):
        pp_set_stream(self.h, stream)

    def query(self):
        return pp_loader_query(self.h)

    def epoch(self, seed, chunk=1, depth=2, labels=False, nodes=False, consumer_stream=None):
        """Iterate one epoch with the paper's double buffer: ``depth`` batch
        buffers, batch t+1.. assembled on the loader stream while the consumer works on batch t.

        Yields ``(x, y, v)`` per step: ``x`` the [rows, H, F] batch, ``y`` int32 labels or None,
        ``v`` int64 node ids or None -- views into the ring, valid until the consumer's work
        enqueued on ``consumer_stream`` (default: torch's current stream) after the yield.
        Ordering is by per-buffer events (pp_next_batches_ev); bookkeeping only, no compute."""
        import torch

        H, F = self.info_hops
        B = self._batch_size
        dt = {PP_BF16: torch.bfloat16, PP_F16: torch.float16, PP_F32: torch.float32}[self._out_dtype]
        dev = torch.device("cuda", self._device)
        cons = consumer_stream if consumer_stream is not None else torch.cuda.current_stream(dev)
        bufs = torch.empty((depth, B, H, F), dtype=dt, device=dev)
        ys = torch.empty((depth, B), dtype=torch.int32, device=dev) if labels else None
        vs = torch.empty((depth, B), dtype=torch.int64, device=dev) if nodes else None
        ready = [torch.cuda.Event() for _ in range(depth)]
        free = [torch.cuda.Event() for _ in range(depth)]
        for ev in ready + free:  # torch creates events lazily: materialise them
            ev.record(cons)
        self.epoch_permute(seed, chunk, cons)
        steps = pp_loader_query(self.h)["steps_per_epoch"]
        rows = [0] * depth
        issued = 0

        def issue(t):
            b = t % depth
            r = self.next_batches_ev(1, bufs[b], 0, None if ys is None else ys[b], None if vs is None else vs[b],
                                     free[b], ready[b])
            rows[b] = r[0] if r else 0

        while issued < min(depth - 1, steps):
            issue(issued)
            issued += 1
        for t in range(steps):
            if issued < steps:  # keep depth - 1 batches in flight ahead of the consumer
                issue(issued)
                issued += 1
            b = t % depth
            cons.wait_event(ready[b])
            n = rows[b]
            yield bufs[b, :n], (None if ys is None else ys[b, :n]), (None if vs is None else vs[b, :n])
            free[b].record(cons)

    def fill_synthetic(self, data_seed):
        pp_fill_synthetic(self.h, data_seed)

    def get_order(self):
        return pp_get_order(self.h)

    def read_store(self, row0, n):
        return pp_read_store(self.h, row0, n)
