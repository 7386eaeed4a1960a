"""Process-group plumbing for sharded loaders (W > 1, one process per GPU).

torch.distributed only carries bootstrap metadata here (store handles, the NCCL
unique id, the per-epoch arguments); batch data never goes through it -- each
rank's gather kernel reads the owners' stores over NVLink through the imported
handles (PP_PEERS_IPC), or the library's own NCCL communicator exchanges the
rows (PP_PEERS_NCCL).

    import torch.distributed as dist
    from paper_2504_13266_b200 import Loader, PP_PEERS_IPC, dist as ppd
    dist.init_process_group("nccl")
    L = Loader(num_nodes=N, num_hops=H, feat_dim=F, batch_size=B, world_size=W, rank=r,
               peers=PP_PEERS_IPC, device=local_rank, ...)
    ppd.link_ipc(L)                       # or: L = ppd.nccl_loader(num_nodes=N, ...)
    for e in range(E):
        L.epoch_permute(seed0 + e, chunk)  # collective: checked inside the library
        ...
"""
from __future__ import annotations

import hashlib

import torch.distributed as dist

from . import IPC_HANDLE_BYTES, PP_PEERS_NCCL, Loader, pp_export_store, pp_import_peer_stores, pp_nccl_unique_id

HANDLE_BYTES = IPC_HANDLE_BYTES


def exchange_handles(local: bytes, group=None) -> bytes:
    """All-gather every rank's store handle (HANDLE_BYTES bytes); returns them rank-ordered, concatenated."""
    if len(local) != HANDLE_BYTES:
        raise ValueError(f"store handles are {HANDLE_BYTES} bytes")
    W = dist.get_world_size(group)
    out = [None] * W
    dist.all_gather_object(out, local, group=group)
    return b"".join(out)


def link_ipc(loader, group=None) -> None:
    """Export this rank's store, all-gather the handles, import the peers' (PP_PEERS_IPC)."""
    pp_import_peer_stores(loader.h, exchange_handles(pp_export_store(loader.h), group))


def check_epoch_args(seed: int, chunk: int, group=None) -> None:
    """pp_epoch_permute is collective: every rank must pass the same (seed, chunk), otherwise
    the ranks' slices of the global permutation would overlap or leave gaps."""
    digest = hashlib.sha256(f"{seed}:{chunk}".encode()).hexdigest()
    W = dist.get_world_size(group)
    out = [None] * W
    dist.all_gather_object(out, digest, group=group)
    if len(set(out)) != 1:
        raise ValueError(f"pp_epoch_permute arguments differ across ranks: {out}")


def broadcast_nccl_id(group=None, make_id=pp_nccl_unique_id) -> bytes:
    """A fresh NCCL unique id made on rank 0 of `group` and broadcast to every rank (PP_PEERS_NCCL)."""
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def nccl_loader(group=None, **desc) -> Loader:
    """A loader whose steps are exchanged by the library's NCCL all-to-all.  Collective:
    every rank of `group` calls it; world_size / rank default to the group's."""
    desc.setdefault("world_size", dist.get_world_size(group))
    desc.setdefault("rank", dist.get_rank(group))
    return Loader(peers=PP_PEERS_NCCL, nccl_unique_id=broadcast_nccl_id(group), **desc)
