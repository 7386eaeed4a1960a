"""Process-group plumbing for sharded loaders (W > 1, one process per GPU).

torch.distributed only carries bootstrap metadata here (store handles and the
per-epoch arguments); batch data never goes through it -- each rank's gather
kernel reads the owners' stores over NVLink through the imported handles.
"""
from __future__ import annotations

import hashlib

import torch.distributed as dist

from . import IPC_HANDLE_BYTES, pp_export_store, pp_import_peer_stores

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
