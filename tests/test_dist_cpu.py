"""Host-side multi-process logic of the sharded path on CPU: world_size 2 over gloo."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_13266_b200 import dist as ppd

        n = ppd.HANDLE_BYTES
        hs = ppd.exchange_handles(bytes([rank]) * n)
        ok_handles = hs == b"".join(bytes([r]) * n for r in range(world))
        ppd.check_epoch_args(250413266, 8192)
        try:
            ppd.check_epoch_args(250413266 + rank, 8192)
            mismatch_raised = False
        except ValueError:
            mismatch_raised = True
        uid = ppd.broadcast_nccl_id(make_id=lambda: bytes(range(128)))  # plumbing only: a fake id
        q.put((rank, ok_handles and uid == bytes(range(128)), mismatch_raised))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_handle_exchange_and_arg_check_gloo(world):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.environ["PYTHONPATH"] = root + os.pathsep + os.environ.get("PYTHONPATH", "")
    sys.path.insert(0, root)
    import __graft_entry__ as ge

    ge.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_handles, mismatch_raised in res:
        assert ok_handles and mismatch_raised
