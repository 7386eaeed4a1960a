"""The real multi-process sharded path (PP_PEERS_IPC) with two processes on ONE GPU:
CUDA IPC handles are exchanged over gloo and each rank reads the other's store through
the imported mapping -- the same code that reads a peer GPU's HBM over NVLink."""
import os
import socket
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, chunk, xcast, q, compact=False):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PPLOAD_EXCHANGE_CAST=str(xcast[rank]))
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2504_13266_b200 as pp
    from inputs import hop_tensor
    from paper_2504_13266_b200 import dist as ppd

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H, N, F, B = 4, 6007, 64, 96
        X, hs, rs = hop_tensor(40, H, N, F)
        S = np.random.default_rng(41).choice(N, size=2500, replace=False).astype(np.int64) if compact else None
        L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                      batch_size=B, out_dtype=pp.PP_BF16, world_size=world, rank=rank, peers=pp.PP_PEERS_IPC,
                      node_set=S, store_set_only=compact)
        has_x = L.query()["exchange_cast"]
        ppd.link_ipc(L)
        ppd.check_epoch_args(17, chunk)
        L.epoch_permute(17, chunk)
        order = oracle.epoch_order(17, N if S is None else S.shape[0], chunk, node_set=S)
        out = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
        nodes = torch.empty(B, dtype=torch.int64, device="cuda")
        t, bad = 0, 0
        while (rows := L.next_batch(out, None, nodes)) >= 0:
            torch.cuda.synchronize()
            want, _, wn = oracle.batch(X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, world, t, rank,
                                       oracle.BF16)
            got = out[:rows].view(torch.int16).cpu().numpy().view(np.uint16)
            bad += int(not np.array_equal(got, want)) + int(not np.array_equal(nodes[:rows].cpu().numpy(), wn))
            t += 1
        dist.barrier()  # peers keep their stores alive until everyone is done
        L.close()
        q.put((rank, bad, t == oracle.num_steps(order.shape[0], B, world), has_x))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e), False, None))
    finally:
        dist.destroy_process_group()


# xcast: per-rank PPLOAD_EXCHANGE_CAST -- peers read the owner's cast exchange copy (1) or its fp32
# records (0); mixed ranks exercise both in one epoch.  Batches are bit-identical either way.
@pytest.mark.parametrize("chunk,xcast,compact", [(1, (1, 1), False), (64, (1, 1), False), (1, (0, 0), False),
                                                 (64, (1, 0), False), (16, (1, 0), True)])
def test_ipc_two_processes_one_gpu(chunk, xcast, compact):
    import torch.multiprocessing as mp

    import __graft_entry__ as ge

    ge.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, chunk, xcast, q, compact)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, bad, steps_ok, has_x in res:
        assert bad == 0 and steps_ok, (rank, bad)
        assert has_x == xcast[rank]
