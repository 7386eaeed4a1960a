"""Two real processes on one GPU (PP_PEERS_IPC), round-2 additions:

* a spilled shard: the owner's spill is a shared-memory file that the peer maps and registers at
  pp_import_peer_stores, so rows beyond a rank's HBM budget are readable by every rank (host
  placement of data beyond GPU memory) -- batches bit-identical to the oracle;
* the collective check of pp_epoch_permute over the IPC-mapped flag words: differing (seed, chunk)
  -> PP_ERR_INVALID on both ranks with the previous epoch kept; a rank that never arrives ->
  PP_ERR_STATE after PPLOAD_COLLECTIVE_TIMEOUT_S.
"""
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


def _worker(rank, world, port, mode, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PPLOAD_COLLECTIVE_TIMEOUT_S="3")
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2504_13266_b200 as pp
    from inputs import hop_tensor
    from paper_2504_13266_b200 import dist as ppd

    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {"rank": rank}
    try:
        H, N, F, B = 4, 6007, 64, 96
        X, hs, rs = hop_tensor(60, H, N, F)
        budget = (1000 + 700 * rank) * H * F * 4 if mode == "spill" else 0
        L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                      batch_size=B, out_dtype=pp.PP_BF16, world_size=world, rank=rank, peers=pp.PP_PEERS_IPC,
                      hbm_budget_bytes=budget)
        info = L.query()
        res["spill"] = (info["rows_spill"], info["spill_shared"], info["host_spill_bytes"])
        ppd.link_ipc(L)

        def epoch_ok(seed, chunk):
            order = oracle.epoch_order(seed, N, chunk)
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
            return bad == 0 and t == oracle.num_steps(N, B, world)

        if mode == "spill":
            L.epoch_permute(17, 1)
            res["ok"] = epoch_ok(17, 1)
            L.epoch_permute(18, 32)
            res["ok"] = res["ok"] and epoch_ok(18, 32)
        elif mode == "mismatch":
            L.epoch_permute(5, 1)
            try:
                L.epoch_permute(6 + rank, 1)  # ranks disagree
                res["status"] = 0
            except pp.PPError as e:
                res["status"] = e.status
            L.seek(0)
            res["ok"] = epoch_ok(5, 1)  # the previous epoch is kept
            L.epoch_permute(9, 4)  # agreeing again: the sequence numbers stay in step
            res["ok"] = res["ok"] and epoch_ok(9, 4)
        elif mode == "timeout":
            if rank == 0:
                try:
                    L.epoch_permute(5, 1)
                    res["status"] = 0
                except pp.PPError as e:
                    res["status"] = e.status
            dist.barrier()
            L.epoch_permute(7, 1)  # both arrive now
            res["ok"] = epoch_ok(7, 1)
        dist.barrier()  # peers keep their stores alive until everyone is done
        L.close()
    except Exception as e:  # pragma: no cover - reported through the queue
        res["error"] = repr(e)
    finally:
        q.put(res)
        dist.destroy_process_group()


def _run(mode):
    import torch.multiprocessing as mp

    import __graft_entry__ as ge

    ge.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(2)), key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
    for d in res:
        assert "error" not in d, d
    return res


def test_ipc_spilled_shards_shared():
    res = _run("spill")
    for d in res:
        rows_spill, shared, spill_bytes = d["spill"]
        assert rows_spill > 0 and shared == 1 and spill_bytes >= rows_spill * 4 * 64 * 4, d
        assert d["ok"], d


def test_ipc_epoch_argument_mismatch():
    import paper_2504_13266_b200 as pp

    for d in _run("mismatch"):
        assert d["status"] == pp.PP_ERR_INVALID, d
        assert d["ok"], d


def test_ipc_epoch_peer_timeout():
    import paper_2504_13266_b200 as pp

    res = _run("timeout")
    assert res[0]["status"] == pp.PP_ERR_STATE, res
    assert all(d["ok"] for d in res), res


def test_shard_larger_than_hbm_spills_to_shared_host_memory():
    """The memory plan at scale (configs[4]'s situation: a rank's shard exceeds its HBM): the
    automatic budget keeps 2 GiB + the loader's own scratch free, the remaining rows go to the shared
    spill, and records on both sides of the split hold the generator's values (O11)."""
    import numpy as np
    import torch

    import __graft_entry__ as ge
    import oracle

    ge.build()
    import paper_2504_13266_b200 as pp

    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    H, F = 1, 1024
    rec = H * F * 4
    rows = (free + (3 << 30)) // rec  # 3 GiB more than the whole free HBM
    N = 2 * rows
    with pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=4096, out_dtype=pp.PP_BF16,
                   world_size=2, rank=1, peers=pp.PP_PEERS_IPC) as L:
        q = L.query()
        assert q["local_rows"] == rows and q["rows_spill"] > 0 and q["spill_shared"] == 1
        assert q["rows_hbm"] + q["rows_spill"] == rows
        assert q["host_spill_bytes"] == q["rows_spill"] * rec
        assert q["hbm_store_bytes"] <= free - (2 << 30) - N * 4  # order + sort scratch + reserve stay free
        assert q["hbm_store_bytes"] >= free - (2 << 30) - 4 * N * 4 - (1 << 27)
        L.fill_synthetic(2504)
        for lr in (0, q["rows_hbm"] - 1, q["rows_hbm"], rows - 1):
            got = L.read_store(int(lr), 1)[0].view(np.uint32)
            assert np.array_equal(got, oracle.gen_rows(2504, oracle.F32, H, F, np.array([lr * 2 + 1]))[0].ravel())
        L.epoch_permute_local(3, 1)  # this rank's own rows, HBM and spill: no peers needed
        out = torch.empty((4096, H, F), dtype=torch.bfloat16, device="cuda")
        nodes = torch.empty(4096, dtype=torch.int64, device="cuda")
        assert L.next_batch(out, None, nodes) == 4096
        torch.cuda.synchronize()
        v = nodes.cpu().numpy()
        assert np.all(v % 2 == 1)
        want = oracle.cast_bf16(oracle.gen_rows(2504, oracle.F32, H, F, v))
        assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), want)
