"""§8(f)-2, sharded: pre-propagation into the loader's node-major store (pp_propagate_store).

Each rank computes hop slot k of the nodes it owns from hop slot k-1 of every owner's records
(local HBM, the pinned spill, or a peer store).  The arithmetic is the oracle's definition
(O2/O3), so every slot of every rank must equal oracle.propagate bit for bit, and batches
assembled afterwards (including peer rows read from the exchange copy) must equal the
oracle's batches of those hops."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def local_csr(rp, ci, W, r):
    """CSR rows of the nodes r, r+W, r+2W, ... (global column ids), as device tensors."""
    rows = np.arange(r, rp.shape[0] - 1, W)
    lens = rp[rows + 1] - rp[rows]
    lrp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    lci = np.concatenate([ci[rp[i]:rp[i + 1]] for i in rows]).astype(np.int64) if rows.size else np.zeros(0, np.int64)
    return torch.from_numpy(lrp).cuda(), torch.from_numpy(lci).cuda()


def store_hops(L, H, F):
    q = L.query()
    return L.read_store(0, q["local_rows"]).view(np.float32).reshape(q["local_rows"], H, F)


def graph(n, m, seed):
    rng = np.random.default_rng(seed)
    return oracle.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m))


def make_shards(pp, monkeypatch, W, X, H, xcast=1, **kw):
    n, F = X.shape
    Ls = []
    for r in range(W):
        monkeypatch.setenv("PPLOAD_EXCHANGE_CAST", str(xcast))
        # hop_stride = 0: X broadcast into every hop slot (slots 1..K are overwritten)
        Ls.append(pp.Loader(data=X, num_nodes=n, num_hops=H, feat_dim=F, hop_stride=0, row_stride=F, dtype=pp.PP_F32,
                            world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK if W > 1 else pp.PP_PEERS_NONE, **kw))
    if W > 1:
        pp.pp_link_loopback([L.h for L in Ls])
    return Ls


def propagate_all(Ls, rp, ci, K):
    W = len(Ls)
    deg = torch.from_numpy(np.diff(rp).astype(np.int32)).cuda()
    csrs = [local_csr(rp, ci, W, r) for r in range(W)]
    s = torch.cuda.current_stream()
    for k in range(1, K + 1):
        for L, (lrp, lci) in zip(Ls, csrs):
            L.propagate_store(k, lrp, lci, deg, s)  # one stream: hop k of every shard after hop k-1
    torch.cuda.synchronize()


def check_store(Ls, want, H, F):
    W = len(Ls)
    for r, L in enumerate(Ls):
        got = store_hops(L, H, F)
        exp = np.ascontiguousarray(want[:, r::W, :].transpose(1, 0, 2))
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), r


def test_config1_single_rank(pp, monkeypatch):
    n, m, F, K = 2708, 5429, 128, 3
    src, dst = oracle.gen_graph(2504, n, m)
    rp, ci = oracle.build_csr(n, src, dst)
    X = oracle.gen_rows(2504, oracle.F32, 1, F, np.arange(n)).reshape(n, F).view(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    Ls = make_shards(pp, monkeypatch, 1, X, K + 1, batch_size=256, out_dtype=pp.PP_BF16)
    propagate_all(Ls, rp, ci, K)
    check_store(Ls, want, K + 1, F)
    # the loader then serves the oracle's batches of the propagated hops
    L = Ls[0]
    hops = np.ascontiguousarray(want)  # [H, n, F]
    order = oracle.epoch_order(9, n, 1)
    L.epoch_permute(9, 1)
    out = torch.empty((256, K + 1, F), dtype=torch.bfloat16, device="cuda")
    for t in range(oracle.num_steps(n, 256)):
        rows = L.next_batch(out)
        torch.cuda.synchronize()
        exp, _, _ = oracle.batch(hops.view(np.uint32), oracle.F32, n * F, F, K + 1, F, order, 256, 1, t, 0, oracle.BF16)
        assert np.array_equal(out[:rows].view(torch.int16).cpu().numpy().view(np.uint16), exp), t
    L.close()


@pytest.mark.parametrize("n,m,F,K", [(1, 0, 4, 1), (300, 1500, 7, 3), (1000, 9000, 100, 2), (700, 5000, 256, 2),
                                     (900, 3000, 132, 1)])
@pytest.mark.parametrize("W", [1, 2, 3])
def test_random_graphs_sharded(pp, monkeypatch, n, m, F, K, W):
    if W > n:
        pytest.skip("more ranks than nodes")
    rp, ci = graph(n, m, n + F + W)
    X = np.random.default_rng(F).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    Ls = make_shards(pp, monkeypatch, W, X, K + 1, batch_size=64, out_dtype=pp.PP_BF16)
    propagate_all(Ls, rp, ci, K)
    check_store(Ls, want, K + 1, F)
    for L in Ls:
        L.close()


@pytest.mark.parametrize("F", [64, 100])
def test_spilled_rows(pp, monkeypatch, F):
    # W = 1 with most rows in pinned host memory: neighbours are read and results written over PCIe
    n, m, K = 3000, 20000, 3
    rp, ci = graph(n, m, 77)
    X = np.random.default_rng(1).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    rec = (K + 1) * F * 4
    Ls = make_shards(pp, monkeypatch, 1, X, K + 1, batch_size=64, out_dtype=pp.PP_BF16, hbm_budget_bytes=rec * 1000)
    assert Ls[0].query()["rows_spill"] == n - 1000
    propagate_all(Ls, rp, ci, K)
    check_store(Ls, want, K + 1, F)
    Ls[0].close()


@pytest.mark.parametrize("xcast", [0, 1])
@pytest.mark.parametrize("out_dt", [oracle.BF16, oracle.F16])
def test_exchange_copy_follows_the_propagated_hops(pp, monkeypatch, xcast, out_dt):
    # W = 3: peers read remote rows from the owner's exchange copy, whose slots 1..K the
    # propagation kernel rewrote with the cast; every batch must match the oracle's
    W, n, m, F, K, B = 3, 2000, 12000, 48, 3, 96
    rp, ci = graph(n, m, 5)
    X = np.random.default_rng(2).standard_normal((n, F)).astype(np.float32)
    want = np.ascontiguousarray(oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K))
    Ls = make_shards(pp, monkeypatch, W, X, K + 1, xcast=xcast, batch_size=B, out_dtype=out_dt)
    assert [L.query()["exchange_cast"] for L in Ls] == [xcast] * W
    propagate_all(Ls, rp, ci, K)
    order = oracle.epoch_order(3, n, 8)
    tdt = torch.bfloat16 if out_dt == oracle.BF16 else torch.float16
    for r, L in enumerate(Ls):
        L.epoch_permute(3, 8)
        out = torch.empty((B, K + 1, F), dtype=tdt, device="cuda")
        for t in range(oracle.num_steps(n, B, W)):
            rows = L.next_batch(out)
            torch.cuda.synchronize()
            exp, _, _ = oracle.batch(want.view(np.uint32), oracle.F32, n * F, F, K + 1, F, order, B, W, t, r, out_dt)
            assert rows == exp.shape[0]
            assert np.array_equal(out[:rows].view(torch.int16).cpu().numpy().view(np.uint16), exp), (r, t)
    for L in Ls:
        L.close()


@pytest.mark.parametrize("F", [8, 100])
def test_scalar_and_vector_kernels_agree(pp, monkeypatch, F):
    n, m, K = 800, 6000, 2
    rp, ci = graph(n, m, F)
    X = np.random.default_rng(F).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    monkeypatch.setenv("PPLOAD_SPMM", "scalar")
    Ls = make_shards(pp, monkeypatch, 2, X, K + 1, batch_size=64, out_dtype=pp.PP_BF16)
    propagate_all(Ls, rp, ci, K)
    check_store(Ls, want, K + 1, F)
    for L in Ls:
        L.close()


def test_invalid_arguments(pp, monkeypatch):
    n, F = 50, 8
    rp, ci = graph(n, 100, 0)
    lrp, lci = local_csr(rp, ci, 1, 0)
    deg = torch.from_numpy(np.diff(rp).astype(np.int32)).cuda()
    X = np.zeros((n, F), np.float32)
    L = make_shards(pp, monkeypatch, 1, X, 3, batch_size=8, out_dtype=pp.PP_BF16)[0]
    for k in (0, 3, -1):
        with pytest.raises(pp.PPError) as ei:
            L.propagate_store(k, lrp, lci, deg)
        assert ei.value.status == pp.PP_ERR_INVALID
    with pytest.raises(pp.PPError) as ei:
        L.propagate_store(1, None, lci, deg)
    assert ei.value.status == pp.PP_ERR_INVALID
    L.close()
    L16 = pp.Loader(data=X.astype(np.float16), num_nodes=n, num_hops=2, feat_dim=F, hop_stride=0, row_stride=F,
                    dtype=pp.PP_F16, batch_size=8, out_dtype=pp.PP_F16)
    with pytest.raises(pp.PPError) as ei:
        L16.propagate_store(1, lrp, lci, deg)
    assert ei.value.status == pp.PP_ERR_INVALID
    L16.close()
    # an unlinked loopback shard refuses (its peers' stores are unknown)
    Lu = pp.Loader(data=X, num_nodes=n, num_hops=2, feat_dim=F, hop_stride=0, row_stride=F, dtype=pp.PP_F32,
                   batch_size=8, out_dtype=pp.PP_BF16, world_size=2, rank=0, peers=pp.PP_PEERS_LOOPBACK)
    with pytest.raises(pp.PPError) as ei:
        Lu.propagate_store(1, lrp, lci, deg)
    assert ei.value.status == pp.PP_ERR_STATE
    Lu.close()


def _ipc_worker(rank, world, port, q):
    import os
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2504_13266_b200 as pp
    from paper_2504_13266_b200 import dist as ppd

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m, F, K = 3001, 20000, 64, 3
        rp, ci = graph(n, m, 11)
        X = np.random.default_rng(12).standard_normal((n, F)).astype(np.float32)
        L = pp.Loader(data=X, num_nodes=n, num_hops=K + 1, feat_dim=F, hop_stride=0, row_stride=F, dtype=pp.PP_F32,
                      batch_size=64, out_dtype=pp.PP_BF16, world_size=world, rank=rank, peers=pp.PP_PEERS_IPC)
        ppd.link_ipc(L)
        lrp, lci = local_csr(rp, ci, world, rank)
        deg = torch.from_numpy(np.diff(rp).astype(np.int32)).cuda()
        for k in range(1, K + 1):
            L.propagate_store(k, lrp, lci, deg, torch.cuda.current_stream())
            torch.cuda.synchronize()
            dist.barrier()  # every owner's slot k is complete before anyone reads it
        want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
        got = store_hops(L, K + 1, F)
        exp = np.ascontiguousarray(want[:, rank::world, :].transpose(1, 0, 2))
        ok = bool(np.array_equal(got.view(np.uint32), exp.view(np.uint32)))
        dist.barrier()
        L.close()
        q.put((rank, ok))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_ipc_two_processes_one_gpu(pp):
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)], res
