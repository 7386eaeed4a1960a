"""Compact node-set store (store_set_only): only the labelled nodes' records are kept ("the input
data size after preprocessing is proportional to the number of labeled nodes").
Record i holds node S[i]; batches, labels and node ids must be bit-identical to the oracle's
(O8-O10) -- the same as with a full store -- for host and device sources, spill, sharding over
node-set positions, both gather kernels, the synthetic fill and the fused linear consumer."""
import numpy as np
import pytest

import oracle
from inputs import hop_tensor, node_set as make_node_set

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def bits16(t):
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


def run_epoch(L, bits, hs, rs, H, F, order, B, W, r, labels, k=2):
    steps = oracle.num_steps(order.shape[0], B, W)
    ring = torch.empty((k, B, H, F), dtype=torch.bfloat16, device="cuda")
    nodes = torch.empty((k, B), dtype=torch.int64, device="cuda")
    labs = torch.empty((k, B), dtype=torch.int32, device="cuda")
    t = 0
    while t < steps:
        rows = L.next_batches(k, ring, B * H * F * 2, labs, nodes)
        torch.cuda.synchronize()
        for i, nr in enumerate(rows):
            want, wl, wn = oracle.batch(bits, oracle.F32, hs, rs, H, F, order, B, W, t + i, r, oracle.BF16, labels)
            assert nr == want.shape[0]
            assert np.array_equal(bits16(ring[i, :nr]), want), (r, t + i)
            assert np.array_equal(nodes[i, :nr].cpu().numpy(), wn), (r, t + i)
            assert np.array_equal(labs[i, :nr].cpu().numpy(), wl), (r, t + i)
        t += len(rows)


@pytest.mark.parametrize("source", ["host", "device"])
@pytest.mark.parametrize("budget_rows", [0, 700])
@pytest.mark.parametrize("gather", ["ldg", "tma"])
def test_compact_single_rank(pp, monkeypatch, source, budget_rows, gather):
    monkeypatch.setenv("PPLOAD_GATHER", gather)
    H, N, F, B = 4, 9001, 64, 128
    X, hs, rs = hop_tensor(81, H, N, F)
    S = make_node_set(82, N, 1501)  # ~17 % labelled, unsorted
    labels = (np.arange(N) % 97).astype(np.int32)
    data = X if source == "host" else torch.from_numpy(X.view(np.uint32).view(np.int32)).cuda()
    rec = H * F * 4
    kw = dict(hbm_budget_bytes=budget_rows * rec) if budget_rows else {}
    L = pp.Loader(data=data, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  node_set=S, labels=labels, batch_size=B, out_dtype=pp.PP_BF16, store_set_only=True, **kw)
    q = L.query()
    assert q["local_rows"] == S.shape[0]  # one record per labelled node, not per node
    assert q["rows_spill"] == (S.shape[0] - budget_rows if budget_rows else 0)
    for chunk in (1, 16):
        L.epoch_permute(5 + chunk, chunk)
        order = oracle.epoch_order(5 + chunk, S.shape[0], chunk, node_set=S)
        run_epoch(L, X.view(np.uint32), hs, rs, H, F, order, B, 1, 0, labels)
    L.close()


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("xcast", [0, 1])
def test_compact_loopback_sharded(pp, monkeypatch, W, xcast):
    H, N, F, B = 4, 6007, 48, 96
    X, hs, rs = hop_tensor(83, H, N, F)
    S = make_node_set(84, N, 2222)
    labels = (np.arange(N) % 13).astype(np.int32)
    Ls = []
    for r in range(W):
        monkeypatch.setenv("PPLOAD_EXCHANGE_CAST", str(xcast))
        Ls.append(pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs,
                            dtype=pp.PP_F32, node_set=S, labels=labels, batch_size=B, out_dtype=pp.PP_BF16,
                            store_set_only=True, world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK))
    pp.pp_link_loopback([L.h for L in Ls])
    # sharded over node-set positions: rank r keeps positions r, r + W, ...
    assert [L.query()["local_rows"] for L in Ls] == [len(range(r, S.shape[0], W)) for r in range(W)]
    order = oracle.epoch_order(9, S.shape[0], 8, node_set=S)
    for r, L in enumerate(Ls):
        L.epoch_permute(9, 8)
        run_epoch(L, X.view(np.uint32), hs, rs, H, F, order, B, W, r, labels)
    for L in Ls:
        L.close()


def test_compact_fill_synthetic_matches_generator(pp):
    # record i of a compact store holds node S[i]'s generator values (the generator is a
    # function of the global node id)
    H, N, F = 4, 200_000, 100
    S = make_node_set(85, N, 5000)
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, node_set=S, batch_size=512,
                  out_dtype=pp.PP_BF16, store_set_only=True)
    L.fill_synthetic(2504)
    sample = np.arange(0, S.shape[0], 37)
    got = np.stack([L.read_store(int(i), 1)[0] for i in sample]).view(np.uint32)
    want = oracle.gen_rows(2504, oracle.F32, H, F, S[sample]).reshape(sample.shape[0], -1)
    assert np.array_equal(got, want)
    L.close()


def test_compact_fused_linear(pp):
    # the fused consumer indexes the compact store by node-set position
    H, N, F, B, D = 4, 5000, 64, 256, 256
    X, hs, rs = hop_tensor(86, H, N, F)
    S = make_node_set(87, N, 1800)
    rng = np.random.default_rng(88)
    wb = (rng.standard_normal((H, F, D)) / 8).astype(np.float32)
    wb16 = (wb.view(np.uint32) >> 16).astype(np.uint16)  # truncate to bf16 bit patterns
    Wd = torch.from_numpy(wb16.view(np.int16).copy()).cuda().view(torch.bfloat16)
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  node_set=S, batch_size=B, out_dtype=pp.PP_BF16, store_set_only=True)
    Lf = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   node_set=S, batch_size=B, out_dtype=pp.PP_BF16)
    Z = torch.empty((1, B, H, D), dtype=torch.float32, device="cuda")
    Zf = torch.empty((1, B, H, D), dtype=torch.float32, device="cuda")
    for x in (L, Lf):
        x.epoch_permute(4, 1)
    for _ in range(oracle.num_steps(S.shape[0], B)):
        rows = L.next_batches_linear(1, Wd, D, Z, "f32", 0)
        rows_f = Lf.next_batches_linear(1, Wd, D, Zf, "f32", 0)
        torch.cuda.synchronize()
        assert rows == rows_f
        # same rows, same instruction sequence: bit-identical to the full-store kernel
        assert torch.equal(Z[0, :rows[0]].view(torch.int32), Zf[0, :rows[0]].view(torch.int32))
    L.close()
    Lf.close()


def test_compact_rejections(pp, tmp_path):
    H, N, F = 2, 100, 8
    X, hs, rs = hop_tensor(89, H, N, F)
    with pytest.raises(pp.PPError) as ei:  # needs a node set
        pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  batch_size=8, out_dtype=pp.PP_BF16, store_set_only=True)
    assert ei.value.status == pp.PP_ERR_INVALID
    S = np.arange(0, N, 3, dtype=np.int64)
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  node_set=S, batch_size=8, out_dtype=pp.PP_BF16, store_set_only=True)
    rp = torch.zeros(L.query()["local_rows"] + 1, dtype=torch.int64, device="cuda")
    ci = torch.zeros(1, dtype=torch.int64, device="cuda")
    deg = torch.ones(N, dtype=torch.int32, device="cuda")
    with pytest.raises(pp.PPError) as ei:  # propagation needs every node's record
        L.propagate_store(1, rp, ci, deg)
    assert ei.value.status == pp.PP_ERR_INVALID
    L.close()
