"""Exchange copy of sharded loaders (pp_loader.h): every rank keeps its HBM
rows already cast to the batch dtype and peers read remote rows from that copy, so only
the cast bytes cross NVLink.  The batches must stay bit-identical to the oracle (O9/O10)
whether a given owner exports a copy or not, with spill, node sets and both kernels."""
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


TORCH_DT = {oracle.BF16: torch.bfloat16, oracle.F16: torch.float16, oracle.F32: torch.float32}


def bits_of(t, dt):
    x = t.detach().cpu()
    if dt == oracle.F32:
        return x.view(torch.int32).numpy().view(np.uint32)
    return x.view(torch.int16).numpy().view(np.uint16)


def make_ranks(pp, monkeypatch, W, xcast, **kw):
    Ls = []
    for r in range(W):
        monkeypatch.setenv("PPLOAD_EXCHANGE_CAST", str(xcast[r]))
        Ls.append(pp.Loader(world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK, **kw))
    pp.pp_link_loopback([L.h for L in Ls])
    return Ls


def check_ranks(Ls, bits, in_dt, hs, rs, H, F, order, B, out_dt, k=3):
    W = len(Ls)
    n = order.shape[0]
    steps = oracle.num_steps(n, B, W)
    s_out = 4 if out_dt == oracle.F32 else 2
    for r, L in enumerate(Ls):
        ring = torch.empty((k, B, H, F), dtype=TORCH_DT[out_dt], device="cuda")
        nodes = torch.empty((k, B), dtype=torch.int64, device="cuda")
        t = 0
        while t < steps:
            rows = L.next_batches(k, ring, B * H * F * s_out, None, nodes)
            torch.cuda.synchronize()
            for i, nr in enumerate(rows):
                want, _, wn = oracle.batch(bits, in_dt, hs, rs, H, F, order, B, W, t + i, r, out_dt)
                assert nr == want.shape[0]
                assert np.array_equal(nodes[i, :nr].cpu().numpy(), wn), (r, t + i)
                assert np.array_equal(bits_of(ring[i, :nr], out_dt), want), (r, t + i)
            t += len(rows)


@pytest.mark.parametrize("gather", ["ldg", "tma"])
@pytest.mark.parametrize("W,xcast", [(2, (1, 1)), (2, (0, 0)), (3, (1, 0, 1)), (4, (1, 1, 1, 1))])
@pytest.mark.parametrize("out_dt", [oracle.BF16, oracle.F16])
def test_exchange_copy_bit_exact(pp, monkeypatch, gather, W, xcast, out_dt):
    monkeypatch.setenv("PPLOAD_GATHER", gather)
    H, N, F, B = 4, 4007, 56, 160
    X, hs, rs = hop_tensor(71, H, N, F)
    Ls = make_ranks(pp, monkeypatch, W, xcast, data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs,
                    row_stride=rs, dtype=pp.PP_F32, batch_size=B, out_dtype=out_dt)
    try:
        assert [L.query()["exchange_cast"] for L in Ls] == list(xcast)
        order = oracle.epoch_order(5, N, 16)
        for L in Ls:
            L.epoch_permute(5, 16)
        check_ranks(Ls, X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, out_dt)
    finally:
        for L in Ls:
            L.close()


def test_exchange_copy_with_spill_and_node_set(pp, monkeypatch):
    # HBM rows of each owner come from its exchange copy, spilled rows from its fp32 host records
    W, H, N, F, B = 2, 3, 3001, 40, 128
    X, hs, rs = hop_tensor(72, H, N, F, "hop_major")
    S = make_node_set(73, N, 2500)
    Ls = make_ranks(pp, monkeypatch, W, (1, 1), data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs,
                    row_stride=rs, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16, node_set=S,
                    hbm_budget_bytes=900 * H * F * 4)
    try:
        for L in Ls:
            q = L.query()
            assert q["exchange_cast"] == 1 and q["rows_spill"] > 0
        order = oracle.epoch_order(8, S.shape[0], 1, node_set=S)
        for L in Ls:
            L.epoch_permute(8, 1)
        check_ranks(Ls, X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, oracle.BF16)
    finally:
        for L in Ls:
            L.close()


def test_exchange_copy_follows_fill_synthetic(pp, monkeypatch):
    # a store written by pp_fill_synthetic after create: the exchange copy is rewritten with it
    W, H, N, F, B = 2, 4, 2003, 64, 256
    Ls = make_ranks(pp, monkeypatch, W, (1, 1), num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32,
                    batch_size=B, out_dtype=pp.PP_BF16)
    try:
        for L in Ls:
            L.fill_synthetic(2504)
        bits = oracle.gen_rows(2504, oracle.F32, H, F, np.arange(N))  # [N, H, F] node-major
        order = oracle.epoch_order(3, N, 1)
        for L in Ls:
            L.epoch_permute(3, 1)
        check_ranks(Ls, bits, oracle.F32, F, H * F, H, F, order, B, oracle.BF16)
        for L in Ls:  # refill with another seed: batches follow the new values
            L.fill_synthetic(77)
        bits = oracle.gen_rows(77, oracle.F32, H, F, np.arange(N))
        for L in Ls:
            L.epoch_permute(4, 1)
        check_ranks(Ls, bits, oracle.F32, F, H * F, H, F, oracle.epoch_order(4, N, 1), B, oracle.BF16)
    finally:
        for L in Ls:
            L.close()


def test_no_exchange_copy_without_cast(pp, monkeypatch):
    # 16-bit stores are copied bit for bit: there is nothing to cast, so no exchange copy
    W, H, N, F, B = 2, 2, 1001, 64, 64
    X, hs, rs = hop_tensor(74, H, N, F, dtype=np.uint16)
    Ls = make_ranks(pp, monkeypatch, W, (1, 1), data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs,
                    row_stride=rs, dtype=pp.PP_F16, batch_size=B, out_dtype=pp.PP_F16)
    try:
        assert [L.query()["exchange_cast"] for L in Ls] == [0, 0]
        order = oracle.epoch_order(6, N, 1)
        for L in Ls:
            L.epoch_permute(6, 1)
        check_ranks(Ls, X, oracle.F16, hs, rs, H, F, order, B, oracle.F16)
    finally:
        for L in Ls:
            L.close()
