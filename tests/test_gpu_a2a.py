"""The all-to-all exchange of SURVEY.md §8(e) (the NCCL baseline, K9): per step every owner packs the
rows it holds for each rank (cast fused) and the receiver unpacks them into batch order; the
per-step counts come from the shared order ("distributing data across multiple GPUs").

* PP_PEERS_LOOPBACK with PPLOAD_EXCHANGE=a2a runs the count table, the stable compaction by owner
  (k_a2a_index), the pack (the gather kernel over each owner's shard) and the unpack for W shards on
  one GPU -- everything but the transport;
* PP_PEERS_NCCL with W = 1 runs the whole path through NCCL (ncclSend / ncclRecv to itself inside a
  group, the argument all-reduce) on one GPU.
Every batch, label and node id equals the oracle's (O8-O10) bit for bit."""
import numpy as np
import pytest

import oracle
from inputs import hop_tensor, labels as make_labels, node_set as make_node_set

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TORCH_DT = {oracle.BF16: torch.bfloat16, oracle.F16: torch.float16, oracle.F32: torch.float32}


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def bits_of(t, dt):
    x = t.detach().cpu()
    if dt == oracle.F32:
        return x.view(torch.int32).numpy().view(np.uint32)
    return x.view(torch.int16).numpy().view(np.uint16)


def check_ranks(Ls, bits, in_dt, hs, rs, H, F, order, B, out_dt, lab=None, k=3, misalign=False):
    W = len(Ls)
    n = order.shape[0]
    steps = oracle.num_steps(n, B, W)
    s_out = 4 if out_dt == oracle.F32 else 2
    for r, L in enumerate(Ls):
        assert L.query()["all_to_all"] == 1
        if misalign:  # 2-byte aligned slots: the unpack's element path
            buf = torch.empty(k * B * H * F + 8, dtype=TORCH_DT[out_dt], device="cuda")
            ring = buf[1: 1 + k * B * H * F].view(k, B, H, F)
        else:
            ring = torch.empty((k, B, H, F), dtype=TORCH_DT[out_dt], device="cuda")
        nodes = torch.empty((k, B), dtype=torch.int64, device="cuda")
        labs = torch.empty((k, B), dtype=torch.int32, device="cuda") if lab is not None else None
        t = 0
        while t < steps:
            rows = L.next_batches(k, ring, B * H * F * s_out, labs, nodes)
            torch.cuda.synchronize()
            for i, nr in enumerate(rows):
                want, wl, wn = oracle.batch(bits, in_dt, hs, rs, H, F, order, B, W, t + i, r, out_dt, lab)
                assert nr == want.shape[0], (r, t + i)
                assert np.array_equal(nodes[i, :nr].cpu().numpy(), wn), (r, t + i)
                assert np.array_equal(bits_of(ring[i, :nr], out_dt), want), (r, t + i)
                if lab is not None:
                    assert np.array_equal(labs[i, :nr].cpu().numpy(), wl), (r, t + i)
            t += len(rows)
        assert L.next_batch(ring[0]) == -1


def loopback(pp, monkeypatch, W, **kw):
    monkeypatch.setenv("PPLOAD_EXCHANGE", "a2a")
    Ls = [pp.Loader(world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK, **kw) for r in range(W)]
    pp.pp_link_loopback([L.h for L in Ls])
    return Ls


@pytest.mark.parametrize("W", [2, 3, 4, 8])
@pytest.mark.parametrize("chunk", [1, 16, 3000])
def test_loopback_a2a_bit_exact(pp, monkeypatch, W, chunk):
    H, N, F, B = 4, 6007, 56, 300
    X, hs, rs = hop_tensor(90 + W, H, N, F)
    lab = make_labels(91, N)
    Ls = loopback(pp, monkeypatch, W, data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs,
                  dtype=pp.PP_F32, labels=lab, batch_size=B, out_dtype=pp.PP_BF16)
    try:
        for L in Ls:
            assert L.query()["exchange_cast"] == 0  # the a2a path casts while packing
            L.epoch_permute(12, chunk)
        check_ranks(Ls, X.view(np.uint32), oracle.F32, hs, rs, H, F, oracle.epoch_order(12, N, chunk), B,
                    oracle.BF16, lab)
    finally:
        for L in Ls:
            L.close()


@pytest.mark.parametrize("case", ["f16", "copy16", "nodeset", "compact", "spill", "scalar", "drop_last", "misalign"])
def test_loopback_a2a_variants(pp, monkeypatch, case):
    W, H, N, F, B = 3, 3, 4001, 40, 256
    out_dt = oracle.F16 if case in ("f16", "copy16") else oracle.BF16
    dt16 = case == "copy16"
    if case == "scalar":
        F = 7  # H*F*4 not a multiple of 32: the scalar gather packs
    X, hs, rs = hop_tensor(95, H, N, F, "hop_major", dtype=np.uint16 if dt16 else np.float32)
    in_dt = oracle.F16 if dt16 else oracle.F32
    bits = X if dt16 else X.view(np.uint32)
    kw = dict(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=in_dt,
              batch_size=B, out_dtype=out_dt)
    S = None
    if case in ("nodeset", "compact"):
        S = make_node_set(96, N, 2900)
        kw["node_set"] = S
        kw["store_set_only"] = case == "compact"
    if case == "spill":
        kw["hbm_budget_bytes"] = 500 * H * F * 4
    if case == "drop_last":
        kw["drop_last"] = True
    Ls = loopback(pp, monkeypatch, W, **kw)
    try:
        n = N if S is None else S.shape[0]
        order = oracle.epoch_order(13, n, 8, node_set=S)
        for L in Ls:
            L.epoch_permute(13, 8)
        if case == "drop_last":
            steps = n // (W * B)
            order = order[: steps * W * B]  # the oracle's batches of the kept steps are unchanged
            assert Ls[0].query()["steps_per_epoch"] == steps
        check_ranks(Ls, bits, in_dt, hs, rs, H, F, order, B, out_dt, misalign=case == "misalign")
    finally:
        for L in Ls:
            L.close()


def test_nccl_self_exchange_one_rank(pp):
    # W = 1 through NCCL: the argument all-reduce, the count table, pack -> ncclSend / ncclRecv to
    # itself -> unpack; batches equal the oracle's
    H, N, F, B = 4, 20_011, 64, 1024
    X, hs, rs = hop_tensor(97, H, N, F)
    lab = make_labels(98, N)
    uid = pp.pp_nccl_unique_id()
    assert len(uid) == pp.NCCL_ID_BYTES
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  labels=lab, batch_size=B, out_dtype=pp.PP_BF16, peers=pp.PP_PEERS_NCCL, nccl_unique_id=uid)
    try:
        for seed, chunk in ((5, 1), (6, 128)):
            L.epoch_permute(seed, chunk)
            check_ranks([L], X.view(np.uint32), oracle.F32, hs, rs, H, F, oracle.epoch_order(seed, N, chunk), B,
                        oracle.BF16, lab)
    finally:
        L.close()
    with pytest.raises(pp.PPError) as ei:  # NCCL loaders need the id
        pp.Loader(num_nodes=10, num_hops=1, feat_dim=8, batch_size=2, peers=pp.PP_PEERS_NCCL)
    assert ei.value.status == pp.PP_ERR_INVALID
