"""Chunk reshuffling over host-resident rows through the copy engines (the paper's chunk transfer,
PAPER.md:269): under chunk reshuffling a batch is a few runs of consecutive records, each moved
by one cudaMemcpyAsync into a staging area in batch order, then cast on the GPU.  Every batch,
label and node id must equal the oracle's (O8-O10), whatever mix of HBM and pinned-host rows
the runs cross."""
import numpy as np
import pytest

import oracle
from inputs import hop_tensor, node_set as make_node_set

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


def check_epoch(L, bits, in_dt, hs, rs, H, F, order, B, out_dt, labels=None, k=3):
    steps = oracle.num_steps(order.shape[0], B)
    s_out = 4 if out_dt == oracle.F32 else 2
    ring = torch.empty((k, B, H, F), dtype=TORCH_DT[out_dt], device="cuda")
    nodes = torch.empty((k, B), dtype=torch.int64, device="cuda")
    labs = torch.empty((k, B), dtype=torch.int32, device="cuda") if labels is not None else None
    t = 0
    while t < steps:
        rows = L.next_batches(k, ring, B * H * F * s_out, labs, nodes)
        torch.cuda.synchronize()
        for i, nr in enumerate(rows):
            want, wl, wn = oracle.batch(bits, in_dt, hs, rs, H, F, order, B, 1, t + i, 0, out_dt, labels)
            assert nr == want.shape[0]
            assert np.array_equal(bits_of(ring[i, :nr], out_dt), want), t + i
            assert np.array_equal(nodes[i, :nr].cpu().numpy(), wn), t + i
            if labels is not None:
                assert np.array_equal(labs[i, :nr].cpu().numpy(), wl), t + i
        t += len(rows)


@pytest.mark.parametrize("budget_rows", [-1, 1000])
@pytest.mark.parametrize("chunk", [64, 256, 4007])
def test_dma_path_chunks(pp, budget_rows, chunk):
    H, N, F, B = 4, 4007, 64, 200
    X, hs, rs = hop_tensor(91, H, N, F)
    labels = (np.arange(N) % 41).astype(np.int32)
    budget = -1 if budget_rows < 0 else budget_rows * H * F * 4
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  labels=labels, batch_size=B, out_dtype=pp.PP_BF16, hbm_budget_bytes=budget)
    assert L.query()["rows_spill"] == (N if budget_rows < 0 else N - budget_rows)
    for seed in (1, 2):
        L.epoch_permute(seed, chunk)
        check_epoch(L, X.view(np.uint32), oracle.F32, hs, rs, H, F, oracle.epoch_order(seed, N, chunk), B,
                    oracle.BF16, labels)
    L.close()


@pytest.mark.parametrize("compact", [False, True])
def test_dma_path_node_set_forced(pp, monkeypatch, compact):
    # forced (c = 1 and 8 are below the automatic threshold): runs of length 1 still assemble exactly
    monkeypatch.setenv("PPLOAD_SPILL_PATH", "dma")
    H, N, F, B = 3, 3001, 40, 128
    X, hs, rs = hop_tensor(92, H, N, F)
    S = make_node_set(93, N, 1700)
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  node_set=S, batch_size=B, out_dtype=pp.PP_F16, hbm_budget_bytes=500 * H * F * 4,
                  store_set_only=compact)
    for chunk in (1, 8):
        L.epoch_permute(3 + chunk, chunk)
        check_epoch(L, X.view(np.uint32), oracle.F32, hs, rs, H, F, oracle.epoch_order(3 + chunk, S.shape[0], chunk, S),
                    B, oracle.F16)
    L.close()


@pytest.mark.parametrize("F,dt", [(128, oracle.F16), (5, oracle.F16), (7, oracle.F32)])
def test_dma_path_copy_and_scalar_records(pp, F, dt):
    # 16-bit stores are copied bit for bit; F = 5 / 7 rule out 16-byte vectors (scalar cast kernel)
    H, N, B, chunk = 2, 2500, 96, 32
    rng = np.random.default_rng(F)
    if dt == oracle.F32:
        X = rng.standard_normal((H, N, F)).astype(np.float32)
        bits, pdt, out_dt = X.view(np.uint32), pp.PP_F32, oracle.BF16
    else:
        bits = (rng.integers(0, 1 << 16, (H, N, F), dtype=np.uint16) & 0xFBFF).astype(np.uint16)
        X, pdt, out_dt = bits.view(np.float16), pp.PP_F16, oracle.F16
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F, dtype=pdt,
                  batch_size=B, out_dtype=out_dt, hbm_budget_bytes=-1)
    L.epoch_permute(6, chunk)
    check_epoch(L, bits, dt, N * F, F, H, F, oracle.epoch_order(6, N, chunk), B, out_dt)
    L.close()


def test_dma_and_kernel_paths_agree_with_seek(pp, monkeypatch):
    # the same epoch through the copy-engine path and the zero-copy kernel, resumed mid-epoch
    H, N, F, B, chunk = 4, 6000, 32, 256, 128
    X, hs, rs = hop_tensor(94, H, N, F)
    outs = {}
    for path in ("dma", "kernel"):
        monkeypatch.setenv("PPLOAD_SPILL_PATH", path)
        L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                      batch_size=B, out_dtype=pp.PP_BF16, hbm_budget_bytes=-1)
        L.epoch_permute(8, chunk)
        L.seek(5)
        out = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
        got = []
        while (rows := L.next_batch(out)) >= 0:
            torch.cuda.synchronize()
            got.append(bits_of(out[:rows], oracle.BF16).copy())
        outs[path] = got
        L.close()
    assert len(outs["dma"]) == len(outs["kernel"]) == oracle.num_steps(N, B) - 5
    for a, b in zip(outs["dma"], outs["kernel"]):
        assert np.array_equal(a, b)


def test_epoch_iterator_over_dma_path(pp):
    # the double-buffered iterator (per-buffer events) with host rows moved by the copy engines
    H, N, F, B, chunk = 4, 3000, 32, 128, 128
    X, hs, rs = hop_tensor(95, H, N, F)
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                  batch_size=B, out_dtype=pp.PP_BF16, hbm_budget_bytes=-1)
    order = oracle.epoch_order(6, N, chunk)
    got = [(x.clone(), v.clone()) for x, _, v in L.epoch(6, chunk, depth=2, nodes=True)]
    torch.cuda.synchronize()
    assert len(got) == oracle.num_steps(N, B)
    for t, (x, v) in enumerate(got):
        want, _, wn = oracle.batch(X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, 1, t, 0, oracle.BF16)
        assert np.array_equal(bits_of(x, oracle.BF16), want), t
        assert np.array_equal(v.cpu().numpy(), wn), t
    L.close()
