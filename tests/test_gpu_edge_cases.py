"""Degenerate shapes through every assembly path (gather kernels, copy-engine DMA, storage tier,
compact store): a single node, a batch larger than the epoch, drop_last, chunk = N.  Batches must
equal the oracle's (O7-O10) and epochs must end exactly when the oracle's do."""
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


def make(pp, path, tmp_path, X, N, H, F, B, **kw):
    common = dict(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16, **kw)
    if path == "files":
        paths = []
        for k in range(H):
            p = tmp_path / f"h{k}.bin"
            np.ascontiguousarray(X[k]).tofile(p)
            paths.append(str(p))
        return pp.Loader(files=paths, **common)
    extra = dict(hbm_budget_bytes=-1) if path == "dma" else {}
    return pp.Loader(data=X, hop_stride=N * F, row_stride=F, **common, **extra)


def run(L, X, N, H, F, B, order, drop_last=False):
    steps = oracle.num_steps(order.shape[0], B, 1, drop_last)
    out = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
    nodes = torch.empty(B, dtype=torch.int64, device="cuda")
    t = 0
    while (rows := L.next_batch(out, None, nodes)) >= 0:
        torch.cuda.synchronize()
        want, _, wn = oracle.batch(X.view(np.uint32), oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
        assert rows == want.shape[0], t
        assert np.array_equal(out[:rows].cpu().view(torch.int16).numpy().view(np.uint16), want), t
        assert np.array_equal(nodes[:rows].cpu().numpy(), wn), t
        t += 1
    assert t == steps


PATHS = ["gather", "dma", "files"]


@pytest.mark.parametrize("path", PATHS)
def test_single_node(pp, tmp_path, monkeypatch, path):
    if path == "dma":
        monkeypatch.setenv("PPLOAD_SPILL_PATH", "dma")
    H, N, F, B = 2, 1, 8, 4
    X = np.random.default_rng(1).standard_normal((H, N, F)).astype(np.float32)
    L = make(pp, path, tmp_path, X, N, H, F, B)
    L.epoch_permute(3, 1)
    run(L, X, N, H, F, B, oracle.epoch_order(3, N, 1))
    L.close()


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("chunk", [1, 7, 50])
def test_batch_larger_than_epoch(pp, tmp_path, monkeypatch, path, chunk):
    if path == "dma":
        monkeypatch.setenv("PPLOAD_SPILL_PATH", "dma")
    H, N, F, B = 3, 50, 16, 64
    X = np.random.default_rng(chunk).standard_normal((H, N, F)).astype(np.float32)
    L = make(pp, path, tmp_path, X, N, H, F, B)
    L.epoch_permute(5, chunk)
    run(L, X, N, H, F, B, oracle.epoch_order(5, N, chunk))
    L.close()


@pytest.mark.parametrize("path", PATHS)
def test_drop_last_and_chunk_n(pp, tmp_path, monkeypatch, path):
    if path == "dma":
        monkeypatch.setenv("PPLOAD_SPILL_PATH", "dma")
    H, N, F, B = 2, 1001, 24, 100
    X = np.random.default_rng(9).standard_normal((H, N, F)).astype(np.float32)
    L = make(pp, path, tmp_path, X, N, H, F, B, drop_last=True)
    assert L.query()["steps_per_epoch"] == N // B
    for chunk in (N, 64):
        L.epoch_permute(11, chunk)
        run(L, X, N, H, F, B, oracle.epoch_order(11, N, chunk), drop_last=True)
    L.close()


def test_compact_store_single_member_node_set(pp):
    H, N, F, B = 2, 500, 8, 16
    X = np.random.default_rng(4).standard_normal((H, N, F)).astype(np.float32)
    S = np.array([321], dtype=np.int64)
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F, dtype=pp.PP_F32,
                  node_set=S, batch_size=B, out_dtype=pp.PP_BF16, store_set_only=True)
    L.epoch_permute(1, 1)
    run(L, X, N, H, F, B, oracle.epoch_order(1, 1, 1, node_set=S))
    L.close()
