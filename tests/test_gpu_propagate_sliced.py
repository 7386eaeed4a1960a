"""§8(f)-2: the L2-sliced propagation kernel (k_spmm_sliced, propagate.cu) against the oracle (O1-O3).

A hop first copies X_{k-1} window-major (32-byte windows of 8 features), then runs one pass per
window; one thread per output row sums the window's features over the row's nonzeros in ascending
column order with separately rounded fp64 products and sums, so every hop slot is bit-identical to
oracle.propagate (Eq. (2); operator PAPER.md:182) -- for the hop-major
pp_propagate and for pp_propagate_store (W = 1, spilled rows, exchange copies; sharded stores keep
the row kernels, whose peer reads the sliced form would not shorten).  The kernel is opt-in
(PPLOAD_SPMM=sliced): on B200 it measured slower than the row kernels."""
import numpy as np
import pytest

import oracle
from test_gpu_propagate_store import check_store, graph, make_shards, propagate_all

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def gpu_propagate(pp, rp, ci, X, K):
    n, F = X.shape
    hops = torch.empty((K + 1, n, F), dtype=torch.float32, device="cuda")
    pp.pp_propagate(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(X).cuda(), K, hops)
    torch.cuda.synchronize()
    return hops.cpu().numpy()


@pytest.mark.parametrize("n,m,F,K", [(1, 0, 4, 1), (300, 1500, 12, 3), (2000, 16000, 100, 2), (700, 5000, 256, 2),
                                     (1001, 7000, 8, 3), (500, 4000, 36, 2)])
def test_hop_major_sliced(pp, monkeypatch, n, m, F, K):
    monkeypatch.setenv("PPLOAD_SPMM", "sliced")
    rp, ci = graph(n, m, n + F)
    X = np.random.default_rng(F).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    got = gpu_propagate(pp, rp, ci, X, K)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_hub_row_sliced(pp, monkeypatch):
    # a star: the hub walks n nonzeros (the thread-per-row loop over a long row)
    monkeypatch.setenv("PPLOAD_SPMM", "sliced")
    n, F, K = 3000, 40, 3
    rp, ci = oracle.build_csr(n, np.zeros(n - 1, dtype=np.int64), np.arange(1, n))
    X = np.random.default_rng(3).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    assert np.array_equal(gpu_propagate(pp, rp, ci, X, K).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("window", ["16", "32"])
def test_above_l2_size(pp, monkeypatch, window):
    # n * F * 4 = 80 MB: larger than the L2, several thread blocks per window; both window widths
    monkeypatch.setenv("PPLOAD_SPMM", "sliced")
    monkeypatch.setenv("PPLOAD_SPMM_WINDOW", window)
    n, m, F, K = 200_000, 1_000_000, 100, 2
    rp, ci = graph(n, m, 8)
    X = np.random.default_rng(9).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    assert np.array_equal(gpu_propagate(pp, rp, ci, X, K).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("W", [1, 2, 3])
@pytest.mark.parametrize("F", [4, 100, 132])
def test_store_sliced_sharded(pp, monkeypatch, W, F):
    monkeypatch.setenv("PPLOAD_SPMM", "sliced")
    n, m, K = 1500, 9000, 3
    rp, ci = graph(n, m, F + W)
    X = np.random.default_rng(F).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    Ls = make_shards(pp, monkeypatch, W, X, K + 1, batch_size=64, out_dtype=pp.PP_BF16)
    try:
        propagate_all(Ls, rp, ci, K)
        check_store(Ls, want, K + 1, F)
    finally:
        for L in Ls:
            L.close()


@pytest.mark.parametrize("W", [1, 2])
def test_store_sliced_spill_and_exchange_copy(pp, monkeypatch, W):
    # spilled rows and (W = 2) exchange copies: W = 1 takes the sliced kernel (slot k-1 of spilled
    # records read over UVA by the window copy, slot k written back over UVA); batches afterwards
    # equal the oracle's
    monkeypatch.setenv("PPLOAD_SPMM", "sliced")
    n, m, F, K, B = 2400, 15000, 48, 3, 96
    rp, ci = graph(n, m, 6)
    X = np.random.default_rng(2).standard_normal((n, F)).astype(np.float32)
    want = np.ascontiguousarray(oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K))
    rec = (K + 1) * F * 4
    Ls = make_shards(pp, monkeypatch, W, X, K + 1, batch_size=B, out_dtype=pp.PP_BF16, hbm_budget_bytes=700 * rec)
    try:
        assert all(L.query()["rows_spill"] > 0 and L.query()["exchange_cast"] == (W > 1) for L in Ls)
        propagate_all(Ls, rp, ci, K)
        check_store(Ls, want, K + 1, F)
        order = oracle.epoch_order(3, n, 8)
        for r, L in enumerate(Ls):
            L.epoch_permute(3, 8)
            out = torch.empty((B, K + 1, F), dtype=torch.bfloat16, device="cuda")
            for t in range(oracle.num_steps(n, B, W)):
                rows = L.next_batch(out)
                torch.cuda.synchronize()
                exp, _, _ = oracle.batch(want.view(np.uint32), oracle.F32, n * F, F, K + 1, F, order, B, W, t, r,
                                         oracle.BF16)
                assert np.array_equal(out[:rows].view(torch.int16).cpu().numpy().view(np.uint16), exp), (r, t)
    finally:
        for L in Ls:
            L.close()
