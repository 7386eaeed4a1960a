"""§8(f)-2: the wave-synchronous propagation kernel (k_spmm_wave) against the oracle.

The kernel changes only which rows are in flight together (a wave of R rows per CTA, partial sums in
shared memory, columns swept in C ascending windows); each output row is still the oracle's O3 sum
in ascending column order with separately rounded fp64 products and sums, so every hop must be
bit-identical to oracle.propagate.  PPLOAD_WAVE_ROWS / PPLOAD_WAVE_WINDOWS shrink the waves and
windows so small graphs cover many waves, ragged last waves, rows that saturate their 8 column
slots inside one window, empty windows and the loose CTA sync (PPLOAD_WAVE_LAG)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from test_gpu_propagate import gpu_propagate  # noqa: E402
from test_gpu_propagate_store import check_store, make_shards, propagate_all  # noqa: E402


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def wave_env(monkeypatch, rows, windows, lag=2, variant=0):
    monkeypatch.setenv("PPLOAD_SPMM", "wave")
    monkeypatch.setenv("PPLOAD_WAVE_ROWS", str(rows))
    monkeypatch.setenv("PPLOAD_WAVE_WINDOWS", str(windows))
    monkeypatch.setenv("PPLOAD_WAVE_LAG", str(lag))
    monkeypatch.setenv("PPLOAD_WAVE_VARIANT", str(variant))


def want_hops(rp, ci, X, K):
    n = X.shape[0]
    return oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)


def random_graph(n, m, seed):
    rng = np.random.default_rng(seed)
    return oracle.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m))


@pytest.mark.parametrize("rows,windows", [(1, 1), (3, 7), (16, 32), (64, 4), (1 << 20, 32)])
@pytest.mark.parametrize("n,m,F,K", [(1, 0, 4, 2), (300, 1500, 8, 3), (2000, 12000, 100, 2), (777, 9000, 128, 1)])
def test_hop_major_bit_exact(pp, monkeypatch, rows, windows, n, m, F, K):
    wave_env(monkeypatch, rows, windows)
    rp, ci = random_graph(n, m, n + m + F)
    X = np.random.default_rng(F).standard_normal((n, F)).astype(np.float32)
    got = gpu_propagate(pp, rp, ci, X, K)
    assert np.array_equal(got.view(np.uint32), want_hops(rp, ci, X, K).view(np.uint32))


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("lag", [0, 1, 2, 5])
def test_kernel_variants_and_sync(pp, monkeypatch, variant, lag):
    # 1024 x 4 / 512 x 4 / 512 x 8 (threads x rows in flight per warp); lag 0 = no window counter
    wave_env(monkeypatch, 5, 9, lag=lag, variant=variant)
    rp, ci = random_graph(5000, 60000, 11)
    X = np.random.default_rng(12).standard_normal((5000, 100)).astype(np.float32)
    got = gpu_propagate(pp, rp, ci, X, 2)
    assert np.array_equal(got.view(np.uint32), want_hops(rp, ci, X, 2).view(np.uint32))


@pytest.mark.parametrize("windows", [1, 2, 5])
def test_hub_rows_saturate_their_slots(pp, monkeypatch, windows):
    # a star plus a clique: the hub and the clique rows have hundreds of neighbours inside one
    # window, i.e. many rounds of 8 slots, in a group whose other rows finish after one round
    n, F, K = 1500, 64, 3
    src = np.concatenate([np.zeros(n - 1, np.int64), np.repeat(np.arange(1, 40), 39)])
    dst = np.concatenate([np.arange(1, n), np.tile(np.arange(1, 40), 39)])
    rp, ci = oracle.build_csr(n, src, dst)
    wave_env(monkeypatch, 6, windows)
    X = np.random.default_rng(3).standard_normal((n, F)).astype(np.float32)
    got = gpu_propagate(pp, rp, ci, X, K)
    assert np.array_equal(got.view(np.uint32), want_hops(rp, ci, X, K).view(np.uint32))


def test_at_scale_fixed_point_and_sampled_rows(pp, monkeypatch):
    # one full-size wave: the sqrt(d~) fixed point is independent of the oracle, and a sample of
    # rows is compared with the per-row O3 definition written out
    wave_env(monkeypatch, 1 << 20, 32)
    n, m = 300_000, 3_000_000
    rng = np.random.default_rng(4)
    rp, ci = oracle.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m))
    x = np.sqrt(np.diff(rp).astype(np.float64)).astype(np.float32)[:, None].repeat(4, 1)
    x[:, 1:] = rng.standard_normal((n, 3)).astype(np.float32)
    got = gpu_propagate(pp, rp, ci, x, 2)
    for k in range(3):
        err = np.linalg.norm(got[k][:, 0].astype(np.float64) - x[:, 0]) / np.linalg.norm(x[:, 0])
        assert err <= 1e-6, (k, err)
    val = oracle.operator_values(n, rp, ci)
    rows = rng.choice(n, 200, replace=False)
    for i in rows:  # O3 for one row: ascending columns, separately rounded fp64 products and sums
        for f in range(4):
            acc = np.float64(0.0)
            for p in range(rp[i], rp[i + 1]):
                acc = np.float64(acc + np.float64(val[p] * np.float64(got[0][ci[p], f])))
            assert np.float32(acc).view(np.uint32) == got[1][i, f].view(np.uint32), (i, f)


@pytest.mark.parametrize("rows,windows", [(2, 3), (32, 32)])
@pytest.mark.parametrize("n,m,F,K", [(1, 0, 4, 1), (1000, 9000, 100, 3), (700, 5000, 128, 2)])
def test_store_single_rank(pp, monkeypatch, rows, windows, n, m, F, K):
    wave_env(monkeypatch, rows, windows)
    rp, ci = random_graph(n, m, n + F)
    X = np.random.default_rng(n).standard_normal((n, F)).astype(np.float32)
    Ls = make_shards(pp, monkeypatch, 1, X, K + 1, batch_size=128, out_dtype=pp.PP_BF16)
    propagate_all(Ls, rp, ci, K)
    check_store(Ls, want_hops(rp, ci, X, K), K + 1, F)
    for L in Ls:
        L.close()


def test_wave_and_row_kernels_agree_on_products_degree_mix(pp, monkeypatch):
    # ER graph with the products mean degree (~51 per row) at 1/10 of the rows: wave vs row kernel
    n = 244_903
    rp, ci = random_graph(n, n * 25, 7)
    X = np.random.default_rng(8).standard_normal((n, 100)).astype(np.float32)
    monkeypatch.setenv("PPLOAD_SPMM", "rows")
    ref = gpu_propagate(pp, rp, ci, X, 2)
    wave_env(monkeypatch, 1 << 20, 32)
    got = gpu_propagate(pp, rp, ci, X, 2)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


# ---- k_spmm_rows_cp: the row kernel with neighbour rows staged in shared memory by cp.async ----------
def cp_env(monkeypatch, variant=0):
    monkeypatch.setenv("PPLOAD_SPMM", "cp")
    monkeypatch.setenv("PPLOAD_CP_VARIANT", str(variant))


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("n,m,F,K", [(1, 0, 4, 2), (300, 1500, 8, 3), (2000, 12000, 100, 2), (777, 9000, 128, 1),
                                     (5000, 150000, 64, 2)])
def test_cp_hop_major_bit_exact(pp, monkeypatch, variant, n, m, F, K):
    # cp.async 16 B per lane: 1024 threads x 16 / 8 / 12 slots, 512 x 32; one cp.async.bulk per row:
    # 1024 x 12 / 8, 512 x 24, 256 x 48 -- rings that wrap inside rows and across row boundaries
    cp_env(monkeypatch, variant)
    rp, ci = random_graph(n, m, n + m + F)
    X = np.random.default_rng(F).standard_normal((n, F)).astype(np.float32)
    got = gpu_propagate(pp, rp, ci, X, K)
    assert np.array_equal(got.view(np.uint32), want_hops(rp, ci, X, K).view(np.uint32))


@pytest.mark.parametrize("variant", [0, 4])
def test_cp_hub_rows_and_empty_rows(pp, monkeypatch, variant):
    # a star (the hub row has n entries: its stream wraps the ring many times) plus rows with no
    # nonzeros at all (a CSR the API accepts as long as nnz >= n): those rows must come out zero
    n, F, K = 1500, 100, 2
    leaves = np.setdiff1d(np.arange(1, n), [5, 6, 700])  # 5, 6, 700: only their diagonal, then none
    rp, ci = oracle.build_csr(n, np.zeros(leaves.size, np.int64), leaves)
    keep = np.ones(ci.shape[0], bool)
    for i in (5, 6, 700):  # drop every entry of three leaf rows
        keep[rp[i]:rp[i + 1]] = False
    lens = np.diff(rp).copy()
    lens[[5, 6, 700]] = 0
    rp2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci2 = ci[keep]
    X = np.random.default_rng(3).standard_normal((n, F)).astype(np.float32)
    val = oracle.operator_values(n, rp2, ci2)
    want = oracle.propagate(n, rp2, ci2, val, X, K)
    cp_env(monkeypatch, variant)
    got = gpu_propagate(pp, rp2, ci2, X, K)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert not got[1][[5, 6, 700]].any()


@pytest.mark.parametrize("variant", [0, 4])
@pytest.mark.parametrize("n,m,F,K", [(1, 0, 4, 1), (1000, 9000, 100, 3), (700, 5000, 128, 2)])
def test_cp_store_single_rank(pp, monkeypatch, variant, n, m, F, K):
    cp_env(monkeypatch, variant)
    rp, ci = random_graph(n, m, n + F)
    X = np.random.default_rng(n).standard_normal((n, F)).astype(np.float32)
    Ls = make_shards(pp, monkeypatch, 1, X, K + 1, batch_size=128, out_dtype=pp.PP_BF16)
    propagate_all(Ls, rp, ci, K)
    check_store(Ls, want_hops(rp, ci, X, K), K + 1, F)
    for L in Ls:
        L.close()


def test_cp_and_row_kernels_agree_on_products_degree_mix(pp, monkeypatch):
    n = 244_903
    rp, ci = random_graph(n, n * 25, 7)
    X = np.random.default_rng(8).standard_normal((n, 100)).astype(np.float32)
    monkeypatch.setenv("PPLOAD_SPMM", "rows")
    ref = gpu_propagate(pp, rp, ci, X, 2)
    for variant in (0, 4):
        cp_env(monkeypatch, variant)
        got = gpu_propagate(pp, rp, ci, X, 2)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), variant
