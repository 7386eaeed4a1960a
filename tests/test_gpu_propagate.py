"""§8(f)-2: GPU pre-propagation (pp_propagate) against the oracle's CSR SpMM (O1-O3).

The GPU follows the oracle's arithmetic definition (fp64 weights 1/sqrt(d_i d_j), fp64 row
sums in ascending column order with separately rounded products and sums, one RNE rounding
to fp32), so every hop must be bit-identical -- stronger than the 1e-5 relative Frobenius
tolerance SPEC.md:84 asks of propagation."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    import paper_2504_13266_b200 as pp

    return pp


def gpu_propagate(pp, rp, ci, X, K):
    n, F = X.shape
    hops = torch.empty((K + 1, n, F), dtype=torch.float32, device="cuda")
    pp.pp_propagate(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(X).cuda(), K, hops)
    torch.cuda.synchronize()
    return hops.cpu().numpy()


def test_config1_bit_exact(pp):
    n, m, F, K = 2708, 5429, 128, 3
    src, dst = oracle.gen_graph(2504, n, m)
    rp, ci = oracle.build_csr(n, src, dst)
    X = oracle.gen_rows(2504, oracle.F32, 1, F, np.arange(n)).reshape(n, F).view(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    got = gpu_propagate(pp, rp, ci, X, K)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("n,m,F,K", [(1, 0, 5, 2), (50, 200, 1, 1), (300, 1500, 7, 4), (1000, 9000, 33, 2),
                                     (2000, 4000, 100, 3), (500, 20000, 200, 2), (777, 3000, 256, 1),
                                     (100, 300, 64, 0)])
def test_random_graphs_bit_exact(pp, n, m, F, K):
    rng = np.random.default_rng(n + m + F)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    rp, ci = oracle.build_csr(n, src, dst)
    X = rng.standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    got = gpu_propagate(pp, rp, ci, X, K)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_hub_rows_longer_than_a_warp(pp):
    # a star graph: the hub's row has n entries (> 32: several shuffle rounds), leaves have 2
    n, F, K = 1500, 40, 3
    src = np.zeros(n - 1, dtype=np.int64)
    dst = np.arange(1, n)
    rp, ci = oracle.build_csr(n, src, dst)
    X = np.random.default_rng(3).standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, K)
    got = gpu_propagate(pp, rp, ci, X, K)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_sqrt_degree_fixed_point_at_scale(pp):
    # independent of the oracle: x = sqrt(d~) is a fixed point of B on any undirected graph
    n, m = 200_000, 1_000_000
    rng = np.random.default_rng(4)
    rp, ci = oracle.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m))
    x = np.sqrt(np.diff(rp).astype(np.float64)).astype(np.float32)[:, None]
    got = gpu_propagate(pp, rp, ci, x, 3)
    for k in range(4):
        err = np.linalg.norm(got[k].astype(np.float64) - x) / np.linalg.norm(x)
        assert err <= 1e-6, (k, err)


def test_invalid_arguments(pp):
    rp = torch.zeros(3, dtype=torch.int64, device="cuda")
    ci = torch.zeros(1, dtype=torch.int64, device="cuda")
    X = torch.zeros((2, 300), dtype=torch.float32, device="cuda")
    hops = torch.zeros((2, 2, 300), dtype=torch.float32, device="cuda")
    with pytest.raises(pp.PPError) as ei:
        pp.pp_propagate(rp, ci, X, 1, hops)  # F = 300 > 256
    assert ei.value.status == pp.PP_ERR_INVALID
    X = torch.zeros((2, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(pp.PPError) as ei:
        pp.pp_propagate(rp, ci, X, 1, hops)  # row_ptr[n] = 0 < n: no diagonal
    assert ei.value.status == pp.PP_ERR_INVALID


@pytest.mark.parametrize("F", [4, 100, 132, 256])
def test_scalar_and_vector_kernels_agree(pp, monkeypatch, F):
    # F % 4 == 0 takes the 16-byte-per-lane kernel; PPLOAD_SPMM=scalar forces the per-element one.
    # Both sum in ascending column order, so both equal the oracle bit for bit.
    n, m = 900, 7000
    rng = np.random.default_rng(F)
    rp, ci = oracle.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m))
    X = rng.standard_normal((n, F)).astype(np.float32)
    want = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), X, 2)
    vec = gpu_propagate(pp, rp, ci, X, 2)
    monkeypatch.setenv("PPLOAD_SPMM", "scalar")
    sca = gpu_propagate(pp, rp, ci, X, 2)
    assert np.array_equal(vec.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(sca.view(np.uint32), want.view(np.uint32))
