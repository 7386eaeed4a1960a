"""A0 pins: Eq. (2) propagation S = {X, BX, ..., B^K X} with B = D~^-1/2 (I+A) D~^-1/2
(PAPER.md:158-167, 182).  Tolerance: relative Frobenius <= 1e-5."""
import numpy as np
import pytest

import oracle
from golden_util import spec_values


def dense_operator(n, src, dst):
    # independent textbook construction with numpy: A~ = I + A (symmetric, no duplicates)
    A = np.zeros((n, n))
    for a, b in zip(src, dst):
        if a != b:
            A[a, b] = 1.0
            A[b, a] = 1.0
    At = A + np.eye(n)
    d = At.sum(axis=1)
    Dm = np.diag(1.0 / np.sqrt(d))
    return Dm @ At @ Dm


def relfro(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("n,m,K,seed", [(30, 60, 3, 1), (50, 200, 4, 2), (100, 150, 4, 3), (64, 0, 2, 4)])
def test_matches_dense_matrix_power(n, m, K, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    X = rng.standard_normal((n, 7)).astype(np.float32)
    hops = oracle.propagate_graph(n, src, dst, X, K)
    Bd = dense_operator(n, src, dst)
    assert hops[0].tobytes() == X.tobytes()  # hop 0 bit-identical (SPEC.md "hops[0] is bit-identical")
    for k in range(1, K + 1):
        ref = np.linalg.matrix_power(Bd, k) @ X.astype(np.float64)
        assert relfro(hops[k].astype(np.float64), ref) <= 1e-5, k


def test_single_edge_and_spmm_worked_values():
    sv = spec_values()
    rp, ci = oracle.build_csr(2, [0], [1])
    val = oracle.operator_values(2, rp, ci)
    dense = np.zeros((2, 2))
    for i in range(2):
        for p in range(rp[i], rp[i + 1]):
            dense[i, ci[p]] = val[p]
    assert dense.ravel().tolist() == sv["single_edge_operator"]
    y = oracle.spmm(2, rp, ci, val, np.array([[1.0], [0.0]], np.float32))
    assert y.ravel().tolist() == sv["spmm_single_edge"]


def test_path_degrees_and_entry():
    sv = spec_values()
    rp, ci = oracle.build_csr(3, [0, 1], [1, 2])
    assert np.diff(rp).tolist() == sv["path3_degrees"]  # d~ = row length of A~
    val = oracle.operator_values(3, rp, ci)
    p01 = [p for p in range(rp[0], rp[1]) if ci[p] == 1][0]
    assert abs(val[p01] - sv["path3_entry01"][0]) < 1e-15


def test_edgeless_identity():
    X = np.random.default_rng(5).standard_normal((10, 3)).astype(np.float32)
    hops = oracle.propagate_graph(10, [], [], X, 3)
    for k in range(4):
        assert hops[k].tobytes() == X.tobytes()


def test_dedup_loops_and_direction():
    # duplicates, reversed duplicates and self loops collapse to the same operator
    a = oracle.build_csr(4, [0, 1, 2], [1, 2, 3])
    b = oracle.build_csr(4, [1, 0, 0, 2, 3, 2, 2], [0, 1, 1, 1, 2, 2, 3])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("j", [0, 1, 7])
def test_ring_closed_form(j):
    # ring C_n: B = (I + A)/3, x_i = cos(2 pi j i / n) is an eigenvector with eigenvalue (1 + 2 cos(2 pi j / n))/3
    n, K = 1000, 4
    src = np.arange(n)
    dst = (src + 1) % n
    x = np.cos(2 * np.pi * j * np.arange(n) / n).astype(np.float32)[:, None]
    hops = oracle.propagate_graph(n, src, dst, x, K)
    lam = (1 + 2 * np.cos(2 * np.pi * j / n)) / 3
    for k in range(K + 1):
        ref = lam ** k * x.astype(np.float64)
        assert relfro(hops[k].astype(np.float64), ref) <= 1e-5


def test_complete_graph_closed_form():
    # K_n: B = J/n, so every row of X_k (k >= 1) is the column mean of X
    n = 64
    iu = np.triu_indices(n, 1)
    X = np.random.default_rng(6).standard_normal((n, 5)).astype(np.float32)
    hops = oracle.propagate_graph(n, iu[0], iu[1], X, 3)
    mean = X.astype(np.float64).mean(axis=0)
    for k in (1, 2, 3):
        assert relfro(hops[k].astype(np.float64), np.broadcast_to(mean, (n, 5))) <= 1e-5


def test_sqrt_degree_fixed_point_on_tiny_graph():
    # any undirected graph: x = sqrt(d~) satisfies B x = x (config-1 graph, n = 2708)
    n, m = 2708, 5429
    src, dst = oracle.gen_graph(2504, n, m)
    rp, ci = oracle.build_csr(n, src, dst)
    x = np.sqrt(np.diff(rp).astype(np.float64)).astype(np.float32)[:, None]
    hops = oracle.propagate(n, rp, ci, oracle.operator_values(n, rp, ci), x, 3)
    for k in range(4):
        assert relfro(hops[k].astype(np.float64), x.astype(np.float64)) <= 1e-5


def test_symmetric_operator_values():
    src, dst = oracle.gen_graph(9, 200, 700)
    rp, ci = oracle.build_csr(200, src, dst)
    val = oracle.operator_values(200, rp, ci)
    w = {}
    for i in range(200):
        for p in range(rp[i], rp[i + 1]):
            w[(i, int(ci[p]))] = val[p]
    for (i, j), v in w.items():
        assert w[(j, i)] == v
