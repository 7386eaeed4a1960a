"""Every permutation kernel path against the oracle (O5-O7), forced where it would not be chosen:
one-CTA bitonic sort (U <= 4096), two-level radix (4096 < U <= 2^22) including its oversize
level-2 fallback, and the global bucket sort (U > 2^22, or forced with the bucket-bits knob)."""
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


@pytest.mark.parametrize("two_level", [0, 1])
@pytest.mark.parametrize("N,chunk", [(4097, 1), (8192, 1), (50_000, 1), (123_457, 2), (1 << 22, 1),
                                     ((1 << 22) + 1, 1), (9_000_001, 2)])
def test_two_level_and_bucket_boundaries(pp, monkeypatch, two_level, N, chunk):
    if two_level:
        monkeypatch.setenv("PPLOAD_PERMUTE", "two_level")
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=64, out_dtype=pp.PP_BF16,
                   hbm_budget_bytes=1 << 20) as L:
        for seed in (3, 250413266):
            L.epoch_permute(seed, chunk)
            assert np.array_equal(L.get_order(), oracle.epoch_order(seed, N, chunk)), (N, chunk, seed)


@pytest.mark.parametrize("cap", [1, 64, 600])
def test_two_level_oversize_fallback(pp, monkeypatch, cap):
    monkeypatch.setenv("PPLOAD_PERMUTE", "two_level")
    monkeypatch.setenv("PPLOAD_DEBUG_L2CAP", str(cap))
    N = 200_003
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=64, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(11, 1)
        assert np.array_equal(L.get_order(), oracle.epoch_order(11, N, 1))


def test_prefetch_with_two_level(pp, monkeypatch):
    monkeypatch.setenv("PPLOAD_PERMUTE", "two_level")
    N = 300_001
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=1000, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(1, 1)
        for e in range(2, 6):
            L.epoch_prefetch(e, 1)
            L.epoch_permute(e, 1)
            assert np.array_equal(L.get_order(), oracle.epoch_order(e, N, 1))
