"""Property-based pins of the oracle loader (O5-O10) over random shapes: the laws every epoch must
satisfy whatever (seed, N, chunk, B, W) -- independent of the implementation's arithmetic."""
import numpy as np
import pytest

import oracle

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402


@st.composite
def epoch_args(draw):
    N = draw(st.integers(1, 3000))
    c = draw(st.integers(1, N))
    seed = draw(st.integers(0, 2**64 - 1))
    return seed, N, c


@settings(max_examples=60, deadline=None)
@given(epoch_args())
def test_order_is_a_permutation_of_contiguous_ascending_chunks(args):
    seed, N, c = args
    order = oracle.epoch_order(seed, N, c)
    assert order.shape == (N,)
    assert np.array_equal(np.sort(order), np.arange(N))  # every node exactly once
    # chunk structure: order splits into the U chunks in the permuted unit order,
    # each the contiguous ascending range of its unit
    U = -(-N // c)
    pi = oracle.unit_permutation(seed, U)
    p = 0
    for u in pi:
        lo, hi = u * c, min(u * c + c, N)
        assert np.array_equal(order[p:p + hi - lo], np.arange(lo, hi))
        p += hi - lo
    assert p == N


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 5000), st.integers(1, 700), st.integers(1, 8), st.booleans())
def test_slicing_covers_each_position_once_in_rank_order(N, B, W, drop_last):
    # O9: step t covers positions [tWB, min((t+1)WB, N)) split into W consecutive slices of B
    steps = oracle.num_steps(N, B, W, drop_last)
    covered = []
    for t in range(steps):
        for r in range(W):
            s, e = oracle.batch_range(N, B, W, t, r)
            assert s == min(t * W * B + r * B, N) and e == min(s + B, N) or (s == e)
            covered.extend(range(s, e))
    if drop_last:
        assert covered == list(range(steps * W * B))
    else:
        assert covered == list(range(N))


@settings(max_examples=40, deadline=None)
@given(st.integers(1, 400), st.integers(1, 6), st.integers(1, 40), st.integers(0, 2**32 - 1))
def test_gather_rows_equal_source_rows(N, H, F, seed):
    # O10 with s_in == s_out: every batch row is a bit copy of its source record, for any layout
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 2**32, (H, N, F), dtype=np.uint32)
    rows = rng.integers(0, N, size=min(N, 64))
    got = oracle.gather_cast(X, oracle.F32, N * F, F, H, F, rows, oracle.F32)
    assert np.array_equal(got, X[:, rows, :].transpose(1, 0, 2))
    # node-major layout of the same data gives the same batch
    Xn = np.ascontiguousarray(X.transpose(1, 0, 2))
    got_n = oracle.gather_cast(Xn, oracle.F32, F, H * F, H, F, rows, oracle.F32)
    assert np.array_equal(got, got_n)
