"""O9 pins: batch slicing and exactly-once coverage."""
import numpy as np
import pytest

import oracle
from golden_util import spec_values


def test_spec_batch_sizes():
    want = [int(x) for x in spec_values()["rr_batch_sizes"]]
    N, B = 5, 2
    sizes = []
    for t in range(oracle.num_steps(N, B)):
        s, e = oracle.batch_range(N, B, 1, t, 0)
        sizes.append(e - s)
    assert sizes == want


@pytest.mark.parametrize("N,B,W", [(5, 2, 1), (100, 8, 3), (8192 * 3 + 17, 8192, 2), (64, 8, 8), (7, 8, 4)])
def test_exactly_once_over_steps_and_ranks(N, B, W):
    order = oracle.epoch_order(1, N, 1)
    seen = np.zeros(N, dtype=np.int64)
    for t in range(oracle.num_steps(N, B, W)):
        for r in range(W):
            s, e = oracle.batch_range(N, B, W, t, r)
            assert 0 <= e - s <= B
            np.add.at(seen, order[s:e], 1)
    assert (seen == 1).all()


@pytest.mark.parametrize("W", [2, 4, 8])
def test_w_independence(W):
    # concatenation over ranks of step t == the W*B positions of that step with W = 1
    N, B = 1000, 16
    for t in range(oracle.num_steps(N, B, W)):
        cat = []
        for r in range(W):
            s, e = oracle.batch_range(N, B, W, t, r)
            cat.extend(range(s, e))
        s1, e1 = oracle.batch_range(N, W * B, 1, t, 0)
        assert cat == list(range(s1, e1))


def test_drop_last():
    assert oracle.num_steps(10, 3, 1, drop_last=True) == 3
    assert oracle.num_steps(10, 3, 1, drop_last=False) == 4
    assert oracle.num_steps(2449029, 8192) == 299
    s, e = oracle.batch_range(2449029, 8192, 1, 298, 0)
    assert e - s == 7813  # last batch has 7,813 rows
