"""O10 pins: batch assembly."""
import numpy as np
import pytest

import oracle
from golden_util import spec_values


def test_spec_ids_2_0():
    X = np.array([[0], [1], [2]], np.float32).view(np.uint32)
    out = oracle.gather_cast(X, oracle.F32, 3, 1, 1, 1, np.array([2, 0]), oracle.F32)
    assert out.view(np.float32).ravel().tolist() == spec_values()["gather_ids_20"]


def test_identity_order_is_prefix():
    rng = np.random.default_rng(0)
    H, N, F = 3, 50, 5
    X = rng.standard_normal((H, N, F)).astype(np.float32).view(np.uint32)
    order = oracle.epoch_order(1, N, N)  # one chunk -> identity
    out = oracle.gather_cast(X, oracle.F32, N * F, F, H, F, order[:20], oracle.F32)
    assert np.array_equal(out, X[:, :20, :].transpose(1, 0, 2))


@pytest.mark.parametrize("out_dtype", [oracle.F32, oracle.BF16, oracle.F16])
def test_rows_equal_source_rows_any_layout(out_dtype):
    # per-row copy oracle: numpy fancy indexing + the oracle cast, hop-major and node-major
    rng = np.random.default_rng(1)
    H, N, F = 4, 300, 12
    X = rng.standard_normal((H, N, F)).astype(np.float32)
    rows = rng.integers(0, N, 97)
    hm = X.view(np.uint32)
    nm = np.ascontiguousarray(X.transpose(1, 0, 2)).view(np.uint32)
    a = oracle.gather_cast(hm, oracle.F32, N * F, F, H, F, rows, out_dtype)
    b = oracle.gather_cast(nm, oracle.F32, F, H * F, H, F, rows, out_dtype)
    assert np.array_equal(a, b)
    ref = nm[rows]
    if out_dtype == oracle.F32:
        assert np.array_equal(a, ref)
    elif out_dtype == oracle.BF16:
        assert np.array_equal(a, oracle.cast_bf16(ref))
    else:
        assert np.array_equal(a, oracle.cast_f16(ref))
    for j, v in enumerate(rows):  # memcmp per row
        assert a[j].tobytes() == (ref[j] if out_dtype == oracle.F32 else a[j]).tobytes()


def test_f16_store_copy():
    rng = np.random.default_rng(2)
    X = rng.integers(0, 1 << 16, (2, 40, 6), dtype=np.uint64).astype(np.uint16)
    rows = np.array([39, 0, 5, 5])
    out = oracle.gather_cast(X, oracle.F16, 40 * 6, 6, 2, 6, rows, oracle.F16)
    assert np.array_equal(out, X[:, rows, :].transpose(1, 0, 2))
    with pytest.raises(ValueError):
        oracle.gather_cast(X, oracle.F16, 240, 6, 2, 6, rows, oracle.BF16)


@pytest.mark.parametrize("c", [1, 64, 256])
def test_epoch_column_sums_and_exactly_once(c):
    # integer-valued features: sum over all batches of out[., k, f] == sum_v X_k[v, f] exactly
    rng = np.random.default_rng(3)
    H, N, F, B = 4, 2708, 16, 256
    Xi = rng.integers(-256, 257, (H, N, F))
    X = Xi.astype(np.float32).view(np.uint32)
    order = oracle.epoch_order(250413266, N, c)
    total = np.zeros((H, F), dtype=np.int64)
    nodes = []
    for t in range(oracle.num_steps(N, B)):
        feat, _, rows = oracle.batch(X, oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
        vals = (feat.astype(np.uint32) << 16).view(np.float32)
        total += vals.astype(np.int64).sum(axis=0)
        nodes.append(rows)
    assert np.array_equal(total, Xi.sum(axis=1))
    assert np.array_equal(np.sort(np.concatenate(nodes)), np.arange(N))


def test_labels():
    lab = np.arange(100, dtype=np.int32) * 3
    rows = np.array([5, 99, 0])
    assert oracle.gather_labels(lab, rows).tolist() == [15, 297, 0]
