"""O11 pins: the synthetic generators of SURVEY.md §8(d) (values are inputs, not method output)."""
import numpy as np

import oracle


def test_g_values_normal_and_in_range():
    rows = np.arange(0, 5000, 7)
    bits = oracle.gen_rows(2504, oracle.F32, 4, 100, rows).ravel()
    f = bits.view(np.float32)
    a = np.abs(f)
    assert np.isfinite(f).all()
    assert (a >= 2.0 ** -7).all() and (a < 2.0 ** 9).all()
    # all values normal and finite after the bf16 / fp16 casts
    hb = (oracle.cast_bf16(bits).astype(np.uint32) << 16).view(np.float32)
    hf = oracle.cast_f16(bits).view(np.float16).astype(np.float32)
    assert np.isfinite(hb).all() and np.isfinite(hf).all()
    assert (np.abs(hf) >= 2.0 ** -14).all()
    # sign and exponent field roughly uniform (a dropped word would show up here)
    assert abs((f < 0).mean() - 0.5) < 0.01
    ex = (bits >> np.uint32(23)) & np.uint32(0xFF)
    hist = np.bincount(ex - 120, minlength=16)
    assert hist.min() > 0.8 * hist.mean()


def test_g16_values_normal_and_in_range():
    h = oracle.gen_rows(2504, oracle.F16, 4, 768, np.arange(100)).ravel()
    f = h.view(np.float16).astype(np.float32)
    assert np.isfinite(f).all()
    assert (np.abs(f) >= 2.0 ** -7).all() and (np.abs(f) < 2.0 ** 9).all()


def test_g_pure_function_of_coordinates():
    a = oracle.gen_rows(1, oracle.F32, 3, 9, np.array([5, 1000, 7]))
    b = oracle.gen_rows(1, oracle.F32, 3, 9, np.array([7, 5]))
    assert np.array_equal(a[0], b[1]) and np.array_equal(a[2], b[0])
    assert not np.array_equal(a, oracle.gen_rows(2, oracle.F32, 3, 9, np.array([5, 1000, 7])))


def test_graph_generator():
    n, m = 2708, 5429
    src, dst = oracle.gen_graph(2504, n, m)
    assert src.shape[0] == m
    assert (src != dst).all()
    pairs = set(zip(np.minimum(src, dst).tolist(), np.maximum(src, dst).tolist()))
    assert len(pairs) == m
    assert src.min() >= 0 and max(src.max(), dst.max()) < n
