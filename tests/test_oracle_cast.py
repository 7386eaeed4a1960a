"""O10 pins: fp32 -> bf16 / fp16 round-to-nearest-even.

Independent references: hand-derived IEEE special values (tests/golden), numpy's
float16 conversion and torch CPU's bfloat16 conversion over large bit-pattern
sweeps.  The full 2^32 sweep (0 mismatches, NaN excluded) is run by
scripts/verify_cast_exhaustive.py; its result is recorded in DESIGN.md.
"""
import numpy as np
import torch

import oracle
from golden_util import rows


def test_special_values():
    for line in rows("cast_special_values.txt"):
        f32, bf, hf = [int(x, 16) for x in line.split()]
        assert int(oracle.cast_bf16(np.array([f32], np.uint32))[0]) == bf, hex(f32)
        assert int(oracle.cast_f16(np.array([f32], np.uint32))[0]) == hf, hex(f32)


def _sweep_bits():
    # every exponent x sign with a dense set of low mantissa patterns (ties live in the low
    # bits) plus a stride-9973 sweep of the whole space and random patterns
    rng = np.random.default_rng(2504)
    parts = []
    low = np.arange(1 << 14, dtype=np.uint32)
    for sign in (0, 1):
        for e in range(256):
            base = np.uint32((sign << 31) | (e << 23))
            parts.append(base | low)
            parts.append(base | (low << np.uint32(9)))
    parts.append((np.arange(0, 1 << 32, 9973, dtype=np.uint64)).astype(np.uint32))
    parts.append(rng.integers(0, 1 << 32, size=1 << 22, dtype=np.uint64).astype(np.uint32))
    return np.concatenate(parts)


def test_bf16_matches_torch_cpu():
    b = _sweep_bits()
    f = b.view(np.float32)
    nan = np.isnan(f)
    ref = torch.from_numpy(f.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = oracle.cast_bf16(b)
    bad = (got != ref) & ~nan
    assert not bad.any(), hex(int(b[bad][0]))
    assert (got[nan] == 0x7FFF).all()


def test_f16_matches_numpy():
    b = _sweep_bits()
    f = b.view(np.float32)
    nan = np.isnan(f)
    with np.errstate(over="ignore"):
        ref = f.astype(np.float16).view(np.uint16)
    got = oracle.cast_f16(b)
    bad = (got != ref) & ~nan
    assert not bad.any(), hex(int(b[bad][0]))
    assert (got[nan] == 0x7FFF).all()


def test_integers_exact():
    # integer-valued features |x| <= 256 are exact in bf16, fp16 and fp32 (used by the column-sum pin)
    x = np.arange(-256, 257, dtype=np.float32)
    b = x.view(np.uint32)
    assert np.array_equal(oracle.cast_bf16(b).astype(np.uint32) << 16, b)
    assert np.array_equal(oracle.cast_f16(b).view(np.float16).astype(np.float32), x)
