"""Pins of the oracle's Philox (O4), unit-key layout (O5) and generator words (O11) against an
independent library implementation: cuRAND's device routine curand_Philox4x32_10, run on the B200
(Philox row: "On device, cross-check against the library routine
curand_Philox4x32_10(uint4, uint2)").  tests/native/curand_pin.cu is test infrastructure; it shares
nothing with the product library or the oracle."""
import ctypes
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def curand():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    L = ctypes.CDLL(os.path.join(ROOT, "tests", "native", "libcurand_pin.so"))
    L.cp_philox.restype = ctypes.c_int
    L.cp_philox.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]

    def philox(ctr, key):
        c = np.ascontiguousarray(ctr, dtype=np.uint32)
        k = np.ascontiguousarray(key, dtype=np.uint32)
        out = np.zeros((c.shape[0], 4), dtype=np.uint32)
        rc = L.cp_philox(c.ctypes.data, k.ctypes.data, c.shape[0], out.ctypes.data)
        assert rc == 0, f"cuda error {rc}"
        return out

    return philox


def test_oracle_philox_equals_curand_random_pairs(curand):
    rng = np.random.default_rng(20250413)
    n = 1_000_000
    ctr = rng.integers(0, 1 << 32, (n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 1 << 32, (n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[:4] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [1, 0, 0, 0], [0, 0, 0, 1]]  # edge counters
    key[:4] = [[0, 0], [0xFFFFFFFF] * 2, [0, 1], [1, 0]]
    got = oracle.philox_batch(ctr, key)
    want = curand(ctr, key)
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[0]}: ctr {ctr[bad[0]]} key {key[bad[0]]}"


def test_unit_key_layout_equals_curand(curand):
    # O5: key64(u) = (y0 << 32) | y1 of Philox(ctr = (u_lo, u_hi, 0, 0), key = (seed_lo, seed_hi)).
    # Seeds with both halves nonzero and units >= 2^32, so a swapped or dropped half shows.
    rng = np.random.default_rng(5)
    for seed in (0x299F31D0A4093822, 250413266 | (0xDEADBEEF << 32), 2**64 - 1):
        u = np.concatenate([rng.integers(0, 1 << 62, 20_000, dtype=np.uint64),
                            np.array([0, 1, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, 2**64 - 1], dtype=np.uint64)])
        ctr = np.stack([u & np.uint64(0xFFFFFFFF), u >> np.uint64(32), np.zeros_like(u), np.zeros_like(u)], 1)
        key = np.tile(np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint64), (u.shape[0], 1))
        y = curand(ctr.astype(np.uint32), key.astype(np.uint32))
        want = (y[:, 0].astype(np.uint64) << np.uint64(32)) | y[:, 1].astype(np.uint64)
        assert np.array_equal(oracle.unit_key_at(seed, u), want), hex(seed)
        # the contiguous form used by the permutation agrees with the point form
        assert np.array_equal(oracle.unit_keys(seed, 1000), oracle.unit_key_at(seed, np.arange(1000)))


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.F16])
def test_generator_words_equal_curand(curand, dtype):
    # O11: word (f & 3) of Philox(ctr = (v_lo, v_hi, (k << 16) | (f >> 2), 'PPGF'), key = data_seed),
    # then G / G16 take sign + mantissa bits and a 16-value exponent field from it
    rng = np.random.default_rng(11)
    seed = 2504
    H, F = 4, 768
    v = np.concatenate([rng.integers(0, 244_160_499, 50), np.array([0, (1 << 32) + 3])]).astype(np.int64)
    got = oracle.gen_rows(seed, dtype, H, F, v)  # [rows, H, F] bits
    vv, kk, ff = np.meshgrid(v.astype(np.uint64), np.arange(H, dtype=np.uint64), np.arange(F, dtype=np.uint64),
                             indexing="ij")
    vv, kk, ff = vv.ravel(), kk.ravel(), ff.ravel()
    ctr = np.stack([vv & np.uint64(0xFFFFFFFF), vv >> np.uint64(32), (kk << np.uint64(16)) | (ff >> np.uint64(2)),
                    np.full_like(vv, 0x50504746)], 1).astype(np.uint32)
    key = np.tile(np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint32), (ctr.shape[0], 1))
    y = curand(ctr, key)
    w = y[np.arange(y.shape[0]), (ff & np.uint64(3)).astype(np.int64)].astype(np.uint32)
    if dtype == oracle.F32:
        want = (w & np.uint32(0x807FFFFF)) | ((np.uint32(120) + ((w >> np.uint32(23)) & np.uint32(15))) << np.uint32(23))
    else:
        want = ((w & np.uint32(0x83FF)) | ((np.uint32(8) + ((w >> np.uint32(10)) & np.uint32(15))) << np.uint32(10)))
        want = want.astype(np.uint16)
    assert np.array_equal(got.ravel(), want)
