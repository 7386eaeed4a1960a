"""Seeded synthetic inputs shared by the oracle and the CUDA path in tests.

Holds none of the method's arithmetic: only numpy's seeded generator, shaped like
the paper's workloads (dense hop matrices; labelled-node subsets,
PAPER.md:365).  TB-scale stores are generated in place by pp_fill_synthetic / the
oracle's own generator instead.
"""
import numpy as np


def hop_tensor(seed: int, H: int, N: int, F: int, layout: str = "hop_major", dtype=np.float32):
    """Random hop matrices.  Returns (array, hop_stride, row_stride) in elements.

    fp32 values are drawn from N(0, 1) (bit patterns of every exponent class the
    propagated features have); 16-bit stores get raw random finite bit patterns."""
    rng = np.random.default_rng(seed)
    if dtype == np.float32:
        X = rng.standard_normal((H, N, F)).astype(np.float32)
    else:
        X = rng.integers(0, 1 << 16, (H, N, F), dtype=np.uint64).astype(np.uint16)
        X[(X & 0x7C00) == 0x7C00] &= 0xBFFF  # keep 16-bit values finite
    if layout == "hop_major":
        return np.ascontiguousarray(X), N * F, F
    Xn = np.ascontiguousarray(X.transpose(1, 0, 2))
    return Xn, F, H * F


def integer_hops(seed: int, H: int, N: int, F: int):
    """Integer-valued fp32 features in [-256, 256] (exact in bf16/fp16): column-sum pin."""
    rng = np.random.default_rng(seed)
    return rng.integers(-256, 257, (H, N, F)).astype(np.float32)


def labels(seed: int, N: int, classes: int = 47):
    return np.random.default_rng(seed).integers(0, classes, N).astype(np.int32)


def node_set(seed: int, N_total: int, n: int):
    """A labelled-node subset: n distinct ids, unsorted."""
    rng = np.random.default_rng(seed)
    return rng.choice(N_total, size=n, replace=False).astype(np.int64)


def bit_sweep(n: int, seed: int = 0):
    """fp32 bit patterns for cast checks: every exponent x sign with low-mantissa
    patterns, a strided sweep of the whole space, random patterns."""
    rng = np.random.default_rng(seed)
    low = np.arange(1 << 10, dtype=np.uint32)
    parts = []
    for sign in (0, 1):
        for e in range(256):
            base = np.uint32((sign << 31) | (e << 23))
            parts.append(base | low)
            parts.append(base | (low << np.uint32(13)))
    parts.append(np.arange(0, 1 << 32, 4099, dtype=np.uint64).astype(np.uint32))
    parts.append(rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32))
    return np.concatenate(parts)
