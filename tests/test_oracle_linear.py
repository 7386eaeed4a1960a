"""Pins of the §8(f)-1 consumer oracle (per-hop linear on a bf16 batch)."""
import numpy as np

import oracle


def test_hop_linear_brute_force_loops():
    rng = np.random.default_rng(0)
    R, H, F, D = 3, 2, 5, 4
    xb = oracle.cast_bf16(rng.standard_normal((R, H, F)).astype(np.float32).view(np.uint32))
    wb = oracle.cast_bf16(rng.standard_normal((H, F, D)).astype(np.float32).view(np.uint32))
    Z, S = oracle.hop_linear(xb, wb)
    for j in range(R):
        for k in range(H):
            for d in range(D):
                acc = 0.0
                acc_abs = 0.0
                for f in range(F):
                    x = float(np.uint32(int(xb[j, k, f]) << 16).view(np.float32))
                    w = float(np.uint32(int(wb[k, f, d]) << 16).view(np.float32))
                    acc += x * w
                    acc_abs += abs(x * w)
                assert abs(Z[j, k, d] - acc) <= 1e-12 * max(1.0, acc_abs)
                assert abs(S[j, k, d] - acc_abs) <= 1e-12 * max(1.0, acc_abs)


def test_hop_linear_identity_and_hop_separation():
    # W_k = c_k * I (exact in bf16): Z[:, k, :] = c_k * X[:, k, :]; hops never mix
    rng = np.random.default_rng(1)
    R, H, F = 4, 3, 8
    xb = oracle.cast_bf16(rng.standard_normal((R, H, F)).astype(np.float32).view(np.uint32))
    W = np.stack([np.eye(F, dtype=np.float32) * c for c in (1.0, -2.0, 0.5)])
    Z, _ = oracle.hop_linear(xb, oracle.cast_bf16(W.view(np.uint32)))
    X = oracle.bf16_bits_to_f64(xb)
    for k, c in enumerate((1.0, -2.0, 0.5)):
        assert np.array_equal(Z[:, k, :], c * X[:, k, :])


def test_hop_linear_binary16_brute_force_loops():
    # the fp16 batch / weights form (fp16 stores, e.g. MAG240M): decoded by IEEE binary16 rules written
    # out here (sign, 5-bit exponent, 10-bit mantissa, subnormals), summed in Python floats
    def half(b):
        b = int(b)
        s, e, m = b >> 15, (b >> 10) & 31, b & 1023
        v = (m / 1024.0) * 2.0 ** -14 if e == 0 else (1 + m / 1024.0) * 2.0 ** (e - 15)
        return -v if s else v

    rng = np.random.default_rng(2)
    R, H, F, D = 3, 2, 6, 3
    xb = oracle.cast_f16(rng.standard_normal((R, H, F)).astype(np.float32).view(np.uint32))
    wb = oracle.cast_f16((rng.standard_normal((H, F, D)) * 1e-4).astype(np.float32).view(np.uint32))  # subnormals
    Z, S = oracle.hop_linear(xb, wb, oracle.F16)
    for j in range(R):
        for k in range(H):
            for d in range(D):
                terms = [half(xb[j, k, f]) * half(wb[k, f, d]) for f in range(F)]
                assert abs(Z[j, k, d] - sum(terms)) <= 1e-15 * max(1e-12, sum(map(abs, terms)))
                assert abs(S[j, k, d] - sum(map(abs, terms))) <= 1e-15 * max(1e-12, sum(map(abs, terms)))
