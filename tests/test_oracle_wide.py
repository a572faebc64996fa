"""Pins of the wide-ACU oracle (NEXT-2, b = 10 and 12 with int16 codes): the exact table is the
integer matmul, the bincount reformulation, the row-sum probe, and the quantizer's round trip.
CPU only."""
import numpy as np
import pytest

import datagen
import oracle


@pytest.mark.parametrize("bits", [10, 12])
def test_wide_exact_lut_is_integer_matmul(bits):
    A = datagen.random_int16(1, (7, 33), bits)
    W = datagen.random_int16(2, (5, 33), bits)
    C = oracle.lut_gemm16(A, W, datagen.lut_exact(bits), bits)
    np.testing.assert_array_equal(C, A.astype(np.int64) @ W.astype(np.int64).T)


@pytest.mark.parametrize("bits", [10, 12])
def test_wide_bincount_and_probe(bits):
    T = datagen.lut_randerr(bits, 9, 1)
    A = datagen.random_int16(3, (3, 40), bits)
    W = datagen.random_int16(4, (2, 40), bits)
    C = oracle.lut_gemm16(A, W, T, bits)
    mask = (1 << bits) - 1
    for m in range(3):
        for n in range(2):
            idx = ((A[m].astype(np.int64) & mask) << bits) | (W[n].astype(np.int64) & mask)
            cnt = np.bincount(idx, minlength=1 << (2 * bits))
            assert C[m, n] == int((cnt * T.astype(np.int64)).sum())
    # row-sum probe: T[i][j] = sx(i) gives sum_k a[m][k] (orientation + sign extension)
    sx = datagen.signed_values(bits)
    Tp = np.repeat(sx, 1 << bits).astype(np.int32)
    Cp = oracle.lut_gemm16(A, W, Tp, bits)
    np.testing.assert_array_equal(Cp, np.repeat(A.astype(np.int64).sum(1, keepdims=True), 2, 1))


def test_wide_quantizer_roundtrip():
    rng = np.random.default_rng(5)
    x = rng.standard_normal(5000).astype(np.float32)
    s = oracle.scale(oracle.amax(x), 12)
    q = oracle.quantize16(x, s, 12)
    assert np.abs(q).max() == 2047
    assert np.max(np.abs(q.astype(np.float64) * float(s) - x)) <= float(s) / 2 * (1 + 1e-6)
    # at b <= 8 it is the int8 quantizer
    np.testing.assert_array_equal(oracle.quantize16(x, oracle.scale(oracle.amax(x), 8), 8),
                                  oracle.quantize(x, oracle.scale(oracle.amax(x), 8), 8))
