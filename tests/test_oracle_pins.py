"""Pins for the CPU oracle (oracle/): checks against what the paper and mathematics fix,
never against the oracle's own formula retyped.  CPU only."""
import itertools
import math
import os

import numpy as np
import pytest
import torch

import datagen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                rows.append(line.split())
    return rows


# ----------------------------------------------------------------------------------------
# ACU tables (inputs) -- worked examples
# ----------------------------------------------------------------------------------------

def _lut_lookup(T, bits, a, w):
    ua, uw = a & ((1 << bits) - 1), w & ((1 << bits) - 1)
    return int(T[(ua << bits) | uw])


def test_lut_golden_examples():
    rows = _golden("lut_examples.txt")
    assert len(rows) >= 5
    for name, bits, a, w, exp in rows:
        bits, a, w, exp = int(bits), int(a), int(w), int(exp)
        T = datagen.lut_exact(bits) if name == "exact" else datagen.lut_trunc4()
        assert _lut_lookup(T, bits, a, w) == exp, (name, a, w)


def test_lut_builders_ranges():
    ex = datagen.lut_exact(8).astype(np.int64)
    re = datagen.lut_randerr(8, 0, 2).astype(np.int64)
    tr = datagen.lut_trunc4().astype(np.int64)
    assert (re - ex).min() >= -64 and (re - ex).max() <= 64         # BJ:c0 error in [-64,64]
    assert (re - ex).min() == -64 and (re - ex).max() == 64
    assert (tr - ex).min() >= -15 and (tr - ex).max() <= 0           # A10: floor to 16
    assert (tr % 16 == 0).all()
    for b in (4, 6, 8):
        e = datagen.lut_randerr(b, 4, 10 + b).astype(np.int64) - datagen.lut_exact(b)
        assert e.min() >= -(1 << (b - 2)) and e.max() <= (1 << (b - 2))


# ----------------------------------------------------------------------------------------
# LUT-GEMM (O5): closed form, probes, reformulation, brute force
# ----------------------------------------------------------------------------------------

@pytest.mark.parametrize("M,N,K,bits", [(64, 64, 256, 8), (7, 13, 1, 8), (33, 5, 147, 8),
                                         (17, 31, 100, 4), (3, 2, 9, 6), (1, 1, 1, 2)])
def test_gemm_exact_lut_is_integer_matmul(M, N, K, bits):
    """Exact multiplier => the plain integer matmul (numpy int64), BJ:ns pin."""
    A = datagen.random_int8(1 + M, (M, K), bits)
    W = datagen.random_int8(2 + N, (N, K), bits)
    C = oracle.lut_gemm(A, W, datagen.lut_exact(bits), bits)
    ref = A.astype(np.int64) @ W.astype(np.int64).T
    np.testing.assert_array_equal(C, ref)


def test_gemm_config0_exact_equals_int_mm():
    c = datagen.config0()
    C = oracle.lut_gemm(c.A, c.W, datagen.lut_exact(8), 8)
    np.testing.assert_array_equal(C, c.A.astype(np.int64) @ c.W.astype(np.int64).T)


def test_gemm_probes_orientation():
    """Indicator / row-sum / column-sum tables (SURVEY §8(c) pin (ii)): catch a transposed
    table, a swapped operand or a missing sign extension."""
    bits = 4
    rng = np.random.default_rng(5)
    A = datagen.random_int8(11, (9, 37), bits)
    W = datagen.random_int8(12, (6, 37), bits)
    vals = datagen.signed_values(bits)
    n = 1 << bits
    # T[i][j] = sx(i): sum_k a[m,k]
    T = np.repeat(vals, n).astype(np.int32)
    C = oracle.lut_gemm(A, W, T, bits)
    np.testing.assert_array_equal(C, np.repeat(A.astype(np.int64).sum(1, keepdims=True), 6, 1))
    # T[i][j] = sx(j): sum_k w[n,k]
    T = np.tile(vals, n).astype(np.int32)
    C = oracle.lut_gemm(A, W, T, bits)
    np.testing.assert_array_equal(C, np.repeat(W.astype(np.int64).sum(1)[None, :], 9, 0))
    # indicator delta(i0, j0): counts of k with a = sx(i0), w = sx(j0)
    for i0, j0 in [(0, 0), (3, 12), (12, 3), (8, 7)]:
        T = np.zeros(n * n, np.int32)
        T[(i0 << bits) | j0] = 1
        C = oracle.lut_gemm(A, W, T, bits)
        cnt = ((A[:, None, :] == vals[i0]) & (W[None, :, :] == vals[j0])).sum(-1)
        np.testing.assert_array_equal(C, cnt)


def test_gemm_bincount_reformulation():
    """acc[m,n] = sum_{i,j} cnt_mn(i,j) T[i][j] with one-hot counts (pin (iii))."""
    bits = 4
    n = 1 << bits
    A = datagen.random_int8(21, (10, 50), bits)
    W = datagen.random_int8(22, (7, 50), bits)
    T = datagen.random_lut(23, bits)
    oa = np.eye(n, dtype=np.int64)[A.astype(np.int64) & (n - 1)]   # [M,K,n]
    ow = np.eye(n, dtype=np.int64)[W.astype(np.int64) & (n - 1)]   # [N,K,n]
    cnt = np.einsum("mki,nkj->mnij", oa, ow)
    ref = np.einsum("mnij,ij->mn", cnt, T.reshape(n, n).astype(np.int64))
    np.testing.assert_array_equal(oracle.lut_gemm(A, W, T, bits), ref)


def test_gemm_brute_force_b2():
    """b = 2: every operand assignment of tiny shapes against an ACU given as a Python
    function of the SIGNED operands (pin (iv)); the table is built from the function with
    the (ua << b) | uw encoding, so an encoding or orientation bug fails here."""
    bits = 2
    rng = np.random.default_rng(7)
    vals = [-2, -1, 0, 1]
    acu = {(a, w): int(rng.integers(-50, 50)) for a in vals for w in vals}
    T = np.zeros(16, np.int32)
    for (a, w), v in acu.items():
        T[((a & 3) << 2) | (w & 3)] = v
    for (M, K, N) in [(1, 3, 1), (2, 2, 1)]:
        for assign in itertools.product(vals, repeat=M * K + N * K):
            A = np.array(assign[:M * K], np.int8).reshape(M, K)
            W = np.array(assign[M * K:], np.int8).reshape(N, K)
            C = oracle.lut_gemm(A, W, T, bits)
            for m in range(M):
                for nn in range(N):
                    assert C[m, nn] == sum(acu[(int(A[m, k]), int(W[nn, k]))] for k in range(K))


def test_gemm_overflow_detected():
    A = np.full((1, 140000), -128, np.int8)
    W = np.full((1, 140000), -128, np.int8)
    with pytest.raises(OverflowError):
        oracle.lut_gemm(A, W, datagen.lut_exact(8), 8)


# ----------------------------------------------------------------------------------------
# conv (O6)
# ----------------------------------------------------------------------------------------

CONV_CASES = [
    # N, C, H, W, K, R, S, stride, pad, groups
    (2, 3, 9, 11, 4, 3, 3, 1, 1, 1),
    (1, 3, 16, 16, 5, 7, 7, 2, 3, 1),
    (2, 8, 7, 6, 6, 1, 1, 1, 0, 1),
    (1, 4, 10, 10, 4, 3, 3, 2, 2, 2),
    (2, 6, 5, 5, 6, 3, 3, 1, 1, 6),
    (1, 5, 6, 8, 3, 3, 3, 2, 0, 1),
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_exact_lut_is_torch_conv(case):
    """Exact LUT => float64 torch conv2d on integer tensors (exact below 2^53)."""
    Nb, C, H, Wd, K, R, S, st, pd, g = case
    X = datagen.random_int8(100 + H, (Nb, C, H, Wd))
    Wt = datagen.random_int8(200 + K, (K, C // g, R, S))
    Y = oracle.lut_conv2d(X, Wt, datagen.lut_exact(8), 8, (st, st), (pd, pd), groups=g)
    ref = torch.nn.functional.conv2d(torch.from_numpy(X.astype(np.float64)),
                                     torch.from_numpy(Wt.astype(np.float64)),
                                     stride=st, padding=pd, groups=g).numpy()
    np.testing.assert_array_equal(Y, ref.astype(np.int64))


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_equals_explicit_im2col_gemm(case):
    """Random ACU: direct conv == materialised im2col (torch unfold, padding as a = 0)
    through the LUT-GEMM ("multiplying these 2 matrices would compute the same dot
    product"); a grouped conv is that product per group (the group's input channels
    against the group's filters), outputs concatenated in group order."""
    Nb, C, H, Wd, K, R, S, st, pd, g = case
    X = datagen.random_int8(300 + H, (Nb, C, H, Wd))
    Wt = datagen.random_int8(400 + K, (K, C // g, R, S))
    T = datagen.random_lut(5, 8)
    Y = oracle.lut_conv2d(X, Wt, T, 8, (st, st), (pd, pd), groups=g)
    Ho, Wo = Y.shape[2:]
    cg, kg = C // g, K // g
    parts = []
    for gi in range(g):
        Xg = X[:, gi * cg:(gi + 1) * cg]
        cols = torch.nn.functional.unfold(torch.from_numpy(Xg.astype(np.float64)), (R, S),
                                          padding=pd, stride=st)           # [N, cg*R*S, L]
        Am = cols.permute(0, 2, 1).reshape(-1, cg * R * S).numpy().astype(np.int8)
        Wm = Wt[gi * kg:(gi + 1) * kg].reshape(kg, -1)
        parts.append(oracle.lut_gemm(Am, Wm, T, 8).reshape(Nb, Ho * Wo, kg).transpose(0, 2, 1))
    np.testing.assert_array_equal(Y.reshape(Nb, K, -1), np.concatenate(parts, axis=1))


def test_conv_padding_probe():
    """T = 1 everywhere: every output (border pixels included) counts R*S*C lookups --
    padded taps are looked up (A11)."""
    X = datagen.random_int8(9, (2, 5, 6, 7))
    Wt = datagen.random_int8(10, (3, 5, 3, 3))
    Y = oracle.lut_conv2d(X, Wt, np.ones(1 << 16, np.int32), 8, (1, 1), (2, 2))
    assert (Y == 5 * 9).all()
    # T[0][w] = 1, else 0: counts the zero taps (padding + genuine zeros) per output
    T = np.zeros(1 << 16, np.int32)
    T[:256] = 1
    X = np.ones((1, 1, 4, 4), np.int8)
    Y = oracle.lut_conv2d(X, np.ones((1, 1, 3, 3), np.int8), T, 8, (1, 1), (1, 1))
    expect = np.array([[5, 3, 3, 5], [3, 0, 0, 3], [3, 0, 0, 3], [5, 3, 3, 5]])
    np.testing.assert_array_equal(Y[0, 0], expect)


# ----------------------------------------------------------------------------------------
# quantize / dequantize (O2-O4, O7)
# ----------------------------------------------------------------------------------------

def test_quantizer_golden():
    rows = _golden("quantize_examples.txt")
    assert len(rows) >= 10
    for r in rows:
        if r[0] == "scale":
            s = oracle.scale(np.float32(r[1]), int(r[2]))
            assert s == np.float32(r[3]), r
        elif r[0] == "quantize":
            q = oracle.quantize(np.array([float(r[1])], np.float32), np.float32(r[2]), int(r[3]))
            assert int(q[0]) == int(r[4]), r
        elif r[0] == "dequant":
            y = oracle.dequantize(np.array([[int(r[1])]], np.int32), np.float32(r[2]), 1.0)
            assert abs(float(y[0, 0]) - float(r[3])) <= 1e-7, r


def test_amax_exact_and_zero():
    x = datagen.normal(9, 0, (1000, 37))
    assert oracle.amax(x) == np.max(np.abs(x))
    assert oracle.amax(np.zeros(10, np.float32)) == 0.0
    assert oracle.scale(0.0, 8) == 1.0                                   # A4


@pytest.mark.parametrize("bits", [2, 4, 6, 8])
def test_quantize_properties(bits):
    qmax = (1 << (bits - 1)) - 1
    x = datagen.normal(9, bits, (20000,), 1.7)
    q, s = oracle.quantize_tensor(x, bits)
    s64 = float(s)
    assert q.min() >= -qmax and q.max() <= qmax
    # nearest grid point (fp64 check, fp32 division rounding allowance): |x/s - q| <= 1/2
    r = x.astype(np.float64) / s64 - q.astype(np.float64)
    assert np.abs(r).max() <= 0.5 + 1e-5
    # round trip within half a scale step for |x| <= amax (BJ:ns "within one scale step")
    assert np.abs(q * s64 - x.astype(np.float64)).max() <= s64 / 2 * (1 + 1e-5)
    # amax maps to +-qmax exactly, oddness, monotonicity, idempotence
    i = np.argmax(np.abs(x))
    assert abs(int(q[i])) == qmax
    np.testing.assert_array_equal(oracle.quantize(-x, s, bits), -q)
    o = np.argsort(x, kind="stable")
    assert (np.diff(q[o].astype(np.int64)) >= 0).all()
    y = (q.astype(np.float32) * s).astype(np.float32)
    np.testing.assert_array_equal(oracle.quantize(y, s, bits), q)


def test_quantize_clamps_out_of_range():
    q = oracle.quantize(np.array([1e9, -1e9, 300.0, -300.0], np.float32), np.float32(1.0), 8)
    np.testing.assert_array_equal(q, [127, -127, 127, -127])


def test_dequantize_closed_form():
    rng = np.random.default_rng(3)
    acc = rng.integers(-2**31, 2**31, size=(37, 19), dtype=np.int64).astype(np.int32)
    b = rng.standard_normal(19).astype(np.float32)
    sa, sw = np.float32(0.0123), np.float32(0.00077)
    y = oracle.dequantize(acc, sa, sw, b)
    ref = acc.astype(np.float64) * float(sa) * float(sw) + b.astype(np.float64)[None, :]
    scale_ref = np.maximum(np.abs(ref), float(sa) * float(sw))
    assert (np.abs(y - ref) / scale_ref).max() <= 1e-6
    # NCHW channel bias
    acc4 = rng.integers(-1000, 1000, size=(2, 3, 4, 5), dtype=np.int64).astype(np.int32)
    b3 = np.array([1.0, -2.0, 3.0], np.float32)
    y4 = oracle.dequantize(acc4, 1.0, 1.0, b3, channel_axis=1)
    np.testing.assert_array_equal(y4, acc4 + b3[None, :, None, None])


def test_linear_exact_lut_tracks_float():
    """Sanity (not a pin of the LUT path): with the exact multiplier the approximate linear
    layer is plain quantized inference and tracks the fp32 layer within quantization error."""
    c = datagen.config1()
    x, W, b = c.x[:16], c.W[:64], c.b[:64]
    y, acc, (qa, sa, qw, sw) = oracle.linear(x, W, b, datagen.lut_exact(8), 8)
    ref = x.astype(np.float64) @ W.astype(np.float64).T + b
    err_bound = (np.abs(x).astype(np.float64) @ np.full(W.shape[::-1], sw / 2)
                 + np.full(x.shape, sa / 2) @ np.abs(W.T).astype(np.float64)
                 + x.shape[1] * sa * sw / 4)
    assert (np.abs(y - ref) <= err_bound * 1.001 + 1e-6).all()
