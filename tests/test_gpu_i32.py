"""GPU parity of the int32 tables: an ACU whose error E = LUT - a*w does not fit int16, so
neither the int8-E (P4W) nor the int16-E (P4W16) packed tables can hold it.  Both kernel forms
run every case: the L1 gather (lut_mm_kernel<REPR_I32>) and the SM-resident halves
(lut_mm_kernel<REPR_I32H>: the 256 KiB table as two 128 KiB shared-memory halves by the
activation's high bit, a second pass only for tiles with codes of the other half; north_star
"int32 split across SM-resident halves").

Against the CPU oracle, bit-exact: ragged GEMM shapes (activations of both signs, so both halves
contribute), tiles walked several per CTA (the resident half carries over between tiles),
non-negative activations (one pass), split-K, K-tail padding, low bitwidths, convolutions, and
the fused dequant epilogue."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda"
BIG = 100_000      # |E| up to 1e5: beyond int16


@pytest.fixture(params=[False, True], ids=["l1", "resident"])
def resident(request):
    return request.param


@pytest.fixture(scope="module")
def ax():
    from paper_2203_04071_b200 import _lib
    _lib.load()
    return _lib


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _table(bits, idx, err=BIG):
    return datagen.lut_bigerr(bits, err, 7, idx)


def _gemm(ax, A, W, T, bits, resident):
    lut = ax.Lut(bits, T)
    assert lut.repr == "int32"
    lut.set_i32_resident(resident)
    C = torch.empty(A.shape[0], W.shape[0], dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm(_t(A), _t(W), lut, C)
    path = ax.axq_last_path()[0]
    torch.cuda.synchronize()
    out = C.cpu().numpy()
    lut.close()
    return out, path


SHAPES = [(1, 1, 1), (7, 13, 5), (33, 5, 147), (129, 65, 300), (600, 40, 77),
          (2049, 33, 1040), (20000, 64, 100), (64, 64, 8192), (5000, 7, 19)]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_i32_gemm_ragged(ax, resident, M, N, K):
    A = datagen.random_int8(110 + M, (M, K))
    W = datagen.random_int8(120 + N, (N, K))
    T = _table(8, 1)
    C, path = _gemm(ax, A, W, T, 8, resident)
    assert path.startswith("v1")
    np.testing.assert_array_equal(C, oracle.lut_gemm(A, W, T, 8))


def test_i32_one_sign_of_weights(ax, resident):
    """All weights >= 0 and all < 0."""
    M, N, K = 300, 48, 96
    A = datagen.random_int8(131, (M, K))
    T = _table(8, 2)
    for sign in (1, -1):
        W = (np.abs(datagen.random_int8(132, (N, K)).astype(np.int64)) % 128).astype(np.int8)
        if sign < 0:
            W = (-W.astype(np.int64) - 1).astype(np.int8)
        C, _ = _gemm(ax, A, W, T, 8, resident)
        np.testing.assert_array_equal(C, oracle.lut_gemm(A, W, T, 8))


def test_i32_extreme_corners(ax, resident):
    """Codes -128 / 127 and 0 only: the corner entries of both halves, K-tail padding."""
    M, N, K = 97, 17, 37
    vals = np.array([-128, 127, 0, -1], np.int8)
    A = vals[datagen.random_int8(141, (M, K)).astype(np.int64) & 3]
    W = vals[datagen.random_int8(142, (N, K)).astype(np.int64) & 3]
    T = _table(8, 3)
    C, _ = _gemm(ax, A, W, T, 8, resident)
    np.testing.assert_array_equal(C, oracle.lut_gemm(A, W, T, 8))


@pytest.mark.parametrize("bits", [6, 7])
def test_i32_low_bitwidths(ax, resident, bits):
    M, N, K = 200, 40, 129
    half = 1 << (bits - 1)
    A = (datagen.random_int8(150 + bits, (M, K)).astype(np.int64) % half).astype(np.int8)
    W = (datagen.random_int8(160 + bits, (N, K)).astype(np.int64) % half - half // 2).astype(np.int8)
    T = _table(bits, 4 + bits)
    C, _ = _gemm(ax, A, W, T, bits, resident)
    np.testing.assert_array_equal(C, oracle.lut_gemm(A, W, T, bits))


CONV_SHAPES = [
    # N, C, H, W, K, R, S, stride, pad
    (2, 64, 14, 14, 64, 3, 3, 1, 1),
    (1, 3, 32, 32, 64, 7, 7, 2, 3),
    (2, 20, 6, 6, 8, 3, 3, 2, 0),
]


@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_i32_conv(ax, resident, shape):
    Nb, C, H, Wd, K, R, S, st, pd = shape
    X = datagen.random_int8(170 + C, (Nb, C, H, Wd))
    Wt = datagen.random_int8(180 + K, (K, C, R, S))
    T = _table(8, 20, err=20_000)        # K * max|LUT| stays below 2^31 at C*R*S = 576
    ref = oracle.lut_conv2d(X, Wt, T, 8, (st, st), (pd, pd))
    lut = ax.Lut(8, T)
    assert lut.repr == "int32"
    lut.set_i32_resident(resident)
    d = ax.conv_desc(Nb, H, Wd, C, K, R, S, (st, st), (pd, pd))
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    Y = torch.empty(Nb, Ho, Wo, K, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d(d, _t(X.transpose(0, 2, 3, 1)), _t(Wt.transpose(0, 2, 3, 1)), lut, Y)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)
    lut.close()


def test_i32_fused_linear(ax, resident):
    """quantize -> LUT-GEMM (int32 table) -> dequant + bias, against the oracle's layer."""
    from paper_2203_04071_b200.layers import ApproxLinear
    c1 = datagen.config1()
    x, W, b = c1.x[:200], c1.W[:96], c1.b[:96]
    T = _table(8, 30, err=40_000)
    lut = ax.Lut(8, T)
    assert lut.repr == "int32"
    lut.set_i32_resident(resident)
    y = ApproxLinear(_t(W), _t(b), lut)(_t(x))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.linear(x, W, b, T, 8)[0])


@pytest.mark.parametrize("sign", ["nonneg", "neg", "mixed_rows"])
def test_i32_activation_halves(ax, resident, sign):
    """Activations all >= 0 (half 0 only: one pass), all < 0 (half 1 only), and only a few rows
    with negative codes (the second pass runs for their tiles alone)."""
    M, N, K = 3000, 40, 150
    A = (np.abs(datagen.random_int8(191, (M, K)).astype(np.int64)) % 128).astype(np.int64)
    if sign == "neg":
        A = -A - 1
    elif sign == "mixed_rows":
        A[::997] = -A[::997] - 1
    A = A.astype(np.int8)
    W = datagen.random_int8(192, (N, K))
    T = _table(8, 40)
    C, _ = _gemm(ax, A, W, T, 8, resident)
    np.testing.assert_array_equal(C, oracle.lut_gemm(A, W, T, 8))


def test_i32_mode_switch_is_int32_only(ax):
    lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
    with pytest.raises(ax.AxqError):
        lut.set_i32_resident(True)
    lut.close()
