"""GPU parity of the P4W activation loads by TMA: GEMM rows through a 2D tiled tensor map and
convs through an im2col-mode tensor map (padding taps, strides, dilation, rows running past
the last image, ragged K and M).  Each case checks that the launch took the TMA path
(axq_last_path flags) and is bit-exact against the oracle (integer accumulators)."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def ax():
    from paper_2203_04071_b200 import _lib
    _lib.load()
    prev = _lib.axq_wpack_kernel(3)      # P4W
    yield _lib
    _lib.axq_wpack_kernel(prev)


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("M,N,K", [(1, 16, 16), (127, 16, 48), (1000, 32, 200), (2305, 48, 64),
                                   (9000, 16, 1040)])
def test_tma_gemm_rows(ax, M, N, K):
    T = datagen.lut_randerr(8, 0, 2)
    A = datagen.random_int8(700 + M, (M, K))
    W = datagen.random_int8(800 + N, (N, K))
    ref = oracle.lut_gemm(A, W, T, 8)
    Kp = (K + 15) // 16 * 16
    dA = torch.zeros(M, Kp, dtype=torch.int8, device=DEV)      # row stride % 16 == 0
    dA[:, :K] = _t(A)
    wp = ax.WPack(ax.Lut(8, T), _t(W))
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm_wp(dA.narrow(1, 0, K), wp, None, C)
    fam, flags = ax.axq_last_path()
    torch.cuda.synchronize()
    assert fam == "p4w" and flags & ax.PATH_TMA, (fam, hex(flags))
    np.testing.assert_array_equal(C.cpu().numpy(), ref)


# (N, C, H, W, K, R, stride, pad, dil): stride 2 / valid / dilated / 7x7 windows, images whose
# pixel count is not a multiple of 128 (slices cross image boundaries), M past a whole tile
@pytest.mark.parametrize("shape", [(3, 32, 14, 14, 16, 3, 1, 1, 1), (2, 16, 17, 13, 32, 3, 2, 1, 1),
                                   (2, 64, 12, 12, 16, 1, 2, 0, 1), (1, 16, 20, 20, 16, 5, 1, 2, 1),
                                   (2, 32, 11, 11, 16, 3, 1, 0, 1), (1, 16, 15, 15, 16, 3, 1, 2, 2),
                                   (2, 16, 30, 30, 16, 7, 2, 3, 1), (5, 48, 9, 9, 32, 3, 1, 1, 1)])
def test_tma_im2col_conv(ax, shape):
    Nb, C, H, Wd, K, R, st, pd, dl = shape
    X = datagen.random_int8(900 + C + H, (Nb, C, H, Wd))
    Wt = datagen.random_int8(950 + K + R, (K, C, R, R))
    T = datagen.lut_randerr(8, 0, 2)
    ref = oracle.lut_conv2d(X, Wt, T, 8, (st, st), (pd, pd), (dl, dl))
    d = ax.conv_desc(Nb, H, Wd, C, K, R, R, (st, st), (pd, pd), (dl, dl))
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    wp = ax.WPack(ax.Lut(8, T), _t(Wt.transpose(0, 2, 3, 1).reshape(K, -1)))
    Y = torch.empty(Nb, Ho, Wo, K, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d_wp(d, _t(X.transpose(0, 2, 3, 1)), wp, None, Y)
    fam, flags = ax.axq_last_path()
    torch.cuda.synchronize()
    pointwise = R == 1 and st == 1 and pd == 0
    want = ax.PATH_TMA if pointwise else ax.PATH_TMA_IM2COL
    assert fam == "p4w" and flags & want, (fam, hex(flags))
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)


@pytest.mark.parametrize("M,N,K", [(3000, 64, 64), (20000, 48, 256), (641, 32, 128)])
def test_tma_residual_rows_and_y_store(ax, M, N, K):
    """The residual-layer shape's TMA residual staging and y stores (swizzled rows, one box per
    128-row slice): ragged M (rows past M zero-filled on the way in, clipped on the way out),
    a ragged column block when N % 16 != 0 is not used here (the generic path covers it), stream-K
    tails at M = 20000.  Residual + ReLU + y + requantize against the oracle, bit-exact."""
    T = datagen.lut_randerr(8, 0, 2)
    A = np.random.default_rng(1100 + M).integers(0, 128, (M, K)).astype(np.int8)   # ReLU-input codes
    W = datagen.random_int8(1200 + N, (N, K))
    acc = oracle.lut_gemm(A, W, T, 8)
    sa, sw = np.float32(0.0213), np.float32(0.0071)
    R = datagen.normal(1300 + M, 3, (M, N), 1.0)
    y_ref = (oracle.dequantize(acc, sa, sw) + R).astype(np.float32)
    y_ref = np.where(y_ref > 0, y_ref, np.float32(0)).astype(np.float32)
    so = np.float32(0.05)
    q_ref = oracle.quantize(y_ref, so, 8)
    wp = ax.WPack(ax.Lut(8, T), _t(W), a_nonneg=True)
    y = torch.full((M, N), np.nan, device=DEV)
    q = torch.zeros(M, N, dtype=torch.int8, device=DEV)
    ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
    ep = ax.make_epilogue(_t(np.array([sa])), _t(np.array([sw])), workspace=ws, residual=_t(R), ldr=N,
                          relu=True, y=y, ldy=N, q_out=q, ldq=N, d_scale_out=_t(np.array([so])), bits_out=8)
    ax.axq_lut_gemm_wp(_t(A), wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
    np.testing.assert_array_equal(q.cpu().numpy(), q_ref)
