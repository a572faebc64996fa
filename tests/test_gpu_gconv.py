"""GPU parity of grouped and depthwise approximate convolution (NEXT-3; P:119 groups, the conv
of Eq. 2) against the oracle's direct seven-loop conv with groups: raw int32 bit-exact
for every table representation, and the fused dequantizing epilogue."""
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
    return _lib


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _table(kind):
    if kind == "randerr":
        return datagen.lut_randerr(8, 0, 2), 8
    if kind == "int16":
        return datagen.random_lut(33, 8), 8                                     # |T| <= 2^14
    if kind == "int32":
        return np.random.default_rng(41).integers(-10**6, 10**6, 1 << 16).astype(np.int32), 8
    return datagen.lut_randerr(4, 4, 14), 4


# N, C, H, W, K, R, S, stride, pad, dil, groups
CASES = [(2, 32, 10, 9, 32, 3, 3, 1, 1, 1, 32),     # depthwise 3x3
         (3, 24, 7, 70, 24, 3, 3, 1, 1, 1, 24),     # depthwise 3x3 s1 p1 (DW3): 3 strips, partial channel block
         (1, 40, 31, 61, 40, 3, 3, 1, 1, 1, 40),    # DW3: ragged last strip, 3 channel blocks
         (2, 64, 11, 37, 64, 3, 3, 2, 1, 1, 64),    # depthwise 3x3 stride 2, 2 channel blocks, ragged tiles
         (1, 96, 9, 70, 96, 3, 3, 1, 0, 1, 96),     # depthwise 3x3, no padding, 3 column tiles
         (1, 16, 12, 12, 32, 3, 3, 2, 1, 1, 16),    # depthwise, channel multiplier 2, stride 2
         (2, 24, 8, 11, 36, 1, 1, 1, 0, 1, 3),      # grouped 1x1 (ShuffleNet-like, G = 3)
         (1, 32, 9, 9, 64, 5, 5, 1, 2, 1, 4),       # grouped 5x5
         (1, 8, 13, 7, 8, 3, 3, 1, 2, 2, 8),        # depthwise, dilation 2
         (3, 12, 5, 6, 12, 3, 1, 2, 0, 1, 2),       # rectangular kernel, no padding
         (2, 64, 10, 10, 64, 3, 3, 1, 1, 1, 2),     # wide groups: per-group dense GEMM (16-B loads)
         (1, 48, 7, 9, 96, 1, 1, 2, 0, 1, 3),       # wide groups, 1x1 stride 2
         (1, 80, 6, 6, 40, 3, 3, 1, 1, 1, 4)]       # wide groups, C/G = 20 (4-byte loads)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("kind", ["randerr", "int16", "int32", "b4"])
def test_grouped_conv_raw(ax, case, kind):
    Nb, C, H, Wd, K, R, S, st, pd, dl, G = case
    T, bits = _table(kind)
    X = datagen.random_int8(300 + C + G, (Nb, C, H, Wd), bits)
    Wt = datagen.random_int8(400 + K + G, (K, C // G, R, S), bits)
    ref = oracle.lut_conv2d(X, Wt, T, bits, (st, st), (pd, pd), (dl, dl), groups=G)
    lut = ax.Lut(bits, T)
    d = ax.conv_desc(Nb, H, Wd, C, K, R, S, (st, st), (pd, pd), (dl, dl), groups=G)
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    Y = torch.empty(Nb, Ho, Wo, K, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d(d, _t(X.transpose(0, 2, 3, 1)), _t(Wt.transpose(0, 2, 3, 1)), lut, Y)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)


def test_depthwise_fused_nchw(ax):
    Nb, C, H, Wd = 4, 64, 14, 14
    x = np.maximum(datagen.normal(35, 1, (Nb, C, H, Wd)), 0).astype(np.float32)
    rng = np.random.default_rng(42)
    w = (rng.standard_normal((C, 1, 3, 3)) * 0.3).astype(np.float32)
    b = rng.standard_normal(C).astype(np.float32)
    T = datagen.lut_randerr(8, 0, 2)
    qa, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(w, 8)
    acc = oracle.lut_conv2d(qa, qw, T, 8, (1, 1), (1, 1), groups=C)
    ref = oracle.dequantize(acc, sa, sw, b, channel_axis=1)
    lut = ax.Lut(8, T)
    d = ax.conv_desc(Nb, H, Wd, C, C, 3, 3, (1, 1), (1, 1), groups=C)
    y = torch.empty(Nb, C, H, Wd, device=DEV)
    dsa, dsw, db = torch.tensor([sa], device=DEV), torch.tensor([sw], device=DEV), _t(b)
    ep = ax.make_epilogue(dsa, dsw, bias=db, y=y)
    ax.axq_lut_conv2d_ep(d, _t(qa.transpose(0, 2, 3, 1)), _t(qw.transpose(0, 2, 3, 1)), lut, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


def test_wide_groups_fused_nchw_per_channel(ax):
    """Per-group dense path with the fused epilogue: NCHW output slices, bias and per-channel
    weight scales offset per group, split-K workspace reused across groups."""
    Nb, C, H, Wd, K, G = 2, 64, 12, 12, 96, 2
    rng = np.random.default_rng(50)
    X = datagen.random_int8(51, (Nb, C, H, Wd))
    Wt = datagen.random_int8(52, (K, C // G, 3, 3))
    T = datagen.lut_randerr(8, 0, 2)
    s_w = rng.uniform(1e-4, 1e-2, K).astype(np.float32)
    b = rng.standard_normal(K).astype(np.float32)
    s_a = np.float32(0.02)
    ref = oracle.dequantize_pc(oracle.lut_conv2d(X, Wt, T, 8, (1, 1), (1, 1), groups=G), s_a, s_w, b,
                               channel_axis=1)
    lut = ax.Lut(8, T)
    d = ax.conv_desc(Nb, H, Wd, C, K, 3, 3, (1, 1), (1, 1), groups=G)
    y = torch.empty(Nb, K, H, Wd, device=DEV)
    ws = torch.zeros(Nb * H * Wd * K, dtype=torch.int32, device=DEV)
    dsa, dsw, dones, db = torch.tensor([s_a], device=DEV), _t(s_w), torch.ones(1, device=DEV), _t(b)
    ep = ax.make_epilogue(dsa, dones, bias=db, y=y, workspace=ws, d_scale_w_ch=dsw)
    ax.axq_lut_conv2d_ep(d, _t(X.transpose(0, 2, 3, 1)), _t(Wt.transpose(0, 2, 3, 1)), lut, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("shape", [(2, 3, 4, 20, 18, 7, 2, 3), (1, 5, 8, 9, 9, 3, 1, 1), (3, 16, 16, 5, 6, 1, 1, 0),
                                   (2, 3, 4, 31, 29, 7, 2, 3)])
def test_im2col_nhwc_i8(ax, shape):
    """Explicit im2col (axq_im2col_nhwc_i8) against a direct numpy construction: k = (r, s, c) over
    the c_valid channels, 0 at padded taps and past K."""
    N, cv, C, H, W, R, st, pd = shape
    X = datagen.random_int8(90 + C, (N, H, W, C))
    Ho, Wo = (H + 2 * pd - R) // st + 1, (W + 2 * pd - R) // st + 1
    K = R * R * cv
    lda = 160 if (C, cv, R) == (4, 3, 7) and (H, W) == (31, 29) else (K + 15) // 16 * 16 + 16
    Xp = np.zeros((N, H + 2 * pd, W + 2 * pd, C), np.int8)
    Xp[:, pd:pd + H, pd:pd + W] = X
    ref = np.zeros((N * Ho * Wo, lda), np.int8)
    for ho in range(Ho):
        for wo in range(Wo):
            patch = Xp[:, ho * st:ho * st + R, wo * st:wo * st + R, :cv].reshape(N, -1)
            ref[np.arange(N) * Ho * Wo + ho * Wo + wo, :K] = patch
    A = torch.full((N * Ho * Wo, lda), 77, dtype=torch.int8, device=DEV)
    ax.axq_im2col_nhwc_i8(_t(X), cv, R, R, (st, st), (pd, pd), A)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(A.cpu().numpy(), ref)


@pytest.mark.parametrize("shape", [(2, 32, 13, 40), (1, 64, 9, 31), (3, 48, 7, 70)])
@pytest.mark.parametrize("per_channel", [False, True])
@pytest.mark.parametrize("with_y", [True, False], ids=["y+q", "q-only"])
def test_depthwise_dw3_fused_nhwc(ax, shape, per_channel, with_y):
    """The depthwise 3x3 / stride 1 / pad 1 kernel's fused NHWC epilogue (fp32 y and requantized
    codes, bias, ReLU, per-channel weight scales), computed in-loop and stored through shared
    memory, against the oracle."""
    Nb, C, H, Wd = shape
    T = datagen.lut_randerr(8, 0, 2)
    qa = datagen.random_int8(700 + C, (Nb, C, H, Wd), full_range=False)
    qw = datagen.random_int8(701 + C, (C, 1, 3, 3))
    acc = oracle.lut_conv2d(qa, qw, T, 8, (1, 1), (1, 1), groups=C)          # NCHW int
    rng = np.random.default_rng(C + H)
    s_a = np.float32(0.011)
    s_w = rng.uniform(0.002, 0.02, C).astype(np.float32) if per_channel else np.float32(0.009)
    b = rng.standard_normal(C).astype(np.float32)
    s_o = np.float32(0.37)
    acc_nhwc = acc.transpose(0, 2, 3, 1).reshape(-1, C)
    y_ref = (oracle.dequantize_pc(acc_nhwc, s_a, s_w, b) if per_channel
             else oracle.dequantize(acc_nhwc, s_a, s_w, b))
    y_ref = np.maximum(y_ref, 0).astype(np.float32)
    q_ref = oracle.quantize(y_ref, s_o, 8)
    lut = ax.Lut(8, T)
    d = ax.conv_desc(Nb, H, Wd, C, C, 3, 3, (1, 1), (1, 1), groups=C)
    M = Nb * H * Wd
    y = torch.full((M, C), np.nan, device=DEV)
    q = torch.zeros(M, C, dtype=torch.int8, device=DEV)
    kw = dict(d_scale_w_ch=_t(s_w)) if per_channel else {}
    ep = ax.make_epilogue(torch.tensor([s_a], device=DEV),
                          torch.tensor([1.0 if per_channel else s_w], device=DEV), bias=_t(b),
                          y=y if with_y else None, ldy=C, relu=True, y_nhwc=True, q_out=q, ldq=C,
                          d_scale_out=torch.tensor([s_o], device=DEV), bits_out=8, **kw)
    ax.axq_lut_conv2d_ep(d, _t(qa.transpose(0, 2, 3, 1)), _t(qw.transpose(0, 2, 3, 1)), lut, ep)
    torch.cuda.synchronize()
    if with_y:
        np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
    np.testing.assert_array_equal(q.cpu().numpy(), q_ref)


# grouped convs on the packed-table P4W path (axq_lut_conv2d_wp; C/G and K/G multiples of 16)
WP_CASES = [(2, 64, 10, 10, 64, 3, 3, 1, 1, 2),      # 3x3, G = 2
            (2, 64, 12, 12, 64, 1, 1, 1, 0, 4),      # pointwise 1x1, G = 4 (GEMM-row loader)
            (1, 96, 9, 11, 48, 1, 1, 2, 0, 3),       # 1x1 stride 2, G = 3
            (3, 32, 7, 9, 64, 3, 3, 2, 1, 2),        # 3x3 stride 2, K/G = 32
            (4, 64, 28, 28, 256, 1, 1, 1, 0, 4)]     # the bench's ShuffleNet-like shape, scaled down


@pytest.mark.parametrize("case", WP_CASES)
@pytest.mark.parametrize("half", [False, True])
def test_grouped_conv_packed(ax, case, half):
    """Grouped conv through weight-specialised packed tables: a 16-column tile's group selects its
    input channels (bit-exact against the oracle's direct grouped conv)."""
    Nb, C, H, Wd, K, R, S, st, pd, G = case
    T, bits = _table("randerr")
    X = datagen.random_int8(500 + C + G, (Nb, C, H, Wd), bits, full_range=not half)
    if half:   # half-range tables: non-negative (ReLU'd) activation codes only
        X = np.abs(X.astype(np.int16)).astype(np.int8)
    Wt = datagen.random_int8(600 + K + G, (K, C // G, R, S), bits)
    ref = oracle.lut_conv2d(X, Wt, T, bits, (st, st), (pd, pd), groups=G)
    lut = ax.Lut(bits, T)
    wp = ax.WPack(lut, _t(Wt.transpose(0, 2, 3, 1)).reshape(K, -1), a_nonneg=half)
    d = ax.conv_desc(Nb, H, Wd, C, K, R, S, (st, st), (pd, pd), groups=G)
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    Y = torch.empty(Nb, Ho, Wo, K, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d_wp(d, _t(X.transpose(0, 2, 3, 1)), wp, None, Y)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)


@pytest.mark.parametrize("G,C,K,R", [(4, 64, 64, 3), (3, 24, 36, 1), (2, 64, 64, 3), (4, 256, 128, 1)])
def test_approx_conv2d_layer_groups(ax, G, C, K, R):
    """layers.ApproxConv2d with groups: packed tables when C/G and K/G are multiples of 16 (and
    the per-group K = R*S*C/G >= 128), else the grouped resident-table path; both equal the
    oracle's quantize -> grouped LUT conv -> dequantize chain bit for bit."""
    from paper_2203_04071_b200.layers import ApproxConv2d
    Nb, H, Wd = 3, 12, 12
    x = np.maximum(datagen.normal(70 + G, 1, (Nb, C, H, Wd)), 0).astype(np.float32)
    w = datagen.normal(71 + G, 2, (K, C // G, R, R), 0.1)
    T = datagen.lut_randerr(8, 0, 2)
    s_a = oracle.scale(oracle.amax(x), 8)
    qw, s_w = oracle.quantize_tensor(w, 8)
    acc = oracle.lut_conv2d(oracle.quantize(x, s_a, 8), qw, T, 8, (1, 1), (R // 2, R // 2), groups=G)
    y_ref = oracle.dequantize(acc, s_a, s_w, None, 1)
    layer = ApproxConv2d(_t(w), None, ax.Lut(8, T), (1, 1), (R // 2, R // 2), a_nonneg=True, groups=G)
    assert (layer.wp is not None) == ((C // G) % 16 == 0 and (K // G) % 16 == 0 and (C // G) * R * R >= 128)
    y = layer(_t(x))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
