"""Quantize-on-load variants (SURVEY §8(b) conventions): axq_lut_gemm_f32a (fp32 A + its
device scale) and axq_lut_conv2d_f32 (fp32 NCHW input) must equal the unfused
axq_quantize -> axq_lut_gemm / axq_lut_conv2d chain bit for bit (raw int32 and fused epilogue),
and the oracle."""
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


def _lut(kind):
    return {"randerr": (datagen.lut_randerr(8, 0, 2), 8), "trunc4": (datagen.lut_trunc4(), 8),
            "b4": (datagen.lut_randerr(4, 4, 14), 4),
            "int16": (datagen.lut_randerr(8, 0, 2) + 1000, 8),       # E beyond int8 -> int16 table
            "int32": (datagen.lut_randerr(8, 0, 2) * 3, 8)}[kind]     # beyond int16 -> int32 table


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (100, 33, 77), (256, 1024, 1024), (300, 40, 17),
                                   (64, 64, 256)])
@pytest.mark.parametrize("kind", ["randerr", "trunc4", "b4", "int16", "int32"])
def test_gemm_f32a_equals_unfused_chain(ax, M, N, K, kind):
    T, bits = _lut(kind)
    x = datagen.normal(700 + M, K, (M, K))
    Wf = datagen.normal(710 + N, K, (N, K), 0.02)
    s_a = oracle.scale(oracle.amax(x), bits)
    qw, s_w = oracle.quantize_tensor(Wf, bits)
    qa = oracle.quantize(x, s_a, bits)
    ref = oracle.lut_gemm(qa, qw, T, bits)
    lut = ax.Lut(bits, T)
    dx, dsa, dw = _t(x), _t(np.array([s_a])), _t(qw)
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm_f32a(dx, dsa, dw, lut, None, C)
    assert ax.axq_last_path()[0] == "f32a"
    C2 = torch.empty(M, N, dtype=torch.int32, device=DEV)
    dq = torch.empty(M, K, dtype=torch.int8, device=DEV)
    ax.axq_quantize(dx, dsa, bits, dq)
    ax.axq_lut_gemm(dq, dw, lut, C2)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), ref)
    np.testing.assert_array_equal(C2.cpu().numpy(), ref)
    # fused epilogue, with and without a split-K workspace
    b = datagen.normal(720 + N, 1, (N,), 0.01)
    y_ref = oracle.dequantize(ref, s_a, s_w, b)
    for ws in (None, torch.zeros(M * N, dtype=torch.int32, device=DEV)):
        y = torch.empty(M, N, device=DEV)
        ep = ax.make_epilogue(dsa, _t(np.array([s_w])), bias=_t(b), y=y, ldy=N, workspace=ws)
        ax.axq_lut_gemm_f32a(dx, dsa, dw, lut, ep)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy(), y_ref)


def test_gemm_f32a_ties_and_clamp(ax):
    """Crafted ties at s = 1 (amax = 127): x = k + 1/2 rounds half to even (A1), |x| > 127
    clamps (A2), +-0 give code 0, a strided (lda > K) operand."""
    T, bits = _lut("randerr")
    K = 48
    vals = np.array([2.5, 3.5, -2.5, -0.5, 0.5, 126.5, 127.0, -127.0, 200.0, -300.0, 0.0, -0.0,
                     1.4999999, 1.5, 64.5, -64.5], np.float32)
    x = np.zeros((8, 64), np.float32)
    for i in range(8):
        x[i, :K] = np.resize(np.roll(vals, i), K)
    s_a = np.float32(1.0)
    qa = oracle.quantize(x[:, :K], s_a, bits)
    W = datagen.random_int8(731, (16, K))
    ref = oracle.lut_gemm(qa, W, T, bits)
    lut = ax.Lut(bits, T)
    dx = _t(x)[:, :K]                    # lda = 64 > K
    C = torch.empty(8, 16, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm_f32a(dx, _t(np.array([s_a])), _t(W), lut, None, C)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), ref)


@pytest.mark.parametrize("shape", [
    (2, 64, 14, 14, 64, 3, 3, 1, 1),     # c2-like
    (1, 3, 23, 19, 16, 7, 7, 2, 3),      # stem-like, C = 3
    (2, 16, 9, 11, 40, 3, 3, 2, 2),
    (3, 24, 8, 8, 33, 1, 1, 1, 0),
    (1, 32, 7, 7, 70, 1, 1, 2, 0),
])
@pytest.mark.parametrize("relu", [False, True])
def test_conv2d_f32_equals_unfused_chain(ax, shape, relu):
    Nb, C, H, Wd, K, R, S, st, pd = shape
    T, bits = _lut("randerr")
    x = datagen.normal(740 + C, H, (Nb, C, H, Wd))
    if relu:
        x = np.maximum(x, 0)
    Wf = datagen.normal(750 + K, R, (K, C, R, S), 0.05)
    y_ref, acc_ref, (qx, s_a, qw, s_w) = oracle.conv2d(x, Wf, None, T, bits, (st, st), (pd, pd))
    lut = ax.Lut(bits, T)
    d = ax.conv_desc(Nb, H, Wd, C, K, R, S, (st, st), (pd, pd))
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    dx, dsa = _t(x), _t(np.array([s_a]))
    dw = _t(qw.transpose(0, 2, 3, 1))
    Y = torch.empty(Nb, Ho, Wo, K, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d_f32(d, dx, dsa, dw, lut, None, Y)
    assert ax.axq_last_path()[0] == "f32a"
    # the unfused chain: quantize NCHW -> NHWC int8, then the int8 conv
    dq = torch.empty(Nb, H, Wd, C, dtype=torch.int8, device=DEV)
    ax.axq_quantize_nchw_to_nhwc(dx, dsa, bits, dq)
    Y2 = torch.empty_like(Y)
    ax.axq_lut_conv2d(d, dq, dw, lut, Y2)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), acc_ref)
    np.testing.assert_array_equal(Y2.cpu().numpy(), Y.cpu().numpy())
    y = torch.empty(Nb, K, Ho, Wo, device=DEV)
    ep = ax.make_epilogue(dsa, _t(np.array([s_w])), y=y)
    ax.axq_lut_conv2d_f32(d, dx, dsa, dw, lut, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), y_ref)


def test_conv2d_f32_config2_sampled(ax):
    """BJ configs[2] at full batch through the quantize-on-load conv: sampled images bit-exact."""
    c = datagen.config2()
    lut = ax.Lut(8, c.lut)
    s_a = oracle.scale(oracle.amax(c.x), 8)
    qw, s_w = oracle.quantize_tensor(c.W, 8)
    d = ax.conv_desc(128, 56, 56, 64, 64, 3, 3, (1, 1), (1, 1))
    y = torch.empty(128, 64, 56, 56, device=DEV)
    ep = ax.make_epilogue(_t(np.array([s_a])), _t(np.array([s_w])), y=y)
    ax.axq_lut_conv2d_f32(d, _t(c.x), _t(np.array([s_a])), _t(qw.transpose(0, 2, 3, 1)), lut, ep)
    torch.cuda.synchronize()
    for img in (0, 77):
        acc = oracle.lut_conv2d(oracle.quantize(c.x[img:img + 1], s_a, 8), qw, c.lut, 8, (1, 1), (1, 1))
        np.testing.assert_array_equal(y[img:img + 1].cpu().numpy(), oracle.dequantize(acc, s_a, s_w, None, 1))


def test_f32a_errors(ax):
    T, bits = _lut("randerr")
    lut = ax.Lut(bits, T)
    x = torch.zeros(4, 8, device=DEV)
    W = torch.zeros(4, 8, dtype=torch.int8, device=DEV)
    C = torch.empty(4, 4, dtype=torch.int32, device=DEV)
    with pytest.raises(ax.AxqError) as e:
        ax.axq_lut_gemm_f32a(x, None, W, lut, None, C)
    assert e.value.status == ax.AXQ_ERR_INVALID
    d = ax.conv_desc(1, 4, 4, 4, 4, 1, 1, c_valid=3)
    with pytest.raises(ax.AxqError) as e:
        ax.axq_lut_conv2d_f32(d, torch.zeros(1, 4, 4, 4, device=DEV), torch.ones(1, device=DEV),
                              W.reshape(4, 1, 1, 8)[:, :, :, :4].contiguous(), lut, None,
                              torch.empty(1, 4, 4, 4, dtype=torch.int32, device=DEV))
    assert e.value.status == ax.AXQ_ERR_UNSUPPORTED
