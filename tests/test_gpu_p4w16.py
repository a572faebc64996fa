"""GPU parity of the packed int16-E kernel (P4W16): tables whose error E = LUT - a*w does not
fit int8 (here |E| <= 2000, or LUT values beyond int16) are packed 2 columns per 32-bit word
and run on the warp-specialised tcgen05 kernel instead of the one-lookup-per-load gather.
Bit-exact against the oracle; the path taken is asserted."""
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
    if kind == "err2000":
        return datagen.lut_bigerr(8, 2000, 8, 1)
    if kind == "err30000":                     # E near the int16 limit
        return datagen.lut_bigerr(8, 30000, 8, 2)
    return datagen.lut_randerr(8, 0, 2) * 3     # LUT values beyond int16 (int32 table), E = 2ab+3e


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (1100, 16, 2048), (3000, 48, 576), (600, 40, 100),
                                   (4096, 64, 256), (1025, 17, 1040)])
@pytest.mark.parametrize("kind", ["err2000", "err30000"])
def test_p4w16_gemm_raw_and_fused(ax, M, N, K, kind):
    T = _lut(kind)
    A = (datagen.random_int8(600 + M, (M, K)).astype(np.int64) & 127).astype(np.int8)   # a >= 0
    W = datagen.random_int8(700 + N, (N, K))
    ref = oracle.lut_gemm(A, W, T, 8)
    lut = ax.Lut(8, T)
    assert lut.repr in ("int16", "int32")
    wp = ax.WPack(lut, _t(W), a_nonneg=True)
    Kp = (K + 15) // 16 * 16
    dA = torch.zeros(M, Kp, dtype=torch.int8, device=DEV)
    dA[:, :K] = _t(A)
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm_wp(dA.narrow(1, 0, K), wp, None, C)
    assert ax.axq_last_path()[0] == "p4w16"
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), ref)
    sa, sw = np.float32(0.013), np.float32(0.002)
    b = datagen.normal(6, 6, (N,), 0.1)
    y = torch.empty(M, N, device=DEV)
    ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
    ep = ax.make_epilogue(_t(np.array([sa])), _t(np.array([sw])), bias=_t(b), y=y, ldy=N, workspace=ws)
    ax.axq_lut_gemm_wp(dA.narrow(1, 0, K), wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.dequantize(ref, sa, sw, b))


def test_p4w16_requires_nonneg_activations(ax):
    lut = ax.Lut(8, _lut("err2000"))
    W = _t(datagen.random_int8(5, (16, 64)))
    with pytest.raises(ax.AxqError) as e:
        ax.WPack(lut, W, a_nonneg=False)
    assert e.value.status == ax.AXQ_ERR_UNSUPPORTED


def test_p4w16_residual_epilogue(ax):
    """The residual / ReLU / requantize epilogue on the int16-E kernel (its 512-row shape)."""
    M, N, K = 2048, 48, 64
    T = _lut("err2000")
    A = (datagen.random_int8(811, (M, K)).astype(np.int64) & 127).astype(np.int8)
    W = datagen.random_int8(812, (N, K))
    acc = oracle.lut_gemm(A, W, T, 8)
    res = datagen.normal(8, 13, (M, N))
    sa, sw, so = np.float32(0.003), np.float32(0.01), np.float32(0.05)
    y_ref = oracle.dequantize(acc, sa, sw)
    y_ref = np.maximum((y_ref + res).astype(np.float32), 0)
    q_ref = oracle.quantize(y_ref, so, 8)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(W), a_nonneg=True)
    y = torch.empty(M, N, device=DEV)
    q = torch.empty(M, N, dtype=torch.int8, device=DEV)
    ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
    ep = ax.make_epilogue(_t(np.array([sa])), _t(np.array([sw])), y=y, ldy=N, workspace=ws,
                          residual=_t(res), ldr=N, relu=True, q_out=q, ldq=N,
                          d_scale_out=_t(np.array([so])), bits_out=8)
    ax.axq_lut_gemm_wp(_t(A), wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
    np.testing.assert_array_equal(q.cpu().numpy(), q_ref)


def test_p4w16_config2_err2000_full_batch(ax):
    """BJ configs[2]'s input and weights with a +-2000-error ACU (beyond int8 E): the whole
    128-image conv on the int16-E kernel, sampled images bit-exact."""
    from paper_2203_04071_b200.layers import ApproxConv2d
    c = datagen.config2()
    T = _lut("err2000")
    lut = ax.Lut(8, T)
    conv = ApproxConv2d(_t(c.W), None, lut, (1, 1), (1, 1), a_nonneg=True)
    assert conv.wp is not None
    y = conv(_t(c.x))
    assert ax.axq_last_path()[0] == "p4w16"
    torch.cuda.synchronize()
    sa = oracle.scale(oracle.amax(c.x), 8)
    qw, sw = oracle.quantize_tensor(c.W, 8)
    for img in (0, 99):
        acc = oracle.lut_conv2d(oracle.quantize(c.x[img:img + 1], sa, 8), qw, T, 8, (1, 1), (1, 1))
        np.testing.assert_array_equal(y[img:img + 1].cpu().numpy(), oracle.dequantize(acc, sa, sw, None, 1))


def test_p4w16_reduced_resnet_bit_exact(ax):
    """A whole (reduced) ResNet-50-shaped network with the +-2000-error ACU: ReLU-input convs on
    P4W16, the stem and fc on the gather kernel; scales and logits bit-exact vs the oracle."""
    from oracle import models
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs
    topo = dict(widths=(16, 32, 16, 32), blocks=(1, 2, 1, 1), stem_ch=16, num_classes=24)
    T = _lut("err2000")
    net = ApproxResNet(datagen.network_weights(layer_specs(**topo), 41), Lut(8, T), DEV, **topo)
    assert len(net.wp) > 0
    orc = models.ResNetOracle(T, 8, config=41, **topo)
    x = datagen.normal(41, 0, (3, 3, 40, 36))
    xd = _t(x)
    net.calibrate(xd[:2])
    scales = orc.calibrate(x[:2])
    for name, s in scales.items():
        assert net.s_act[net.slot[name]].item() == s, name
    np.testing.assert_array_equal(net.forward(xd).cpu().numpy(), orc.forward(x, scales))
