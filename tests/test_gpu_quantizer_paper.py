"""GPU parity of the paper's own quantizer (NEXT-1, readings A30-A32) against the
oracle: per-channel weight scales, the 99.9 % histogram calib_max, the per-channel dequantizing
epilogue on every kernel family, the fp32 maxpool of the calibration pass, and a reduced ResNet
calibrated and run with the paper quantizer.  Everything is compared bit for bit."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import models

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def ax():
    from paper_2203_04071_b200 import _lib
    _lib.load()
    return _lib


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("shape", [(64, 64, 3, 3), (1000, 2048), (7, 5), (256, 64, 1, 1)])
@pytest.mark.parametrize("bits", [8, 4])
def test_per_channel_weights(ax, shape, bits):
    rng = np.random.default_rng(sum(shape) + bits)
    W = (rng.standard_normal(shape) * rng.uniform(0.01, 2, (shape[0],) + (1,) * (len(shape) - 1))).astype(np.float32)
    W[1] = 0.0                                              # an all-zero channel: scale 1 (A4)
    a_ref = oracle.amax_rows(W)
    s_ref = oracle.scale_rows(a_ref, bits)
    q_ref = oracle.quantize_rows(W, s_ref, bits)
    dW = _t(W)
    a = torch.empty(shape[0], device=DEV)
    s = torch.empty(shape[0], device=DEV)
    q = torch.empty(shape, dtype=torch.int8, device=DEV)
    ax.axq_amax_rows(dW, a)
    ax.axq_scale_vec(a, bits, s)
    ax.axq_quantize_rows(dW, s, bits, q)
    np.testing.assert_array_equal(a.cpu().numpy(), a_ref)
    np.testing.assert_array_equal(s.cpu().numpy(), s_ref)
    np.testing.assert_array_equal(q.cpu().numpy(), q_ref)


@pytest.mark.parametrize("case", ["normal", "relu", "cauchy", "tiny", "zeros", "c2"])
def test_histogram_calib_max(ax, case):
    rng = np.random.default_rng(11)
    x = {"normal": lambda: rng.standard_normal(100003),
         "relu": lambda: np.maximum(rng.standard_normal(77777), 0),
         "cauchy": lambda: rng.standard_cauchy(50000),
         "tiny": lambda: np.array([0.5, -0.25, 3.0]),
         "zeros": lambda: np.zeros(1000),
         "c2": lambda: datagen.config2().x}[case]().astype(np.float32)
    cm_ref, _ = oracle.hist_calib_max(x)
    for bits in (8, 6):
        s_ref = oracle.scale(cm_ref, bits)
        dx = _t(x)
        amax = torch.empty(1, device=DEV)
        hist = torch.empty(ax.HIST_BINS, dtype=torch.int32, device=DEV)
        cm = torch.empty(1, device=DEV)
        s = torch.empty(1, device=DEV)
        ax.axq_amax(dx, amax)
        ax.axq_calib_histogram(dx, amax, hist)
        ax.axq_calib_percentile(hist, x.size, amax, bits, d_calib_max=cm, d_scale=s)
        assert cm.item() == float(cm_ref) and s.item() == float(s_ref)
        assert int(hist.sum().item()) == (x.size if oracle.amax(x) > 0 else 0)
    # p = 100 % reduces to the max calibrator on the device too
    ax.axq_calib_percentile(hist, x.size, amax, 8, d_calib_max=cm, percentile=(1, 1))
    assert cm.item() == float(oracle.amax(x))


def _pc_case(M, N, K, seed):
    rng = np.random.default_rng(seed)
    A = datagen.random_int8(seed, (M, K))
    W = datagen.random_int8(seed + 1, (N, K))
    s_w = rng.uniform(1e-4, 3e-2, N).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    return A, W, s_w, b


@pytest.mark.parametrize("M,N,K", [(300, 40, 96), (2048, 64, 256), (8, 1000, 2048)])
@pytest.mark.parametrize("kernel", ["v1", "p4", "p4w"])
def test_gemm_per_channel_epilogue(ax, M, N, K, kernel):
    A, W, s_w, b = _pc_case(M, N, K, M + N)
    T = datagen.lut_randerr(8, 0, 2)
    s_a = np.float32(0.0123)
    ref = oracle.dequantize_pc(oracle.lut_gemm(A, W, T, 8), s_a, s_w, b)
    lut = ax.Lut(8, T)
    y = torch.empty(M, N, device=DEV)
    ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
    sa = torch.tensor([s_a], device=DEV)
    ones = torch.ones(1, device=DEV)
    db, dsw = _t(b), _t(s_w)          # the epilogue struct holds raw pointers: keep them alive
    ep = ax.make_epilogue(sa, ones, bias=db, y=y, ldy=N, workspace=ws, d_scale_w_ch=dsw)
    if kernel == "v1":
        ax.axq_lut_gemm_ep(_t(A), _t(W), lut, ep)
    else:
        prev = ax.axq_wpack_kernel(1 if kernel == "p4" else 3)
        try:
            wp = ax.WPack(lut, _t(W))
            ax.axq_lut_gemm_wp(_t(A), wp, ep)
        finally:
            ax.axq_wpack_kernel(prev)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


def test_conv_per_channel_nchw_epilogue(ax):
    rng = np.random.default_rng(21)
    X = datagen.random_int8(70, (2, 32, 9, 11))
    Wt = datagen.random_int8(71, (48, 32, 3, 3))
    T = datagen.lut_randerr(8, 0, 2)
    s_w = rng.uniform(1e-4, 3e-2, 48).astype(np.float32)
    s_a = np.float32(0.02)
    ref = oracle.dequantize_pc(oracle.lut_conv2d(X, Wt, T, 8, (1, 1), (1, 1)), s_a, s_w, None, channel_axis=1)
    lut = ax.Lut(8, T)
    d = ax.conv_desc(2, 9, 11, 32, 48, 3, 3, (1, 1), (1, 1))
    y = torch.empty(2, 48, 9, 11, device=DEV)
    ws = torch.zeros(2 * 48 * 99, dtype=torch.int32, device=DEV)
    dsa, dones, dsw = torch.tensor([s_a], device=DEV), torch.ones(1, device=DEV), _t(s_w)
    ep = ax.make_epilogue(dsa, dones, y=y, workspace=ws, d_scale_w_ch=dsw)
    wp = ax.WPack(lut, _t(Wt.transpose(0, 2, 3, 1)).reshape(48, -1).contiguous())
    ax.axq_lut_conv2d_wp(d, _t(X.transpose(0, 2, 3, 1)), wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


def test_maxpool_f32(ax):
    rng = np.random.default_rng(31)
    x = rng.standard_normal((3, 16, 13, 11)).astype(np.float32)
    ref = models._maxpool(x)                                 # NCHW oracle glue
    dx = _t(x.transpose(0, 2, 3, 1))
    Ho, Wo = ref.shape[2:]
    y = torch.empty(3, Ho, Wo, 16, device=DEV)
    ax.axq_maxpool2d_nhwc_f32(dx, 3, 3, 2, 1, y)
    np.testing.assert_array_equal(y.cpu().numpy().transpose(0, 3, 1, 2), ref)


@pytest.mark.parametrize("bits", [8, 6])
def test_resnet_reduced_paper_quantizer_bit_exact(bits):
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs
    topo = dict(widths=(16, 32, 16, 32), blocks=(1, 2, 1, 1), stem_ch=16, num_classes=24)
    lut = datagen.lut_randerr(bits, 3, 60 + bits)
    x = datagen.normal(34, bits, (3, 3, 40, 36))
    W = datagen.network_weights(layer_specs(**topo), 34)
    net = ApproxResNet(W, Lut(bits, lut), DEV, quantizer="paper", **topo)
    orc = models.ResNetOracle(lut, bits, config=34, quantizer="paper", **topo)
    xd = torch.from_numpy(x).to(DEV)
    net.calibrate(xd[:2])
    scales = orc.calibrate(x[:2])
    for name, s in scales.items():
        assert net.s_act[net.slot[name]].item() == s, name
    y = net.forward(xd).cpu().numpy()
    ref = orc.forward(x, scales)
    np.testing.assert_array_equal(y, ref)
