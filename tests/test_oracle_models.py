"""Pins for the model-level oracles (oracle/models.py): ResNet-50-shaped forward (BJ configs[3])
and the LSTM (BJ configs[4]).  CPU only; reduced sizes."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import datagen
import oracle
from oracle import models

F32 = np.float32


# ----------------------------------------------------------------------------------------
# ResNet topology
# ----------------------------------------------------------------------------------------

def test_resnet50_topology_counts():
    L = models.resnet_layers()
    assert len(L) == 54                                   # 53 convs + fc
    assert sum(l["kind"] == "conv" for l in L) == 53
    assert models.resnet_macs(L) == 4_089_184_256        # the standard ResNet-50 v1.5 count
    params = sum(l["cout"] * l["cin"] * l.get("k", 1) ** 2 for l in L)
    assert params == 25_502_912     # torchvision resnet50: 25,557,032 - 53,120 BN - 1,000 bias


REDUCED = dict(widths=(4, 8, 8, 16), blocks=(1, 2, 1, 1), stem_ch=8, num_classes=10)


def _torch_quant(x, s, bits):
    qm = float((1 << (bits - 1)) - 1)
    t = torch.clamp(x / torch.tensor(s, dtype=torch.float32), -qm, qm)
    return torch.round(t)                                  # half to even (A1)


def _torch_scale(t, bits):
    """s = fl32(amax / qmax), amax == 0 -> 1 (A3/A4), written with torch ops."""
    a = t.abs().max().to(torch.float32)
    if float(a) == 0.0:
        return np.float32(1.0)
    return np.float32((a / torch.tensor(float((1 << (bits - 1)) - 1), dtype=torch.float32)).item())


def _torch_resnet(x, W, lut_bits, scales, widths, blocks, stem_ch, num_classes):
    """Independent re-implementation of the quantized network with the EXACT multiplier:
    every approximate conv is float64 torch conv2d on integer codes (exact), glue in fp32.
    scales=None: the calibration pass of reading A7' -- every approximate layer quantizes its
    input with that input's own per-tensor max scale, computed here from the tensor the layer
    actually receives; the scales are recorded in `calib` (returned with the logits)."""
    b = lut_bits
    calib = {}

    def wq(w):
        w = torch.from_numpy(w)
        s = oracle.scale(oracle.amax(w.numpy()), b)
        return _torch_quant(w, s, b).double(), s

    def in_scale(t, name):
        if scales is None:
            calib[name] = _torch_scale(t, b)
            return calib[name]
        return scales[name]

    def qconv(x32, name, stride, pad):
        s = in_scale(x32, name)
        qx = _torch_quant(x32, s, b).double()
        qw, sw = wq(W[name])
        acc = F.conv2d(qx, qw, stride=stride, padding=pad)
        sc = torch.tensor(np.float32(np.float32(s) * np.float32(sw)))
        return acc.float() * sc

    x = torch.from_numpy(x)
    y = torch.relu(qconv(x, "stem", 2, 3))
    y = F.max_pool2d(y, 3, 2, 1)
    for si in range(len(widths)):
        for bi in range(blocks[si]):
            p = "s%db%d" % (si, bi)
            s = (1 if si == 0 else 2) if bi == 0 else 1
            sc = qconv(y, p + ".down", s, 0) if bi == 0 else y
            t = torch.relu(qconv(y, p + ".c1", 1, 0))
            t = torch.relu(qconv(t, p + ".c2", s, 1))
            t = qconv(t, p + ".c3", 1, 0)
            y = torch.relu(t + sc)
    N, C, H, Wd = y.shape
    acc = torch.zeros(N, C, dtype=torch.float32)
    for h in range(H):
        for w in range(Wd):
            acc = acc + y[:, :, h, w]
    pooled = acc / torch.tensor(np.float32(H * Wd))
    s = in_scale(pooled, "fc")
    qp = _torch_quant(pooled, s, b).double()
    qw, sw = wq(W["fc"])
    acc = qp @ qw.t()
    sc = torch.tensor(np.float32(np.float32(s) * np.float32(sw)))
    logits = (acc.float() * sc + torch.from_numpy(W["fc.b"])).numpy()
    return (logits, calib) if scales is None else logits


def test_resnet_exact_lut_matches_independent_torch_network():
    """Exact multiplier: the oracle network == an independent torch network built on
    float64 conv2d of integer codes (bit for bit; same pinned fp32 glue)."""
    x = datagen.normal(31, 0, (2, 3, 32, 32))
    net = models.ResNetOracle(datagen.lut_exact(8), 8, config=31, **REDUCED)
    scales = net.calibrate(x)
    assert len(scales) == 1 + 5 * 2 + 3 * 3 + 1          # stem, blocks, fc (+ shared down)
    y = net.forward(x, scales)
    ref = _torch_resnet(x, net.W, 8, scales, **REDUCED)
    np.testing.assert_array_equal(y, ref)


@pytest.mark.parametrize("seed", [0, 1])
def test_resnet_calibration_scales_independent(seed):
    """Reading A7' pinned from outside the oracle: the independent torch network, calibrating
    every layer on the tensor it receives (stem: the image; block c1 and its projection: the
    block input, after the max-pool for the first block; c2 / c3: the ReLU'd outputs of c1 /
    c2; fc: the average-pooled features), gives exactly ResNetOracle.calibrate's scales -- a
    scale taken from the wrong tensor (pre-ReLU, pre-pool, the residual sum before its ReLU)
    would differ.  The calibrated logits agree too."""
    x = datagen.normal(33, seed, (2, 3, 32, 32))
    net = models.ResNetOracle(datagen.lut_exact(8), 8, config=31, **REDUCED)
    scales = net.calibrate(x)
    logits_t, calib = _torch_resnet(x, net.W, 8, None, **REDUCED)
    assert set(calib) == set(scales)
    for k in scales:
        assert np.float32(scales[k]) == calib[k], k
    logits_o, _ = net.run(x, None)
    np.testing.assert_array_equal(logits_o, logits_t)
    # the pin has teeth: the shared block-input scale differs from the pre-ReLU stem output's
    xt = torch.from_numpy(x)
    sw = oracle.scale(oracle.amax(net.W["stem"]), 8)
    acc = F.conv2d(_torch_quant(xt, calib["stem"], 8).double(),
                   _torch_quant(torch.from_numpy(net.W["stem"]), sw, 8).double(), stride=2, padding=3)
    pre = acc.float() * torch.tensor(np.float32(np.float32(calib["stem"]) * np.float32(sw)))
    assert _torch_scale(pre, 8) != calib["s0b0.c1"]


def test_resnet_calibrated_forward_is_static_fixed_point():
    """Forward with the scales calibrated on the same batch == the calibration run itself."""
    x = datagen.normal(31, 1, (2, 3, 32, 32))
    net = models.ResNetOracle(datagen.lut_randerr(8, 0, 2), 8, config=31, **REDUCED)
    logits_c, scales = net.run(x, None)
    np.testing.assert_array_equal(net.forward(x, scales), logits_c)


def test_maxpool_and_quantize_commute():
    """A17: pooling the codes == quantizing the pooled values (quantization is monotone)."""
    y = np.maximum(datagen.normal(32, 0, (2, 5, 11, 9)), 0)
    s = oracle.scale(oracle.amax(y), 8)
    a = models._maxpool(oracle.quantize(y, s, 8).astype(np.float32))
    b = oracle.quantize(models._maxpool(y), s, 8).astype(np.float32)
    np.testing.assert_array_equal(a, b)
    assert oracle.amax(models._maxpool(y)) == oracle.amax(y)   # every element is covered


# ----------------------------------------------------------------------------------------
# LSTM
# ----------------------------------------------------------------------------------------

def test_pinned_exp_within_2ulp_of_libm():
    x = np.linspace(-80, 80, 400001).astype(F32)
    e = models.pinned_exp(x).astype(np.float64)
    r = np.exp(x.astype(np.float64))
    ulp = np.abs(e - r) / np.spacing(r.astype(F32)).astype(np.float64)
    assert ulp.max() <= 2.0


def test_pinned_sigmoid_tanh_vs_float64():
    x = np.linspace(-30, 30, 100001).astype(F32)
    sg = models.pinned_sigmoid(x).astype(np.float64)
    th = models.pinned_tanh(x).astype(np.float64)
    x64 = x.astype(np.float64)
    assert np.abs(sg - 1 / (1 + np.exp(-x64))).max() <= 2e-7
    assert np.abs(th - np.tanh(x64)).max() <= 4e-7
    assert (models.pinned_tanh(-x) == -models.pinned_tanh(x)).all()       # odd
    assert models.pinned_sigmoid(np.float32(0)) == 0.5


@pytest.mark.parametrize("bits", [8])
def test_lstm_exact_lut_tracks_torch_lstm(bits):
    """Exact multiplier: the approximate LSTM tracks torch.nn.LSTM (float64, gate order
    i, f, g, o) within quantization error; a permuted gate order would not."""
    T, B, I, H = 6, 3, 16, 8
    c = datagen.config4(T=T, B=B, I=I, H=H)
    c.luts[bits] = datagen.lut_exact(bits)
    net = models.LstmOracle(c, bits)
    hs, cT = net.forward(net.calibrate())
    lstm = torch.nn.LSTM(I, H).double()
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.from_numpy(c.W_ih))
        lstm.weight_hh_l0.copy_(torch.from_numpy(c.W_hh))
        lstm.bias_ih_l0.copy_(torch.from_numpy(c.b_ih))
        lstm.bias_hh_l0.copy_(torch.from_numpy(c.b_hh))
        out, (hT, cT_ref) = lstm(torch.from_numpy(c.x).double())
    err = np.abs(hs - out.numpy()).max()
    assert err < 2e-3, err
    # gate-order sensitivity: swapping the f and g blocks of the reference changes it a lot
    with torch.no_grad():
        perm = torch.cat([torch.arange(0, H), torch.arange(2 * H, 3 * H), torch.arange(H, 2 * H),
                          torch.arange(3 * H, 4 * H)])
        lstm.weight_ih_l0.copy_(torch.from_numpy(c.W_ih)[perm])
        lstm.weight_hh_l0.copy_(torch.from_numpy(c.W_hh)[perm])
        lstm.bias_ih_l0.copy_(torch.from_numpy(c.b_ih)[perm])
        lstm.bias_hh_l0.copy_(torch.from_numpy(c.b_hh)[perm])
        out2, _ = lstm(torch.from_numpy(c.x).double())
    assert np.abs(hs - out2.numpy()).max() > 10 * err


def _torch_lstm_calib(c, bits):
    """Reading A7' for c4 pinned from outside the oracle: a float64 torch LSTM with the exact
    multiplier whose every quantization is dynamic (x: one per-tensor max over all x_t; h_{t-1}:
    its own max, h_{-1} = 0 -> scale 1), gates i, f, g, o through torch's own sigmoid / tanh.
    Returns (s_x, s_h = scale of max_t amax(h_t), amax(h_T) only)."""
    T, B, I = c.x.shape
    H = c.W_hh.shape[1]
    x = torch.from_numpy(c.x)
    s_x = _torch_scale(x, bits)
    qx = _torch_quant(x.reshape(T * B, I), s_x, bits).double()
    sw_ih = _torch_scale(torch.from_numpy(c.W_ih), bits)
    sw_hh = _torch_scale(torch.from_numpy(c.W_hh), bits)
    qw_ih = _torch_quant(torch.from_numpy(c.W_ih), sw_ih, bits).double()
    qw_hh = _torch_quant(torch.from_numpy(c.W_hh), sw_hh, bits).double()
    gih = (qx @ qw_ih.t()) * float(s_x) * float(sw_ih) + torch.from_numpy(c.b_ih).double()
    gih = gih.reshape(T, B, 4 * H)
    h = torch.zeros(B, H, dtype=torch.float64)
    cs = torch.zeros(B, H, dtype=torch.float64)
    amax_h = 0.0
    for t in range(T):
        s_h = _torch_scale(h.float(), bits)
        g = gih[t] + (_torch_quant(h.float(), s_h, bits).double() @ qw_hh.t()) * float(s_h) * float(sw_hh) \
            + torch.from_numpy(c.b_hh).double()
        i_, f_ = torch.sigmoid(g[:, :H]), torch.sigmoid(g[:, H:2 * H])
        g_, o_ = torch.tanh(g[:, 2 * H:3 * H]), torch.sigmoid(g[:, 3 * H:])
        cs = f_ * cs + i_ * g_
        h = o_ * torch.tanh(cs)
        amax_h = max(amax_h, float(h.abs().max()))
    qm = float((1 << (bits - 1)) - 1)
    return s_x, amax_h / qm, float(h.abs().max()) / qm


def test_lstm_calibration_scales_independent():
    """s_x is exact; s_h agrees with the torch recomputation to the fp32 / transcendental
    rounding of the two sides (1e-5 relative), while the plausible wrong reading -- the scale
    of the last hidden state only -- is far off."""
    c = datagen.config4(T=12, B=3, I=16, H=8)
    c.luts[8] = datagen.lut_exact(8)
    net = models.LstmOracle(c, 8)
    s_x, s_h = net.calibrate()
    t_x, t_h, t_last = _torch_lstm_calib(c, 8)
    assert np.float32(s_x) == t_x
    assert abs(float(s_h) - t_h) <= 1e-5 * t_h
    assert abs(t_last - t_h) > 1e-3 * t_h


def test_lstm_calibration_scales():
    c = datagen.config4(T=4, B=2, I=16, H=8)
    net = models.LstmOracle(c, 8)
    s_x, s_h = net.calibrate()
    assert s_x == oracle.scale(oracle.amax(c.x), 8)
    hs, _, _ = net.run(None)
    assert s_h == oracle.scale(oracle.amax(hs), 8)
    assert 0 < s_h <= 1.0 / 127 + 1e-9                   # |h| < 1
