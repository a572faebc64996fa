"""Oracle model drivers -- TEST INFRASTRUCTURE (see oracle/__init__.py).

Plain numpy composition of the pinned C primitives (amax, scale, quantize, LUT-conv, LUT-GEMM,
dequantize) with the model glue written out in fp32 numpy operations (each numpy float32
operation is one IEEE-rounded op, no FMA contraction), in the order DESIGN.md A16-A18 fixes.

* ResNet-50-shaped forward, BASELINE.json configs[3] (A16 topology, A17 glue, A7' calibration).
* LSTM with approximate gate GEMMs, BASELINE.json configs[4] (A18).

Parity status: these drivers are compositions of primitives that tests/test_oracle_pins.py
pins; the model level itself is "parity unpinned" by the paper (it prints no model outputs and
Table II needs datasets / trained weights that are absent).  tests/test_oracle_models.py pins
what can be pinned: the topology by its layer count (54) and MAC total (4,089,184,256 per
224x224 image), each approximate layer against the pinned conv, the pinned exp / sigmoid / tanh
against float64 libm within 2 ulp, and, with the exact multiplier, the approximate network
against an independent float64 torch re-implementation within quantization error.
"""
from __future__ import annotations

import numpy as np

import datagen

from . import (amax, amax_rows, dequantize, dequantize_pc, hist_calib_max, lut_conv2d, lut_gemm,
               quantize, quantize_rows, scale, scale_rows)

F32 = np.float32


def register(L) -> None:
    """No extra C entry points: the model drivers compose the primitives."""
    return None


# =========================================================================================
# ResNet-50-shaped network (A16): stem 7x7/2 p3 + ReLU, maxpool 3x3/2 p1, bottleneck stages
# (3,64) (4,128) (6,256) (3,512) with expansion 4, stride on the 3x3 conv (v1.5), projection
# shortcut on each stage's first block, out = ReLU(main + shortcut), global avgpool, fc.
# No BatchNorm.  Weights: Kaiming-normal fan_out (convs), fan_in (fc), bias U(+-1/sqrt(in)).
# =========================================================================================

def resnet_layers(widths=(64, 128, 256, 512), blocks=(3, 4, 6, 3), in_ch=3, stem_ch=64,
                  num_classes=1000, expansion=4):
    """Layer list in forward order: dicts with name, kind, shapes, stride, pad, weight idx."""
    L = []
    idx = 1

    def conv(name, cout, cin, k, stride, pad):
        nonlocal idx
        L.append(dict(name=name, kind="conv", cout=cout, cin=cin, k=k, stride=stride, pad=pad,
                      widx=idx))
        idx += 1

    conv("stem", stem_ch, in_ch, 7, 2, 3)
    cin = stem_ch
    for si, (w, nb) in enumerate(zip(widths, blocks)):
        for bi in range(nb):
            s = (1 if si == 0 else 2) if bi == 0 else 1
            conv("s%db%d.c1" % (si, bi), w, cin, 1, 1, 0)
            conv("s%db%d.c2" % (si, bi), w, w, 3, s, 1)
            conv("s%db%d.c3" % (si, bi), w * expansion, w, 1, 1, 0)
            if bi == 0:
                conv("s%db%d.down" % (si, bi), w * expansion, cin, 1, s, 0)
            cin = w * expansion
    L.append(dict(name="fc", kind="fc", cout=num_classes, cin=cin, widx=idx, bidx=idx + 1))
    return L


def resnet_weights(layers, config=3):
    W = {}
    for l in layers:
        if l["kind"] == "conv":
            W[l["name"]] = datagen.kaiming_conv(config, l["widx"], l["cout"], l["cin"], l["k"], l["k"])
        else:
            W["fc"] = datagen.kaiming_fc(config, l["widx"], l["cout"], l["cin"])
            W["fc.b"] = datagen.fc_bias(config, l["bidx"], l["cout"], l["cin"])
    return W


def _deq(acc, sa, sw):
    """v = fl(fl((float)acc) * fl(sa*sw)) elementwise (A14)."""
    sc = F32(F32(sa) * F32(sw))
    return acc.astype(F32) * sc


def _relu(v):
    return np.where(v > 0, v, F32(0)).astype(F32)


def _maxpool(x, k=3, s=2, p=1):
    """Max over the window's in-image taps (out-of-image taps ignored, A17)."""
    N, C, H, W = x.shape
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    y = np.full((N, C, Ho, Wo), -np.inf, F32)
    for r in range(k):
        for c in range(k):
            for ho in range(Ho):
                hi = ho * s - p + r
                if hi < 0 or hi >= H:
                    continue
                wi = np.arange(Wo) * s - p + c
                ok = (wi >= 0) & (wi < W)
                y[:, :, ho, ok] = np.maximum(y[:, :, ho, ok], x[:, :, hi, wi[ok]])
    return y


def _avgpool(x):
    """Sequential fp32 sum over (h, w) in row-major order, then one division by H*W (A17)."""
    N, C, H, W = x.shape
    acc = np.zeros((N, C), F32)
    for h in range(H):
        for w in range(W):
            acc = (acc + x[:, :, h, w]).astype(F32)
    return (acc / F32(H * W)).astype(F32)


class ResNetOracle:
    """Approximate ResNet forward on NCHW fp32 numpy tensors.

    calibrate(x): the approximate forward with every layer's input scale computed from that
    input tensor (dynamic per-tensor max, P:94 / BJ "per-layer max calibration"); returns the
    per-layer activation scales (reading A7').  forward(x, scales): the same network with those
    static scales (inputs beyond the calibrated range clamp, A2)."""

    def __init__(self, lut, bits=8, config=3, quantizer="max", **topo):
        """quantizer "max": per-tensor max calibration of weights and activations (BJ north
        star).  "paper": the paper's own quantizer (NEXT-1) -- per-output-channel
        weight scales (A31) and 99.9 % histogram calib_max for activations (A30)."""
        self.layers = resnet_layers(**topo)
        self.W = resnet_weights(self.layers, config)
        self.lut, self.bits = lut, bits
        self.quantizer = quantizer
        self.wq = {}
        for l in self.layers:
            w = self.W[l["name"]]
            if quantizer == "paper":
                s = scale_rows(amax_rows(w), bits)
                self.wq[l["name"]] = (quantize_rows(w, s, bits), s)
            else:
                s = scale(amax(w), bits)
                self.wq[l["name"]] = (quantize(w, s, bits), s)

    def _scale(self, name, x, scales, calib):
        if calib:
            if self.quantizer == "paper":
                scales[name] = scale(hist_calib_max(x)[0], self.bits)
            else:
                scales[name] = scale(amax(x), self.bits)
        return scales[name]

    def _deq_layer(self, acc, sa, sw, bias=None, channel_axis=1):
        if self.quantizer == "paper":
            return dequantize_pc(acc, sa, sw, bias, channel_axis)
        if bias is None:
            return _deq(acc, sa, sw)
        return dequantize(acc, sa, sw, bias, channel_axis)

    def _conv(self, name, xq, sa, layer):
        q, sw = self.wq[name]
        acc = lut_conv2d(xq, q, self.lut, self.bits, (layer["stride"],) * 2, (layer["pad"],) * 2)
        return self._deq_layer(acc, sa, sw)

    def run(self, x, scales=None, trace=None):
        calib = scales is None
        scales = {} if calib else scales
        b = self.bits
        L = {l["name"]: l for l in self.layers}
        # stem: quantize input, conv, ReLU
        s = self._scale("stem", x, scales, calib)
        y = _relu(self._conv("stem", quantize(x, s, b), s, L["stem"]))
        # maxpool; its output is the first block's input
        y = _maxpool(y)
        names = [l["name"] for l in self.layers if l["kind"] == "conv"]
        blocks = sorted({n.rsplit(".", 1)[0] for n in names if n != "stem"},
                        key=lambda n: names.index(n + ".c1"))
        h = y
        for blk in blocks:
            s_in = self._scale(blk + ".c1", h, scales, calib)
            hq = quantize(h, s_in, b)
            if blk + ".down" in L:
                scales[blk + ".down"] = s_in          # shared input -> shared scale (A17)
                sc = self._conv(blk + ".down", hq, s_in, L[blk + ".down"])
            else:
                sc = h
            t = _relu(self._conv(blk + ".c1", hq, s_in, L[blk + ".c1"]))
            s2 = self._scale(blk + ".c2", t, scales, calib)
            t = _relu(self._conv(blk + ".c2", quantize(t, s2, b), s2, L[blk + ".c2"]))
            s3 = self._scale(blk + ".c3", t, scales, calib)
            t = self._conv(blk + ".c3", quantize(t, s3, b), s3, L[blk + ".c3"])
            h = _relu((t + sc).astype(F32))
            if trace is not None:
                trace[blk] = h
        p = _avgpool(h)
        s_fc = self._scale("fc", p, scales, calib)
        q, sw = self.wq["fc"]
        acc = lut_gemm(quantize(p, s_fc, b), q, self.lut, b)
        logits = self._deq_layer(acc, s_fc, sw, self.W["fc.b"], -1)
        return logits, scales

    def calibrate(self, x):
        return self.run(x, None)[1]

    def forward(self, x, scales, trace=None):
        return self.run(x, scales, trace)[0]


def resnet_macs(layers, H=224, W=224):
    """Lookups (MACs) per image of the approximate layers (padded taps included)."""
    tot = 0
    h, w = H, W
    shapes = {}
    for l in layers:
        if l["kind"] == "fc":
            tot += l["cout"] * l["cin"]
            continue
        if l["name"] == "stem":
            hi, wi = h, w
        elif l["name"].endswith(".c1"):
            hi, wi = shapes["block_in"]
            shapes["this_block_in"] = (hi, wi)
        elif l["name"].endswith(".down"):
            hi, wi = shapes["this_block_in"]
        elif l["name"].endswith(".c2"):
            hi, wi = shapes["c1"]
        else:
            hi, wi = shapes["c2"]
        ho = (hi + 2 * l["pad"] - l["k"]) // l["stride"] + 1
        wo = (wi + 2 * l["pad"] - l["k"]) // l["stride"] + 1
        tot += ho * wo * l["cout"] * l["cin"] * l["k"] * l["k"]
        if l["name"] == "stem":
            shapes["block_in"] = ((ho + 2 - 3) // 2 + 1, (wo + 2 - 3) // 2 + 1)
        elif l["name"].endswith(".c1"):
            shapes["c1"] = (ho, wo)
        elif l["name"].endswith(".c2"):
            shapes["c2"] = (ho, wo)
        elif l["name"].endswith(".c3"):
            shapes["block_in"] = (ho, wo)
    return tot


# =========================================================================================
# LSTM (A18).  gates = fl(fl(ih_deq + b_ih) + fl(hh_deq + b_hh)), order i, f, g, o;
# c = fl(fl(f*c) + fl(i*g)); h = fl(o * tanh(c)); sigma / tanh through the pinned exp E.
# =========================================================================================

_LOG2E = F32(1.4426950408889634)
_C1 = F32(355.0 / 512.0)
_C2 = F32(0.6931471805599453 - 355.0 / 512.0)
_COEF = [F32(1.0 / f) for f in (5040.0, 720.0, 120.0, 24.0, 6.0, 2.0, 1.0, 1.0)]


def pinned_exp(x):
    """E(x) of A18: clamp to [-80, 80]; n = rint(x*log2e); r = (x - n*355/512) - n*c2;
    degree-7 Taylor polynomial (Horner, fp32 coefficients 1/k!); times 2^n (exact)."""
    x = np.clip(np.asarray(x, F32), F32(-80), F32(80)).astype(F32)
    n = np.rint((x * _LOG2E).astype(F32)).astype(F32)
    r = ((x - (n * _C1).astype(F32)).astype(F32) - (n * _C2).astype(F32)).astype(F32)
    p = np.full(x.shape, _COEF[0], F32)
    for c in _COEF[1:]:
        p = ((p * r).astype(F32) + c).astype(F32)
    two_n = ((n.astype(np.int32) + 127) << 23).astype(np.int32).view(F32)
    return (p * two_n).astype(F32)


def pinned_sigmoid(x):
    x = np.asarray(x, F32)
    return (F32(1) / (F32(1) + pinned_exp(-x)).astype(F32)).astype(F32)


def pinned_tanh(x):
    x = np.asarray(x, F32)
    e = pinned_exp((F32(-2) * np.abs(x)).astype(F32))
    t = ((F32(1) - e).astype(F32) / (F32(1) + e).astype(F32)).astype(F32)
    return np.copysign(t, x).astype(F32)


class LstmOracle:
    """One-layer LSTM whose ih and hh Linears are approximate (two separately quantized
    layers, A18).  calibrate(): every quantization dynamic (per-tensor max of that tensor);
    returns (s_x, s_h) = (scale of amax over all x_t, scale of max_t amax(h_t)) (A7').
    forward(): static s_x for the hoisted input projection and s_h for every h_{t-1}."""

    def __init__(self, case, bits):
        self.c = case
        self.bits = bits
        self.lut = case.luts[bits]
        b = bits
        self.sw_ih = scale(amax(case.W_ih), b)
        self.sw_hh = scale(amax(case.W_hh), b)
        self.qw_ih = quantize(case.W_ih, self.sw_ih, b)
        self.qw_hh = quantize(case.W_hh, self.sw_hh, b)

    def run(self, static=None):
        c, b = self.c, self.bits
        T, B, I = c.x.shape
        H = c.W_hh.shape[1]
        x2 = c.x.reshape(T * B, I)
        s_x = scale(amax(x2), b) if static is None else static[0]
        acc = lut_gemm(quantize(x2, s_x, b), self.qw_ih, self.lut, b)
        gih = dequantize(acc, s_x, self.sw_ih, c.b_ih).reshape(T, B, 4 * H)
        h = np.zeros((B, H), F32)
        cs = np.zeros((B, H), F32)
        hs = np.empty((T, B, H), F32)
        amax_h = F32(0)
        for t in range(T):
            s_h = scale(amax(h), b) if static is None else static[1]
            acc = lut_gemm(quantize(h, s_h, b), self.qw_hh, self.lut, b)
            ghh = dequantize(acc, s_h, self.sw_hh, c.b_hh)
            g = (gih[t] + ghh).astype(F32)
            i_ = pinned_sigmoid(g[:, 0:H])
            f_ = pinned_sigmoid(g[:, H:2 * H])
            g_ = pinned_tanh(g[:, 2 * H:3 * H])
            o_ = pinned_sigmoid(g[:, 3 * H:4 * H])
            cs = ((f_ * cs).astype(F32) + (i_ * g_).astype(F32)).astype(F32)
            h = (o_ * pinned_tanh(cs)).astype(F32)
            hs[t] = h
            amax_h = max(amax_h, amax(h))
        return hs, cs, (s_x, scale(amax_h, b))

    def calibrate(self):
        return self.run(None)[2]

    def forward(self, scales):
        hs, cs, _ = self.run(scales)
        return hs, cs
