"""Pins of the paper's own quantizer in the oracle (NEXT-1, readings A30-A32):
per-output-channel weight scales and the 99.9 % histogram calib_max for activations.
CPU only.  Every pin compares against something other than the oracle's own formula:
SPEC's worked example, the exact sorted order statistic, the max calibrator as the p = 100 %
special case, the per-tensor quantizer as the equal-channel special case, fp64 closed forms."""
import numpy as np
import pytest

import oracle


def test_hist_spec_worked_example():
    # 1000 values 0.001*k, percentile 99.9 -> calib_max = 0.999 +- one bin width
    x = (np.arange(1, 1001, dtype=np.float64) * 0.001).astype(np.float32)
    cm, _ = oracle.hist_calib_max(x)
    w = np.float32(oracle.amax(x) / np.float32(oracle.HIST_BINS))
    assert abs(float(cm) - 0.999) <= float(w)


@pytest.mark.parametrize("seed,dist", [(1, "normal"), (2, "relu"), (3, "cauchy"), (4, "uniform")])
def test_hist_matches_sorted_order_statistic(seed, dist):
    # within one bin width of the exact order-statistic percentile computed by sorting
    rng = np.random.default_rng(seed)
    n = 20000
    x = {"normal": rng.standard_normal(n), "relu": np.maximum(rng.standard_normal(n), 0),
         "cauchy": rng.standard_cauchy(n), "uniform": rng.uniform(-3, 3, n)}[dist].astype(np.float32)
    cm, _ = oracle.hist_calib_max(x)
    a = np.sort(np.abs(x.astype(np.float64)))
    k = -(-999 * n // 1000)                       # ceil(0.999 n): the k-th smallest |x|
    v = a[k - 1]
    w = float(np.float32(oracle.amax(x) / np.float32(oracle.HIST_BINS)))
    assert v * (1 - 1e-6) <= float(cm) <= v + w * (1 + 1e-6)


def test_hist_p100_is_the_max_calibrator():
    rng = np.random.default_rng(5)
    for _ in range(5):
        x = (rng.standard_normal(3000) * rng.uniform(0.1, 10)).astype(np.float32)
        cm, b = oracle.hist_calib_max(x, percentile=(1, 1))
        assert b == oracle.HIST_BINS - 1 and cm == oracle.amax(x)
    assert oracle.hist_calib_max(np.zeros(7, np.float32))[0] == 0.0   # -> scale 1 (A4)
    assert oracle.scale(np.float32(0.0), 8) == 1.0


def test_hist_outliers_do_not_set_the_range():
    # the point of the percentile calibrator: a few huge outliers barely move calib_max
    rng = np.random.default_rng(6)
    x = rng.standard_normal(100000).astype(np.float32)
    x[:20] = 1000.0
    cm, _ = oracle.hist_calib_max(x)
    assert cm < 5.0 < oracle.amax(x)


def test_per_channel_roundtrip_and_reduction():
    rng = np.random.default_rng(7)
    W = (rng.standard_normal((16, 3, 3, 8)) * rng.uniform(0.01, 1, (16, 1, 1, 1))).astype(np.float32)
    s = oracle.scale_rows(oracle.amax_rows(W), 8)
    q = oracle.quantize_rows(W, s, 8)
    for c in range(16):
        # per-channel max-abs error <= scale_c / 2
        err = np.abs(q[c].astype(np.float64) * float(s[c]) - W[c].astype(np.float64)).max()
        assert err <= float(s[c]) / 2 * (1 + 1e-6)
        assert np.abs(q[c]).max() == 127                       # each channel uses its range
    # equal-amax channels reduce to the per-tensor quantizer bit for bit
    W2 = np.stack([W[0] / np.abs(W[0]).max()] * 4).astype(np.float32)
    s2 = oracle.scale_rows(oracle.amax_rows(W2), 8)
    q2 = oracle.quantize_rows(W2, s2, 8)
    qt, st = oracle.quantize_tensor(W2, 8)
    assert np.all(s2 == st) and np.array_equal(q2, qt)


def test_dequantize_per_channel():
    rng = np.random.default_rng(8)
    acc = rng.integers(-2**20, 2**20, (5, 6, 4, 4)).astype(np.int32)
    s_w = rng.uniform(1e-4, 1e-2, 6).astype(np.float32)
    b = rng.standard_normal(6).astype(np.float32)
    s_a = np.float32(0.037)
    y = oracle.dequantize_pc(acc, s_a, s_w, b, channel_axis=1)
    ref = acc.astype(np.float64) * (np.float64(s_a) * s_w.astype(np.float64))[None, :, None, None] + b[None, :, None, None]
    assert np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1e-3)) < 1e-6
    # constant channel scales reduce to the per-tensor form bit for bit
    yc = oracle.dequantize_pc(acc, s_a, np.full(6, s_w[0], np.float32), b, channel_axis=1)
    assert np.array_equal(yc, oracle.dequantize(acc, s_a, s_w[0], b, channel_axis=1))


def test_resnet_oracle_paper_quantizer_tracks_float():
    """Sanity (not a pin): with the exact multiplier the paper quantizer's network tracks the
    max-quantizer network within quantization error on a reduced ResNet."""
    import datagen
    from oracle import models
    lut = datagen.lut_exact(8)
    topo = dict(widths=(8, 16), blocks=(1, 1), stem_ch=8)
    x = datagen.config3_images(2)[:, :, :32, :32]
    a = models.ResNetOracle(lut, 8, quantizer="paper", **topo)
    m = models.ResNetOracle(lut, 8, quantizer="max", **topo)
    ya = a.forward(x, a.calibrate(x))
    ym = m.forward(x, m.calibrate(x))
    assert np.all(np.isfinite(ya))
    assert np.max(np.abs(ya - ym)) <= 0.2 * np.max(np.abs(ym)) + 1e-3
