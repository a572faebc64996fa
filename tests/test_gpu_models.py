"""GPU parity for the model drivers (a7 rows): ResNet-50-shaped forward (BJ configs[3]) and the
LSTM (BJ configs[4]) on the C ABI against the oracle models.  Everything the GPU computes is
pinned fp32 glue around exact integer LUT sums, so logits / hidden states are compared bit for
bit (the 1e-6 relative bound is asserted first)."""
import numpy as np
import pytest
import torch

import datagen
from oracle import models

pytestmark = pytest.mark.gpu
DEV = "cuda"

REDUCED = dict(widths=(16, 32, 16, 32), blocks=(1, 2, 1, 1), stem_ch=16, num_classes=24)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float((np.abs(a - b) / np.maximum(np.abs(b), 1e-30)).max())


def _gpu_resnet(lut_np, bits, config, **topo):
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs
    W = datagen.network_weights(layer_specs(**topo), config)
    return ApproxResNet(W, Lut(bits, lut_np), DEV, **topo)


@pytest.mark.parametrize("bits", [8, 6])
def test_resnet_reduced_bit_exact(bits):
    lut = datagen.lut_randerr(bits, 3, 50 + bits)
    x = datagen.normal(33, bits, (3, 3, 40, 36))
    net = _gpu_resnet(lut, bits, 33, **REDUCED)
    orc = models.ResNetOracle(lut, bits, config=33, **REDUCED)
    xd = torch.from_numpy(x).to(DEV)
    net.calibrate(xd[:2])
    scales = orc.calibrate(x[:2])
    for name, s in scales.items():
        assert net.s_act[net.slot[name]].item() == s, name
    y = net.forward(xd).cpu().numpy()
    ref = orc.forward(x, scales)
    assert _rel(y, ref) <= 1e-6
    np.testing.assert_array_equal(y, ref)


def test_resnet50_config3_full_batch_sampled():
    """BJ configs[3] at full size: calibrate on images 0-7, forward all 256 images on one GPU
    (the bench launch configuration); the oracle recomputes five images spread over the batch
    (different row tiles, stream-K pieces and TMA boxes of every layer)."""
    lut = datagen.lut_randerr(8, 0, 2)                       # A15: c0's table
    net = _gpu_resnet(lut, 8, 3)
    orc = models.ResNetOracle(lut, 8, config=3)
    x = datagen.config3_images(256)
    xd = torch.from_numpy(x).to(DEV)
    net.calibrate(xd[:8])
    scales = orc.calibrate(x[:8])
    for name, s in scales.items():
        assert net.s_act[net.slot[name]].item() == s, name
    y = net.forward(xd).cpu().numpy()
    for i in (0, 37, 128, 201, 255):
        ref = orc.forward(x[i:i + 1], scales)
        assert _rel(y[i:i + 1], ref) <= 1e-6
        np.testing.assert_array_equal(y[i:i + 1], ref)


def test_resnet50_config3_per_rank_batch_32():
    """The per-rank batch the N = 8 bench runs (256 / 8 = 32 images, images 32-63 = rank 1's
    shard): its layers pick different tile shapes and stream-K plans than the 256-image batch.
    Calibration on images 0-7 as in the bench; the oracle recomputes three images."""
    lut = datagen.lut_randerr(8, 0, 2)
    net = _gpu_resnet(lut, 8, 3)
    orc = models.ResNetOracle(lut, 8, config=3)
    xc = datagen.config3_images(8)
    x = datagen.config3_images(32, start=32)
    net.calibrate(torch.from_numpy(xc).to(DEV))
    scales = orc.calibrate(xc)
    y = net.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    for i in (0, 13, 31):
        np.testing.assert_array_equal(y[i:i + 1], orc.forward(x[i:i + 1], scales))


@pytest.mark.parametrize("bits", [4, 6, 8])
def test_lstm_reduced_bit_exact(bits):
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.lstm import ApproxLSTM
    c = datagen.config4(T=7, B=5, I=48, H=40)
    net = ApproxLSTM(c.W_ih, c.W_hh, c.b_ih, c.b_hh, Lut(bits, c.luts[bits]), DEV)
    orc = models.LstmOracle(c, bits)
    xd = torch.from_numpy(c.x).to(DEV)
    net.calibrate(xd)
    s_x, s_h = orc.calibrate()
    assert net.s_x.item() == s_x and net.s_h.item() == s_h
    hs, cT = net.forward(xd)
    hs_ref, c_ref = orc.forward((s_x, s_h))
    np.testing.assert_array_equal(hs.cpu().numpy(), hs_ref)
    np.testing.assert_array_equal(cT.cpu().numpy(), c_ref)


@pytest.mark.parametrize("bits", [4, 6, 8])
def test_lstm_config4_full(bits):
    """BJ configs[4] at full size (input 512, hidden 1024, seq 128, batch 64)."""
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.lstm import ApproxLSTM
    c = datagen.config4()
    net = ApproxLSTM(c.W_ih, c.W_hh, c.b_ih, c.b_hh, Lut(bits, c.luts[bits]), DEV)
    orc = models.LstmOracle(c, bits)
    xd = torch.from_numpy(c.x).to(DEV)
    net.calibrate(xd)
    s_x, s_h = orc.calibrate()
    assert net.s_x.item() == s_x and net.s_h.item() == s_h
    hs, cT = net.forward(xd)
    hs_ref, c_ref = orc.forward((s_x, s_h))
    np.testing.assert_array_equal(hs.cpu().numpy(), hs_ref)
    np.testing.assert_array_equal(cT.cpu().numpy(), c_ref)


def test_lstm_cuda_graph_replay_matches_forward():
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.lstm import ApproxLSTM
    c = datagen.config4(T=9, B=4, I=64, H=48)
    net = ApproxLSTM(c.W_ih, c.W_hh, c.b_ih, c.b_hh, Lut(8, c.luts[8]), DEV)
    xd = torch.from_numpy(c.x).to(DEV)
    net.calibrate(xd)
    hs, cT = net.forward(xd)
    hs, cT = hs.clone(), cT.clone()
    replay = net.capture(xd)
    hs2, cT2 = replay()
    torch.cuda.synchronize()
    assert torch.equal(hs, hs2) and torch.equal(cT, cT2)


@pytest.mark.parametrize("bits", [4, 8])
def test_lstm_persistent_matches_step_chain(bits):
    """The one-launch recurrence (axq_lstm_recurrent) is bit-identical to the per-step chain
    (LUT-GEMM + epilogue + cell launches), on a shape with a ragged batch row group."""
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.lstm import ApproxLSTM
    c = datagen.config4(T=9, B=40, I=64, H=96)
    net = ApproxLSTM(c.W_ih, c.W_hh, c.b_ih, c.b_hh, Lut(bits, c.luts[bits]), DEV)
    xd = torch.from_numpy(c.x).to(DEV)
    net.calibrate(xd)
    net.recurrent = "steps"
    hs1, c1 = (t.clone() for t in net.forward(xd))
    net.recurrent = "auto"
    hs2, c2 = net.forward(xd)
    assert net._persistent_ok
    torch.cuda.synchronize()
    assert torch.equal(hs1, hs2) and torch.equal(c1, c2)
    orc = models.LstmOracle(c, bits)
    s_x, s_h = orc.calibrate()
    hs_ref, c_ref = orc.forward((s_x, s_h))
    np.testing.assert_array_equal(hs2.cpu().numpy(), hs_ref)
    np.testing.assert_array_equal(c2.cpu().numpy(), c_ref)
