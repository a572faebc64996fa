"""Pins of the oracle's NEXT-4 STE backward (reading A36) against an independent
route -- torch autograd of the fake-quantized forward -- plus closed forms and brute force."""
import numpy as np
import pytest
import torch

import datagen
import oracle


def _operands(M, N, K, seed):
    x = datagen.normal(50 + seed, 1, (M, K))
    W = datagen.normal(50 + seed, 2, (N, K), 0.05)
    qa, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(W, 8)
    gy = datagen.normal(50 + seed, 3, (M, N))
    return x, W, qa, sa, qw, sw, gy


@pytest.mark.parametrize("M,N,K", [(5, 7, 3), (16, 33, 40), (64, 20, 128)])
def test_ste_matches_autograd_of_fake_quant_forward(M, N, K):
    """The STE treats quantizer + ACU as identity: the gradients are those of
    y = fq(qa) fq(qw)^T + b, which torch autograd computes by differentiating the forward."""
    x, W, qa, sa, qw, sw, gy = _operands(M, N, K, M)
    xf = torch.tensor(oracle.fake_quant(qa, sa), dtype=torch.float64, requires_grad=True)
    wf = torch.tensor(oracle.fake_quant(qw, sw), dtype=torch.float64, requires_grad=True)
    b = torch.zeros(N, dtype=torch.float64, requires_grad=True)
    y = torch.nn.functional.linear(xf, wf, b)
    y.backward(torch.tensor(gy, dtype=torch.float64))
    gx, gw, gb = oracle.ste_linear_backward(gy, qa, sa, qw, sw)
    np.testing.assert_allclose(gx, xf.grad.numpy().astype(np.float32), rtol=2e-7, atol=1e-9)
    np.testing.assert_allclose(gw, wf.grad.numpy().astype(np.float32), rtol=2e-7, atol=1e-9)
    np.testing.assert_allclose(gb, b.grad.numpy().astype(np.float32), rtol=2e-7, atol=1e-9)


def test_ste_clip_mask():
    """Inputs outside the calibrated clip range get no gradient; the others are unchanged."""
    M, N, K = 12, 9, 10
    x, W, qa, sa, qw, sw, gy = _operands(M, N, K, 7)
    clip_a = np.float32(np.quantile(np.abs(x), 0.7))
    clip_w = np.float32(np.quantile(np.abs(W), 0.5))
    gx0, gw0, gb0 = oracle.ste_linear_backward(gy, qa, sa, qw, sw)
    gx, gw, gb = oracle.ste_linear_backward(gy, qa, sa, qw, sw, x, clip_a, W, clip_w)
    out_a, out_w = np.abs(x) > clip_a, np.abs(W) > clip_w
    assert out_a.any() and (~out_a).any() and out_w.any()
    assert (gx[out_a] == 0).all() and (gw[out_w] == 0).all()
    np.testing.assert_array_equal(gx[~out_a], gx0[~out_a])
    np.testing.assert_array_equal(gw[~out_w], gw0[~out_w])
    np.testing.assert_array_equal(gb, gb0)


def test_ste_closed_form():
    """All-ones codes with scale 1: gw[n][k] = sum_m gy[m][n], gx[m][k] = sum_n gy[m][n]."""
    M, N, K = 6, 4, 5
    gy = np.arange(M * N, dtype=np.float32).reshape(M, N) - 7
    ones_a, ones_w = np.ones((M, K), np.int8), np.ones((N, K), np.int8)
    gx, gw, gb = oracle.ste_linear_backward(gy, ones_a, np.float32(1), ones_w, np.float32(1))
    np.testing.assert_array_equal(gx, np.repeat(gy.sum(1, keepdims=True), K, 1))
    np.testing.assert_array_equal(gw, np.repeat(gy.sum(0)[:, None], K, 1))
    np.testing.assert_array_equal(gb, gy.sum(0))


def test_ste_brute_force_tiny():
    M, N, K = 3, 2, 4
    x, W, qa, sa, qw, sw, gy = _operands(M, N, K, 3)
    gx, gw, gb = oracle.ste_linear_backward(gy, qa, sa, qw, sw)
    for m in range(M):
        for k in range(K):
            s = sum(float(gy[m, n]) * float(np.float32(sw) * np.float32(qw[n, k])) for n in range(N))
            assert gx[m, k] == np.float32(s)
    for n in range(N):
        for k in range(K):
            s = sum(float(gy[m, n]) * float(np.float32(sa) * np.float32(qa[m, k])) for m in range(M))
            assert gw[n, k] == np.float32(s)
        assert gb[n] == np.float32(sum(float(gy[m, n]) for m in range(M)))


@pytest.mark.parametrize("shape", [(2, 3, 7, 6, 4, 3, 3, 1, 1), (1, 5, 9, 8, 6, 3, 3, 2, 1),
                                   (2, 4, 5, 5, 3, 1, 1, 1, 0), (1, 2, 8, 7, 5, 5, 3, 2, 2)])
def test_ste_conv_matches_autograd(shape):
    """The conv STE backward equals torch autograd of conv2d on the fake-quantized operands."""
    N, C, H, W, K, R, S, st, pd = shape
    x = datagen.normal(70 + C, 1, (N, H, W, C))
    wt = datagen.normal(70 + C, 2, (K, R, S, C), 0.2)
    qx, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(wt, 8)
    Ho, Wo = (H + 2 * pd - R) // st + 1, (W + 2 * pd - S) // st + 1
    gy = datagen.normal(70 + C, 3, (N, Ho, Wo, K))
    xf = torch.tensor(oracle.fake_quant(qx, sa).transpose(0, 3, 1, 2), dtype=torch.float64, requires_grad=True)
    wf = torch.tensor(oracle.fake_quant(qw, sw).transpose(0, 3, 1, 2), dtype=torch.float64, requires_grad=True)
    b = torch.zeros(K, dtype=torch.float64, requires_grad=True)
    y = torch.nn.functional.conv2d(xf, wf, b, stride=st, padding=pd)
    y.backward(torch.tensor(gy.transpose(0, 3, 1, 2), dtype=torch.float64))
    gx, gw, gb = oracle.ste_conv2d_backward(gy, qx, sa, qw, sw, (st, st), (pd, pd))
    np.testing.assert_allclose(gx, xf.grad.numpy().transpose(0, 2, 3, 1).astype(np.float32), rtol=2e-7, atol=1e-9)
    np.testing.assert_allclose(gw, wf.grad.numpy().transpose(0, 2, 3, 1).astype(np.float32), rtol=2e-7, atol=1e-9)
    np.testing.assert_allclose(gb, b.grad.numpy().astype(np.float32), rtol=2e-7, atol=1e-9)


def test_ste_conv_1x1_equals_linear():
    """A 1x1 stride-1 conv is the linear layer over pixels: both STE backwards agree."""
    N, H, W, C, K = 2, 3, 4, 5, 6
    x = datagen.normal(80, 1, (N, H, W, C))
    wt = datagen.normal(80, 2, (K, 1, 1, C), 0.2)
    qx, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(wt, 8)
    gy = datagen.normal(80, 3, (N, H, W, K))
    gx, gw, gb = oracle.ste_conv2d_backward(gy, qx, sa, qw, sw)
    lx, lw, lb = oracle.ste_linear_backward(gy.reshape(-1, K), qx.reshape(-1, C), sa, qw.reshape(K, C), sw)
    np.testing.assert_allclose(gx.reshape(-1, C), lx, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(gw.reshape(K, C), lw, rtol=1e-6, atol=1e-9)
    np.testing.assert_array_equal(gb, lb)


@pytest.mark.parametrize("M,N,K", [(6, 5, 9), (17, 12, 33)])
def test_ste_per_channel_weights_match_autograd(M, N, K):
    """Per-output-channel weight scales and clips ("weight ranges are per channel"; the
    layers of the paper's quantizer, NEXT-1): the gradients are those of y = fq(qa) fq_ch(qw)^T
    with fq_ch(qw)[n] = fl32(s_w[n] * qw[n]) built here with torch, masked per row by
    |w[n][k]| <= clip_w[n]."""
    x = datagen.normal(80 + M, 1, (M, K))
    W = datagen.normal(80 + M, 2, (N, K), 0.05) * np.linspace(0.2, 3.0, N, dtype=np.float32)[:, None]
    qa, sa = oracle.quantize_tensor(x, 8)
    amax_ch = np.abs(W).max(axis=1).astype(np.float32)
    sw_ch = (amax_ch / np.float32(127)).astype(np.float32)
    qw = np.clip(np.rint(W / sw_ch[:, None]), -127, 127).astype(np.int8)
    gy = datagen.normal(80 + M, 3, (M, N))
    clip_w = (amax_ch * np.float32(0.6)).astype(np.float32)
    xf = torch.tensor(oracle.fake_quant(qa, sa), dtype=torch.float64, requires_grad=True)
    wf32 = torch.from_numpy(qw).float() * torch.from_numpy(sw_ch)[:, None]        # fl32 per row
    wf = wf32.double().requires_grad_(True)
    torch.nn.functional.linear(xf, wf).backward(torch.tensor(gy, dtype=torch.float64))
    gx, gw, gb = oracle.ste_linear_backward(gy, qa, sa, qw, sw_ch, w=W, clip_w=clip_w)
    np.testing.assert_allclose(gx, xf.grad.numpy().astype(np.float32), rtol=2e-7, atol=1e-9)
    keep = np.abs(W) <= clip_w[:, None]
    assert keep.any() and (~keep).any()
    ref_gw = np.where(keep, wf.grad.numpy(), 0.0).astype(np.float32)
    np.testing.assert_allclose(gw, ref_gw, rtol=2e-7, atol=1e-9)
    # a per-channel scale is not the per-tensor one: using s_w[0] for every row changes gx
    gx1, _, _ = oracle.ste_linear_backward(gy, qa, sa, qw, sw_ch[0])
    assert np.abs(gx1 - gx).max() > 1e-3 * np.abs(gx).max()
