"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Integer results must be bit-exact; dequantized fp32 within 1e-6 relative
(BASELINE.json north_star; DESIGN.md §4 tolerance) -- the kernels pin the fp32 op order, so
they are expected to be exact as well."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda"
REL_TOL = 1e-6


@pytest.fixture(scope="module")
def ax():
    from paper_2203_04071_b200 import _lib
    _lib.load()
    return _lib


def _t(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    return t if dtype is None else t.to(dtype)


def _fp_close(y_gpu, y_ref, sa, sw):
    y_gpu = np.asarray(y_gpu, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    denom = np.maximum(np.abs(y_ref), float(sa) * float(sw))
    return float((np.abs(y_gpu - y_ref) / denom).max()) if y_ref.size else 0.0


def gpu_gemm(ax, A, W, lut_np, bits, lda=None, offset=0):
    lut = ax.Lut(bits, lut_np)
    M, K = A.shape
    N = W.shape[0]
    if lda is None:
        dA = _t(A)
    else:  # strided / offset view: exercises the byte loader
        buf = torch.zeros(M * lda + offset + 16, dtype=torch.int8, device=DEV)
        view = buf[offset:offset + M * lda].view(M, lda)
        view[:, :K] = _t(A)
        dA = view[:, :K]
    dW = _t(W)
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm(dA, dW, lut, C)
    torch.cuda.synchronize()
    out = C.cpu().numpy()
    lut.close()
    return out


# ----------------------------------------------------------------------------------------
# LUT-GEMM
# ----------------------------------------------------------------------------------------

def test_config0_bit_exact(ax):
    c = datagen.config0()
    C = gpu_gemm(ax, c.A, c.W, c.lut, 8)
    np.testing.assert_array_equal(C, oracle.lut_gemm(c.A, c.W, c.lut, 8))


def test_exact_lut_equals_int_mm(ax):
    """Pin (i) on the device: exact multiplier == cuBLASLt int8 IMMA (torch._int_mm)."""
    A = datagen.random_int8(1, (64, 256))
    W = datagen.random_int8(2, (64, 256))
    C = gpu_gemm(ax, A, W, datagen.lut_exact(8), 8)
    ref = torch._int_mm(_t(A), _t(W).t()).cpu().numpy()      # B = W^T, column-major
    np.testing.assert_array_equal(C, ref)


SHAPES = [(1, 1, 1), (7, 13, 1), (33, 5, 147), (129, 65, 300), (600, 40, 77),
          (2049, 33, 1040), (3000, 96, 64), (64, 1024, 1024), (5000, 7, 19)]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_ragged_shapes_randerr(ax, M, N, K):
    A = datagen.random_int8(10 + M, (M, K))
    W = datagen.random_int8(20 + N, (N, K))
    T = datagen.lut_randerr(8, 0, 2)
    np.testing.assert_array_equal(gpu_gemm(ax, A, W, T, 8), oracle.lut_gemm(A, W, T, 8))


@pytest.mark.parametrize("kind", ["trunc4", "int16", "int32", "exact"])
def test_gemm_table_representations(ax, kind):
    M, N, K = 300, 70, 200
    A = datagen.random_int8(31, (M, K))
    W = datagen.random_int8(32, (N, K))
    if kind == "trunc4":
        T = datagen.lut_trunc4()
    elif kind == "int16":
        T = datagen.random_lut(33, 8)                                     # |T| <= 2^14
    elif kind == "int32":
        T = np.random.default_rng(34).integers(-10**6, 10**6, 1 << 16).astype(np.int32)
    else:
        T = datagen.lut_exact(8)
    lut = ax.Lut(8, T)
    expect_repr = {"trunc4": "delta8", "int16": "int16", "int32": "int32", "exact": "delta8"}[kind]
    assert lut.repr == expect_repr
    lut.close()
    np.testing.assert_array_equal(gpu_gemm(ax, A, W, T, 8), oracle.lut_gemm(A, W, T, 8))


@pytest.mark.parametrize("bits", [2, 3, 4, 6, 7])
def test_gemm_low_bitwidths(ax, bits):
    M, N, K = 200, 40, 129
    A = datagen.random_int8(40 + bits, (M, K), bits)
    W = datagen.random_int8(50 + bits, (N, K), bits)
    for T in (datagen.lut_randerr(bits, 4, 10 + bits) if bits >= 2 else None,
              datagen.random_lut(60 + bits, bits)):
        np.testing.assert_array_equal(gpu_gemm(ax, A, W, T, bits), oracle.lut_gemm(A, W, T, bits))


def test_gemm_strided_and_unaligned_operands(ax):
    M, N, K = 257, 45, 100
    A = datagen.random_int8(70, (M, K))
    W = datagen.random_int8(71, (N, K))
    T = datagen.lut_randerr(8, 0, 2)
    ref = oracle.lut_gemm(A, W, T, 8)
    np.testing.assert_array_equal(gpu_gemm(ax, A, W, T, 8, lda=112), ref)        # aligned ld
    np.testing.assert_array_equal(gpu_gemm(ax, A, W, T, 8, lda=101, offset=3), ref)  # unaligned


def test_gemm_edge_cases(ax):
    T = datagen.lut_randerr(8, 0, 2)
    lut = ax.Lut(8, T)
    # K = 0: zeros
    A = torch.zeros(5, 0, dtype=torch.int8, device=DEV)
    W = torch.zeros(3, 0, dtype=torch.int8, device=DEV)
    C = torch.full((5, 3), 7, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm(A, W, lut, C)
    assert (C.cpu() == 0).all()
    # M = 0 / N = 0: no-ops
    ax.axq_lut_gemm(torch.zeros(0, 4, dtype=torch.int8, device=DEV),
                    torch.zeros(3, 4, dtype=torch.int8, device=DEV), lut,
                    torch.zeros(0, 3, dtype=torch.int32, device=DEV))
    # overflow guard: K * max|T| >= 2^31
    big = torch.zeros(1, 140000, dtype=torch.int8, device=DEV)
    with pytest.raises(ax.AxqError) as e:
        ax.axq_lut_gemm(big, big, lut, torch.zeros(1, 1, dtype=torch.int32, device=DEV))
    assert e.value.status == ax.AXQ_ERR_OVERFLOW
    lut.close()


def test_gemm_max_k_within_guard(ax):
    """Largest K the int32 guard admits for a b=8 table, with extreme operands: exact."""
    T = datagen.lut_exact(8)
    K = (2**31 - 1) // 16384
    A = np.full((3, K), -128, np.int8)
    W = np.full((2, K), -128, np.int8)
    C = gpu_gemm(ax, A, W, T, 8)
    assert (C == K * 16384).all()


# ----------------------------------------------------------------------------------------
# quantizer
# ----------------------------------------------------------------------------------------

def _gpu_quantize(ax, x, bits):
    dx = _t(x)
    amax = torch.empty(1, device=DEV)
    s = torch.empty(1, device=DEV)
    q = torch.empty(dx.shape, dtype=torch.int8, device=DEV)
    ax.axq_amax(dx, amax)
    ax.axq_scale(amax, bits, s)
    ax.axq_quantize(dx, s, bits, q)
    torch.cuda.synchronize()
    return amax.cpu().numpy()[0], s.cpu().numpy()[0], q.cpu().numpy()


@pytest.mark.parametrize("bits", [2, 4, 6, 8])
def test_quantize_bit_exact(ax, bits):
    for x in (datagen.config1().x, datagen.normal(7, 1, (1001, 13), 3.0),
              datagen.config2(batch=2).x):
        a, s, q = _gpu_quantize(ax, x, bits)
        assert a == oracle.amax(x)
        assert s == oracle.scale(a, bits)
        np.testing.assert_array_equal(q, oracle.quantize(x, s, bits))


def test_quantize_ties_and_zero(ax):
    x = np.array([127.0, 2.5, 3.5, -2.5, 0.5, -0.5, 1.5, 126.5], np.float32)
    a, s, q = _gpu_quantize(ax, x, 8)
    assert s == 1.0
    np.testing.assert_array_equal(q, [127, 2, 4, -2, 0, 0, 2, 126])
    a, s, q = _gpu_quantize(ax, np.zeros(37, np.float32), 8)
    assert a == 0.0 and s == 1.0 and (q == 0).all()


def test_quantize_nchw_to_nhwc(ax):
    x = datagen.config2(batch=3).x[:, :, :17, :23].copy()
    s = oracle.scale(oracle.amax(x), 8)
    dx = _t(x)
    ds = torch.tensor([s], device=DEV)
    q = torch.empty(3, 17, 23, 64, dtype=torch.int8, device=DEV)
    ax.axq_quantize_nchw_to_nhwc(dx, ds, 8, q)
    np.testing.assert_array_equal(q.cpu().numpy(), oracle.quantize(x, s, 8).transpose(0, 2, 3, 1))


@pytest.mark.parametrize("C,Cq", [(3, 4), (4, 4), (1, 4), (3, 8)])
def test_quantize_nchw_to_nhwc_few_channels(ax, C, Cq):
    """The network-input path (C <= 4 into 4-byte pixels: reciprocal requantize with the exact
    fallback) and the generic few-channel path give the oracle's codes; padded channels are 0."""
    x = datagen.normal(143, C, (5, C, 19, 23), 2.0)
    x[0, 0, 0, :8] = np.float32([0.5, 1.5, -2.5, 2.5, 126.5, -126.5, 0.0, -0.0]) * np.float32(0.04)
    s = np.float32(0.04)
    ref = np.zeros((5, 19, 23, Cq), np.int8)
    ref[..., :C] = oracle.quantize(x, s, 8).transpose(0, 2, 3, 1)
    q = torch.full((5, 19, 23, Cq), 99, dtype=torch.int8, device=DEV)
    ax.axq_quantize_nchw_to_nhwc(_t(x), torch.tensor([s], device=DEV), 8, q)
    np.testing.assert_array_equal(q.cpu().numpy(), ref)


def test_dequantize(ax):
    rng = np.random.default_rng(3)
    acc = rng.integers(-2**31, 2**31, size=(37, 19), dtype=np.int64).astype(np.int32)
    b = rng.standard_normal(19).astype(np.float32)
    sa, sw = np.float32(0.0123), np.float32(0.00077)
    y = torch.empty(37, 19, device=DEV)
    ax.axq_dequantize(_t(acc), _t(np.array([sa])), _t(np.array([sw])), _t(b), y)
    ref = oracle.dequantize(acc, sa, sw, b)
    assert _fp_close(y.cpu().numpy(), ref, sa, sw) <= REL_TOL
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


# ----------------------------------------------------------------------------------------
# linear layer (config 1) and conv (config 2)
# ----------------------------------------------------------------------------------------

def test_config1_linear_full(ax):
    from paper_2203_04071_b200.layers import ApproxLinear
    c = datagen.config1()
    lut = ax.Lut(8, c.lut)
    layer = ApproxLinear(_t(c.W), _t(c.b), lut)
    y = layer(_t(c.x))
    torch.cuda.synchronize()
    y_ref, acc_ref, (qa, sa, qw, sw) = oracle.linear(c.x, c.W, c.b, c.lut, 8)
    np.testing.assert_array_equal(layer.qw.cpu().numpy(), qw)
    assert layer.d_scale_a.item() == sa and layer.d_scale_w.item() == sw
    assert _fp_close(y.cpu().numpy(), y_ref, sa, sw) <= REL_TOL
    np.testing.assert_array_equal(y.cpu().numpy(), y_ref)


@pytest.mark.parametrize("path", ["gather", "xspec", "wpack"])
def test_config1_linear_paths(ax, path):
    """The three kernel paths of ApproxLinear (per-row gather, activation-specialised tables
    built per call, weight-specialised tables) give the oracle's output bit for bit."""
    from paper_2203_04071_b200.layers import ApproxLinear
    c = datagen.config1()
    lut = ax.Lut(8, c.lut)
    layer = ApproxLinear(_t(c.W), _t(c.b), lut)
    if path == "gather":
        layer.xspec = False
    elif path == "xspec":
        layer.xspec = True
    else:
        layer.XS_MIN_M, layer.WP_MIN_M = 1 << 30, 1
    assert layer.path(c.x.shape[0]) == path
    y_ref, _, _ = oracle.linear(c.x, c.W, c.b, c.lut, 8)
    for _ in range(2):   # the second call reuses the per-M buffers / tables
        y = layer(_t(c.x))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy(), y_ref)


CONV_SHAPES = [
    # N, C, H, W, K, R, S, stride, pad
    (2, 64, 14, 14, 64, 3, 3, 1, 1),
    (1, 3, 32, 32, 64, 7, 7, 2, 3),       # conv1-like: C=3 byte loader, K=147
    (2, 32, 9, 11, 40, 3, 3, 2, 1),
    (3, 16, 8, 8, 33, 1, 1, 1, 0),
    (1, 48, 10, 7, 20, 3, 3, 1, 2),
    (2, 20, 6, 6, 8, 3, 3, 2, 0),          # C not a multiple of 16
    (1, 256, 7, 7, 70, 1, 1, 2, 0),        # strided 1x1 (projection shortcut)
]


@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_conv_int32_and_fused(ax, shape):
    Nb, C, H, Wd, K, R, S, st, pd = shape
    X = datagen.random_int8(80 + C, (Nb, C, H, Wd))
    Wt = datagen.random_int8(90 + K, (K, C, R, S))
    T = datagen.lut_randerr(8, 0, 2)
    ref = oracle.lut_conv2d(X, Wt, T, 8, (st, st), (pd, pd))                  # NCHW int32
    lut = ax.Lut(8, T)
    d = ax.conv_desc(Nb, H, Wd, C, K, R, S, (st, st), (pd, pd))
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    dX = _t(X.transpose(0, 2, 3, 1))
    dW = _t(Wt.transpose(0, 2, 3, 1))
    Y = torch.empty(Nb, Ho, Wo, K, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d(d, dX, dW, lut, Y)
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)
    # fused dequant epilogue == unfused chain, bit for bit, and == oracle dequant
    sa, sw = np.float32(0.0213), np.float32(0.0071)
    dsa, dsw = _t(np.array([sa])), _t(np.array([sw]))
    bias = datagen.normal(5, 5, (K,), 0.1)
    y1 = torch.empty(Nb, K, Ho, Wo, device=DEV)
    y2 = torch.empty(Nb, K, Ho, Wo, device=DEV)
    ax.axq_lut_conv2d_dq(d, dX, dW, lut, dsa, dsw, _t(bias), y1)
    ax.axq_dequantize_nhwc_to_nchw(Y, dsa, dsw, _t(bias), y2)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y1.cpu().numpy(), y2.cpu().numpy())
    np.testing.assert_array_equal(y1.cpu().numpy(), oracle.dequantize(ref, sa, sw, bias, 1))
    lut.close()


def test_config2_conv_sampled_images(ax):
    """BJ:c2 at full size (batch 128) in the bench launch configuration; the oracle
    recomputes whole sampled images (quantization uses the full-tensor amax)."""
    from paper_2203_04071_b200.layers import ApproxConv2d
    c = datagen.config2()
    lut = ax.Lut(8, c.lut)
    layer = ApproxConv2d(_t(c.W), None, lut, c.stride, c.pad)
    y = layer(_t(c.x))
    torch.cuda.synchronize()
    sa = oracle.scale(oracle.amax(c.x), 8)
    qw, sw = oracle.quantize_tensor(c.W, 8)
    assert layer.d_scale_a.item() == sa and layer.d_scale_w.item() == sw
    for img in (0, 77, 127):
        qx = oracle.quantize(c.x[img:img + 1], sa, 8)
        acc = oracle.lut_conv2d(qx, qw, c.lut, 8, c.stride, c.pad)
        ref = oracle.dequantize(acc, sa, sw, None, 1)
        got = y[img:img + 1].cpu().numpy()
        assert _fp_close(got, ref, sa, sw) <= REL_TOL
        np.testing.assert_array_equal(got, ref)


# ----------------------------------------------------------------------------------------
# fused epilogue variants and model glue kernels
# ----------------------------------------------------------------------------------------

def test_conv_fused_residual_relu_requantize(ax):
    Nb, C, H, Wd, K = 2, 32, 9, 7, 48
    X = datagen.random_int8(120, (Nb, C, H, Wd))
    Wt = datagen.random_int8(121, (K, C, 3, 3))
    T = datagen.lut_randerr(8, 0, 2)
    acc = oracle.lut_conv2d(X, Wt, T, 8, (1, 1), (1, 1)).transpose(0, 2, 3, 1)   # NHWC
    sa, sw, so = np.float32(0.013), np.float32(0.0041), np.float32(0.05)
    res = datagen.normal(122, 0, acc.shape, 2.0)
    v = (acc.astype(np.float32) * np.float32(sa * sw)).astype(np.float32)
    v = (v + res).astype(np.float32)
    v = np.where(v > 0, v, np.float32(0)).astype(np.float32)
    q_ref = oracle.quantize(v, so, 8)
    lut = ax.Lut(8, T)
    d = ax.conv_desc(Nb, H, Wd, C, K, 3, 3, (1, 1), (1, 1))
    y = torch.empty(acc.shape, device=DEV)
    q = torch.empty(acc.shape, dtype=torch.int8, device=DEV)
    # the epilogue struct holds raw pointers: keep every tensor alive until the launch
    dsa, dsw, dso, dres = _t(np.array([sa])), _t(np.array([sw])), _t(np.array([so])), _t(res)
    dX, dW = _t(X.transpose(0, 2, 3, 1)), _t(Wt.transpose(0, 2, 3, 1))
    for ws in (None, torch.empty(acc.size, dtype=torch.int32, device=DEV)):
        ep = ax.make_epilogue(dsa, dsw, y=y, ldy=K, workspace=ws, residual=dres, ldr=K,
                              relu=True, y_nhwc=True, q_out=q, ldq=K, d_scale_out=dso, bits_out=8)
        ax.axq_lut_conv2d_ep(d, dX, dW, lut, ep)
        np.testing.assert_array_equal(y.cpu().numpy(), v)
        np.testing.assert_array_equal(q.cpu().numpy(), q_ref)
    lut.close()


def test_conv_padded_channels_c_valid(ax):
    """C = 3 stored as C = 4 with a zero channel: c_valid removes the padding lookups."""
    X = datagen.random_int8(130, (2, 3, 20, 18))
    Wt = datagen.random_int8(131, (16, 3, 7, 7))
    T = datagen.lut_randerr(8, 0, 2)
    ref = oracle.lut_conv2d(X, Wt, T, 8, (2, 2), (3, 3))
    Xp = np.zeros((2, 20, 18, 4), np.int8)
    Xp[..., :3] = X.transpose(0, 2, 3, 1)
    Wp = np.zeros((16, 7, 7, 4), np.int8)
    Wp[..., :3] = Wt.transpose(0, 2, 3, 1)
    lut = ax.Lut(8, T)
    d = ax.conv_desc(2, 20, 18, 4, 16, 7, 7, (2, 2), (3, 3), c_valid=3)
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    Y = torch.empty(2, Ho, Wo, 16, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d(d, _t(Xp), _t(Wp), lut, Y)
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)
    lut.close()


def test_maxpool_int8(ax):
    from oracle.models import _maxpool
    x = datagen.random_int8(140, (2, 13, 11, 12))          # NHWC codes
    y = torch.empty(2, 7, 6, 12, dtype=torch.int8, device=DEV)
    ax.axq_maxpool2d_nhwc_i8(_t(x), 3, 3, 2, 1, y)
    ref = _maxpool(x.transpose(0, 3, 1, 2).astype(np.float32)).transpose(0, 2, 3, 1)
    np.testing.assert_array_equal(y.cpu().numpy(), ref.astype(np.int8))
    x16 = datagen.random_int8(142, (3, 15, 12, 48))        # C % 16 == 0: 16-channel kernel
    y16 = torch.empty(3, 8, 6, 48, dtype=torch.int8, device=DEV)
    ax.axq_maxpool2d_nhwc_i8(_t(x16), 3, 3, 2, 1, y16)
    ref16 = _maxpool(x16.transpose(0, 3, 1, 2).astype(np.float32)).transpose(0, 2, 3, 1)
    np.testing.assert_array_equal(y16.cpu().numpy(), ref16.astype(np.int8))
    x3 = datagen.random_int8(141, (1, 9, 9, 6))            # C % 4 != 0: byte kernel
    y3 = torch.empty(1, 5, 5, 6, dtype=torch.int8, device=DEV)
    ax.axq_maxpool2d_nhwc_i8(_t(x3), 3, 3, 2, 1, y3)
    ref3 = _maxpool(x3.transpose(0, 3, 1, 2).astype(np.float32)).transpose(0, 2, 3, 1)
    np.testing.assert_array_equal(y3.cpu().numpy(), ref3.astype(np.int8))


def test_avgpool_and_quantize(ax):
    from oracle.models import _avgpool
    x = np.abs(datagen.normal(150, 0, (3, 7, 7, 40), 3.0))  # NHWC
    s = np.float32(0.021)
    y = torch.empty(3, 40, device=DEV)
    q = torch.empty(3, 40, dtype=torch.int8, device=DEV)
    ax.axq_avgpool_nhwc(_t(x), y=y, q=q, d_scale=_t(np.array([s])), bits=8)
    ref = _avgpool(x.transpose(0, 3, 1, 2))
    np.testing.assert_array_equal(y.cpu().numpy(), ref)
    np.testing.assert_array_equal(q.cpu().numpy(), oracle.quantize(ref, s, 8))


def test_lstm_cell(ax):
    from oracle.models import pinned_sigmoid, pinned_tanh
    B, H = 5, 33
    gih = datagen.normal(160, 0, (B, 4 * H), 3.0)
    ghh = datagen.normal(160, 1, (B, 4 * H), 3.0)
    c0 = datagen.normal(160, 2, (B, H))
    g = (gih + ghh).astype(np.float32)
    i_, f_ = pinned_sigmoid(g[:, :H]), pinned_sigmoid(g[:, H:2 * H])
    g_, o_ = pinned_tanh(g[:, 2 * H:3 * H]), pinned_sigmoid(g[:, 3 * H:])
    c_ref = ((f_ * c0).astype(np.float32) + (i_ * g_).astype(np.float32)).astype(np.float32)
    h_ref = (o_ * pinned_tanh(c_ref)).astype(np.float32)
    s = np.float32(1.0 / 127)
    c = _t(c0)
    h = torch.empty(B, H, device=DEV)
    q = torch.empty(B, H, dtype=torch.int8, device=DEV)
    ax.axq_lstm_cell(_t(gih), _t(ghh), c, h, q_h=q, d_scale_h=_t(np.array([s])), bits=8)
    np.testing.assert_array_equal(c.cpu().numpy(), c_ref)
    np.testing.assert_array_equal(h.cpu().numpy(), h_ref)
    np.testing.assert_array_equal(q.cpu().numpy(), oracle.quantize(h_ref, s, 8))


@pytest.mark.parametrize("M,N,K", [(64, 4096, 1024), (37, 300, 129), (64, 512, 77), (1, 1000, 2048)])
def test_gemm_small_m_column_split_tiles(ax, M, N, K):
    """M <= 64 takes the column-split tile (warps over N), with and without split-K."""
    A = datagen.random_int8(900 + M, (M, K))
    W = datagen.random_int8(901 + N, (N, K))
    T = datagen.lut_randerr(8, 4, 18)
    np.testing.assert_array_equal(gpu_gemm(ax, A, W, T, 8), oracle.lut_gemm(A, W, T, 8))
