"""GPU parity of the packed-table (P4) kernel: prepared weights + 4 lookups per shared load +
exact part on the tensor cores.  Bit-exact against the oracle and against the v1 kernel."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module", params=[1, 3], ids=["p4", "p4w"])
def ax(request):
    """Every test runs on both packed-table kernels: P4 (mma.sync exact part) and P4W
    (tcgen05.mma exact part, TMEM accumulators, warp-specialised)."""
    from paper_2203_04071_b200 import _lib
    _lib.load()
    global VARIANT
    prev = _lib.axq_wpack_kernel(request.param)
    VARIANT = request.param
    yield _lib
    _lib.axq_wpack_kernel(prev)


VARIANT = 0


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (100, 16, 16), (1500, 40, 77), (2049, 33, 300),
                                   (4096, 64, 256), (1025, 17, 1040)])
@pytest.mark.parametrize("lut_kind", ["randerr", "trunc4", "b4"])
def test_p4_gemm(ax, M, N, K, lut_kind):
    bits = 4 if lut_kind == "b4" else 8
    T = {"randerr": datagen.lut_randerr(8, 0, 2), "trunc4": datagen.lut_trunc4(),
         "b4": datagen.lut_randerr(4, 4, 14)}[lut_kind]
    A = datagen.random_int8(200 + M, (M, K), bits)
    W = datagen.random_int8(300 + N, (N, K), bits)
    ref = oracle.lut_gemm(A, W, T, bits)
    lut = ax.Lut(bits, T)
    assert lut.repr == "delta8"
    Kp = (K + 15) // 16 * 16
    dA = torch.zeros(M, Kp, dtype=torch.int8, device=DEV)      # lda % 16 == 0
    dA[:, :K] = _t(A)
    dW = _t(W)
    wp = ax.WPack(lut, dW)
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm_wp(dA.narrow(1, 0, K), wp, None, C)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), ref)


@pytest.mark.parametrize("shape", [(2, 64, 14, 14, 64, 3, 3, 1, 1), (1, 32, 9, 11, 40, 3, 3, 2, 1),
                                   (3, 16, 8, 8, 33, 1, 1, 1, 0), (1, 256, 7, 7, 70, 1, 1, 2, 0),
                                   (2, 64, 23, 19, 48, 3, 3, 1, 1)])
def test_p4_conv_fused(ax, shape):
    Nb, C, H, Wd, K, R, S, st, pd = shape
    X = datagen.random_int8(80 + C, (Nb, C, H, Wd))
    Wt = datagen.random_int8(90 + K, (K, C, R, S))
    T = datagen.lut_randerr(8, 0, 2)
    ref = oracle.lut_conv2d(X, Wt, T, 8, (st, st), (pd, pd))
    lut = ax.Lut(8, T)
    d = ax.conv_desc(Nb, H, Wd, C, K, R, S, (st, st), (pd, pd))
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    dX = _t(X.transpose(0, 2, 3, 1))
    dW = _t(Wt.transpose(0, 2, 3, 1).reshape(K, -1))
    wp = ax.WPack(lut, dW)
    Y = torch.empty(Nb, Ho, Wo, K, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d_wp(d, dX, wp, None, Y)
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)
    # fused epilogue (NCHW fp32) == oracle dequant
    sa, sw = np.float32(0.0213), np.float32(0.0071)
    dsa, dsw = _t(np.array([sa])), _t(np.array([sw]))
    bias = datagen.normal(5, 5, (K,), 0.1)
    db = _t(bias)
    y = torch.empty(Nb, K, Ho, Wo, device=DEV)
    ep = ax.make_epilogue(dsa, dsw, bias=db, y=y)
    ax.axq_lut_conv2d_wp(d, dX, wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.dequantize(ref, sa, sw, bias, 1))


def test_p4_config2_full(ax):
    """BJ configs[2] at full batch through the P4 path: sampled images bit-exact."""
    c = datagen.config2()
    lut = ax.Lut(8, c.lut)
    sa = oracle.scale(oracle.amax(c.x), 8)
    qw, sw = oracle.quantize_tensor(c.W, 8)
    qx = _t(oracle.quantize(c.x, sa, 8).transpose(0, 2, 3, 1))
    wp = ax.WPack(lut, _t(qw.transpose(0, 2, 3, 1).reshape(64, -1)))
    d = ax.conv_desc(128, 56, 56, 64, 64, 3, 3, (1, 1), (1, 1))
    dsa, dsw = _t(np.array([sa])), _t(np.array([sw]))
    y = torch.empty(128, 64, 56, 56, device=DEV)
    ep = ax.make_epilogue(dsa, dsw, y=y)
    ax.axq_lut_conv2d_wp(d, qx, wp, ep)
    torch.cuda.synchronize()
    for img in (0, 127):
        acc = oracle.lut_conv2d(oracle.quantize(c.x[img:img + 1], sa, 8), qw, c.lut, 8, (1, 1), (1, 1))
        np.testing.assert_array_equal(y[img:img + 1].cpu().numpy(), oracle.dequantize(acc, sa, sw, None, 1))


@pytest.mark.parametrize("M,N,K", [(1600, 512, 4608), (700, 64, 640), (6272, 256, 2304)])
@pytest.mark.parametrize("ws_kind", ["mn", "full"])
def test_p4_small_m_split_k_fused(ax, M, N, K, ws_kind):
    """Small-M shapes: with an M*N workspace an exact split-K (atomics + epilogue kernel); with
    axq_workspace_elems (P4W) stream-K pieces in the caller's workspace.  Both bit-exact, and
    the path taken is the one claimed."""
    T = datagen.lut_randerr(8, 0, 2)
    A = datagen.random_int8(400 + M, (M, K))
    W = datagen.random_int8(500 + N, (N, K))
    ref = oracle.lut_gemm(A, W, T, 8)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(W))
    dA = _t(A)
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm_wp(dA, wp, None, C)
    np.testing.assert_array_equal(C.cpu().numpy(), ref)
    sa, sw = np.float32(0.013), np.float32(0.002)
    dsa, dsw = _t(np.array([sa])), _t(np.array([sw]))
    bias = datagen.normal(6, 6, (N,), 0.1)
    db = _t(bias)
    y = torch.empty(M, N, device=DEV)
    n_ws = M * N if ws_kind == "mn" else ax.axq_workspace_elems(M, N)
    ws = torch.zeros(n_ws, dtype=torch.int32, device=DEV)
    ep = ax.make_epilogue(dsa, dsw, bias=db, y=y, ldy=N, workspace=ws)
    ax.axq_lut_gemm_wp(dA, wp, ep)
    kern, flags = ax.axq_last_path()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.dequantize(ref, sa, sw, bias))
    assert kern == {1: "p4", 3: "p4w"}[VARIANT]
    if VARIANT == 3 and ws_kind == "full":
        assert flags & ax.PATH_STREAMK, "stream-K expected with a full workspace"
    if VARIANT == 3 and ws_kind == "mn" and M * N < ax.axq_workspace_elems(M, N):
        assert not flags & ax.PATH_STREAMK
    # the counters region is left zero (the workspace can be reused by the next call)
    assert int(ws[:256].abs().sum().item()) == 0


@pytest.mark.parametrize("M,N,K", [(3000, 48, 576), (1100, 16, 2048), (600, 40, 100)])
def test_p4_half_range_nonneg(ax, M, N, K):
    """a_nonneg handles (tables for codes 0..127) on non-negative activations."""
    T = datagen.lut_randerr(8, 0, 2)
    A = (datagen.random_int8(600 + M, (M, K)).astype(np.int64) & 127).astype(np.int8)
    W = datagen.random_int8(700 + N, (N, K))
    ref = oracle.lut_gemm(A, W, T, 8)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(W), a_nonneg=True)
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    Kp = (K + 15) // 16 * 16
    dA = torch.zeros(M, Kp, dtype=torch.int8, device=DEV)     # lda % 16 == 0
    dA[:, :K] = _t(A)
    ax.axq_lut_gemm_wp(dA.narrow(1, 0, K), wp, None, C)
    np.testing.assert_array_equal(C.cpu().numpy(), ref)


def test_p4_half_range_conv_relu_input(ax):
    c = datagen.config2(batch=3)
    sa = oracle.scale(oracle.amax(c.x), 8)
    qw, sw = oracle.quantize_tensor(c.W, 8)
    qx = oracle.quantize(c.x, sa, 8)
    assert qx.min() >= 0
    ref = oracle.lut_conv2d(qx, qw, c.lut, 8, (1, 1), (1, 1))
    lut = ax.Lut(8, c.lut)
    wp = ax.WPack(lut, _t(qw.transpose(0, 2, 3, 1).reshape(64, -1)), a_nonneg=True)
    d = ax.conv_desc(3, 56, 56, 64, 64, 3, 3, (1, 1), (1, 1))
    Y = torch.empty(3, 56, 56, 64, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d_wp(d, _t(qx.transpose(0, 2, 3, 1)), wp, None, Y)
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)


def test_p4_conv_c4_padded_stem(ax):
    """C = 3 stored as C = 4 (zero channel, c_valid = 3): the 4-byte-copy operand path."""
    X = datagen.random_int8(130, (2, 3, 20, 18))
    Wt = datagen.random_int8(131, (16, 3, 7, 7))
    T = datagen.lut_randerr(8, 0, 2)
    ref = oracle.lut_conv2d(X, Wt, T, 8, (2, 2), (3, 3))
    Xp = np.zeros((2, 20, 18, 4), np.int8)
    Xp[..., :3] = X.transpose(0, 2, 3, 1)
    Wp = np.zeros((16, 7, 7, 4), np.int8)
    Wp[..., :3] = Wt.transpose(0, 2, 3, 1)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(Wp.reshape(16, -1)))
    d = ax.conv_desc(2, 20, 18, 4, 16, 7, 7, (2, 2), (3, 3), c_valid=3)
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    Y = torch.empty(2, Ho, Wo, 16, dtype=torch.int32, device=DEV)
    ax.axq_lut_conv2d_wp(d, _t(Xp), wp, None, Y)
    np.testing.assert_array_equal(Y.cpu().numpy().transpose(0, 3, 1, 2), ref)


@pytest.mark.parametrize("M,N,K", [(256, 1024, 1024), (100, 300, 77), (17, 900, 256), (1000, 64, 96)])
def test_gemm_xs_activation_specialised(ax, M, N, K):
    """axq_lut_gemm_xs (tables specialised on the activations, built per call, weights as the
    kernel's row operand, result written back in the normal layout): raw int32 and the fused
    epilogue with bias, per-channel weight scales and requantized codes, against the oracle.
    Runs on the default (P4W) kernel only."""
    T = datagen.lut_randerr(8, 0, 2)
    A = datagen.random_int8(500 + M, (M, K))
    W = datagen.random_int8(600 + N, (N, K))
    acc = oracle.lut_gemm(A, W, T, 8)
    lut = ax.Lut(8, T)
    Kp = (K + 15) // 16 * 16
    dA = torch.zeros(M, Kp, dtype=torch.int8, device=DEV)
    dA[:, :K] = _t(A)
    dW = torch.zeros(N, Kp, dtype=torch.int8, device=DEV)
    dW[:, :K] = _t(W)
    prev = ax.axq_wpack_kernel(3)
    try:
        xp = ax.WPack(lut, dA.narrow(1, 0, K), activations=True)
        ax.axq_wpack_repack(xp, dA.narrow(1, 0, K))          # the per-call path
        C = torch.empty(M, N, dtype=torch.int32, device=DEV)
        ax.axq_lut_gemm_xs(dW.narrow(1, 0, K), xp, None, C)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(C.cpu().numpy(), acc)
        rng = np.random.default_rng(M + N)
        s_w = rng.uniform(1e-4, 1e-2, N).astype(np.float32)
        b = rng.standard_normal(N).astype(np.float32)
        s_a, s_o = np.float32(0.013), np.float32(0.02)
        y_ref = oracle.dequantize_pc(acc, s_a, s_w, b)
        q_ref = oracle.quantize(y_ref, s_o, 8)
        y = torch.empty(M, N, device=DEV)
        q = torch.empty(M, N, dtype=torch.int8, device=DEV)
        ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
        dsa, dso, ones, dsw, db = (torch.tensor([s_a], device=DEV), torch.tensor([s_o], device=DEV),
                                   torch.ones(1, device=DEV), _t(s_w), _t(b))
        ep = ax.make_epilogue(dsa, ones, bias=db, y=y, ldy=N, workspace=ws, q_out=q, ldq=N,
                              d_scale_out=dso, bits_out=8, d_scale_w_ch=dsw)
        ax.axq_lut_gemm_xs(dW.narrow(1, 0, K), xp, ep)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
        np.testing.assert_array_equal(q.cpu().numpy(), q_ref)
    finally:
        ax.axq_wpack_kernel(prev)


@pytest.mark.parametrize("s_out", [2.0, 0.5, 3.0, 0.1, 7.3])
def test_requantize_ties_and_boundaries(ax, s_out):
    """The packed-table epilogue's requantize (reciprocal fast path + exact fallback) against the
    oracle's IEEE division: s_a*s_w = 1 makes y the integer sums, so s_out = 2 puts every odd sum
    exactly on a .5 tie (half-even), and the other scales land near rounding boundaries."""
    M, N, K = 2048, 48, 64
    T = datagen.lut_randerr(8, 0, 2)
    A = datagen.random_int8(801, (M, K), full_range=False)
    W = datagen.random_int8(802, (N, K))
    acc = oracle.lut_gemm(A, W, T, 8)
    y_ref = oracle.dequantize(acc, np.float32(1.0), np.float32(1.0))
    q_ref = oracle.quantize(y_ref, np.float32(s_out), 8)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(W))
    y = torch.empty(M, N, device=DEV)
    q = torch.empty(M, N, dtype=torch.int8, device=DEV)
    ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
    one = torch.ones(1, device=DEV)
    so = torch.tensor([s_out], device=DEV)
    ep = ax.make_epilogue(one, one, y=y, ldy=N, workspace=ws, q_out=q, ldq=N, d_scale_out=so, bits_out=8)
    ax.axq_lut_gemm_wp(_t(A), wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
    np.testing.assert_array_equal(q.cpu().numpy(), q_ref)


def test_two_streams_concurrent(ax):
    """Reentrancy (include/axq.h): two packed-table layers in flight on two streams, each with its
    own workspace, both taking stream-K (every CTA writes partial slots and tile counters).  The
    scratch lives in each caller's workspace, so the interleaved launches stay bit-exact."""
    if VARIANT != 3:
        pytest.skip("stream-K is a P4W decomposition")
    T = datagen.lut_randerr(8, 0, 2)
    cases = []
    for i, (M, N, K) in enumerate([(1600, 512, 1024), (700, 256, 640)]):
        A = datagen.random_int8(900 + i, (M, K))
        W = datagen.random_int8(910 + i, (N, K))
        cases.append((M, N, A, W, oracle.lut_gemm(A, W, T, 8)))
    lut = ax.Lut(8, T)
    one = torch.ones(1, device=DEV)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    run = []
    for (M, N, A, W, ref), st in zip(cases, streams):
        wp = ax.WPack(lut, _t(W))
        ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
        ys = [torch.empty(M, N, device=DEV) for _ in range(6)]
        run.append((wp, ws, _t(A), ys, st, ref))
    torch.cuda.synchronize()
    for it in range(6):                      # interleaved launches, no host sync in between
        for wp, ws, dA, ys, st, ref in run:
            ep = ax.make_epilogue(one, one, y=ys[it], ldy=ys[it].shape[1], workspace=ws)
            ax.axq_lut_gemm_wp(dA, wp, ep, stream=st)
            assert ax.axq_last_path()[1] & ax.PATH_STREAMK
    torch.cuda.synchronize()
    for wp, ws, dA, ys, st, ref in run:
        for y in ys:
            np.testing.assert_array_equal(y.cpu().numpy(), ref.astype(np.float32))


@pytest.mark.parametrize("mode", ["relu_q", "res_relu_y_q", "y"])
@pytest.mark.parametrize("N", [64, 40])
def test_specialised_epilogue_modes(ax, mode, N):
    """The packed-table kernels' specialised epilogues (one per ResNet layer kind, decided once per
    launch): ReLU + requantize, residual + ReLU + y + requantize, y only.  s_a*s_w = 1 and s_out = 2
    put every odd integer sum on a half-even tie; N = 40 leaves a ragged last column block, which
    takes the generic path in the same launch."""
    M, K = 2048, 64
    T = datagen.lut_randerr(8, 0, 2)
    A = datagen.random_int8(811, (M, K), full_range=False)
    W = datagen.random_int8(812, (N, K))
    acc = oracle.lut_gemm(A, W, T, 8)
    one_f = np.float32(1.0)
    y_ref = oracle.dequantize(acc, one_f, one_f)
    R = np.random.default_rng(813).integers(-300, 300, (M, N)).astype(np.float32)
    if mode == "res_relu_y_q":
        y_ref = (y_ref + R).astype(np.float32)
    if mode != "y":
        y_ref = np.where(y_ref > 0, y_ref, np.float32(0)).astype(np.float32)
    q_ref = oracle.quantize(y_ref, np.float32(2.0), 8)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(W))
    y = torch.full((M, N), np.nan, device=DEV)
    q = torch.zeros(M, N, dtype=torch.int8, device=DEV)
    ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
    one = torch.ones(1, device=DEV)
    so = torch.tensor([2.0], device=DEV)
    kw = {"relu_q": dict(relu=True, q_out=q, ldq=N, d_scale_out=so, bits_out=8),
          "res_relu_y_q": dict(residual=_t(R), ldr=N, relu=True, y=y, ldy=N, q_out=q, ldq=N,
                               d_scale_out=so, bits_out=8),
          "y": dict(y=y, ldy=N)}[mode]
    ep = ax.make_epilogue(one, one, workspace=ws, **kw)
    ax.axq_lut_gemm_wp(_t(A), wp, ep)
    torch.cuda.synchronize()
    if mode != "relu_q":
        np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
    if mode != "y":
        np.testing.assert_array_equal(q.cpu().numpy(), q_ref)
