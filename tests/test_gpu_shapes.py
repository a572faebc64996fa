"""Every P4W CTA shape (consumer-warp counts selected with axq_wpack_shapes) gives the oracle's
results bit for bit: the non-residual half-range shape (28 / 24 / 20 warps), the residual shape
(16 / 20 / 24 / 28), the small-M shape (16, or off) -- raw int32 sums and the fused residual
epilogue (dequantize + residual + ReLU + fp32 out + requantize), over ragged row counts."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda"

SHAPES = [(28, 16, 16), (20, 20, 28), (24, 24, 16), (28, 28, 28), (20, 16, 16)]


@pytest.fixture(scope="module", params=SHAPES, ids=["main%d-res%d-small%d" % s for s in SHAPES])
def ax(request):
    from paper_2203_04071_b200 import _lib
    _lib.load()
    _lib.axq_wpack_shapes(*request.param)
    yield _lib
    _lib.axq_wpack_shapes(28, 16, 16)   # the defaults


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def test_shapes_reject_unknown():
    from paper_2203_04071_b200 import _lib
    with pytest.raises(_lib.AxqError):
        _lib.axq_wpack_shapes(32, 0, 0)
    with pytest.raises(_lib.AxqError):
        _lib.axq_wpack_shapes(0, 12, 0)


@pytest.mark.parametrize("M,N,K", [(700, 48, 64), (2100, 32, 192), (4000, 16, 96), (300, 40, 576)])
@pytest.mark.parametrize("half", [True, False])
def test_shape_raw_sums(ax, M, N, K, half):
    T = datagen.lut_randerr(8, 0, 2)
    A = datagen.random_int8(900 + M, (M, K))
    if half:
        A = (A.astype(np.int64) & 127).astype(np.int8)
    W = datagen.random_int8(910 + N, (N, K))
    ref = oracle.lut_gemm(A, W, T, 8)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(W), a_nonneg=half)
    Kp = (K + 15) // 16 * 16
    dA = torch.zeros(M, Kp, dtype=torch.int8, device=DEV)
    dA[:, :K] = _t(A)
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm_wp(dA.narrow(1, 0, K), wp, None, C)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), ref)


@pytest.mark.parametrize("M,N,K", [(700, 64, 64), (2100, 48, 128), (3000, 32, 256)])
def test_shape_residual_epilogue(ax, M, N, K):
    """The block-output epilogue of a residual layer (A17: one fp32 residual add, then ReLU)."""
    T = datagen.lut_randerr(8, 0, 2)
    A = (datagen.random_int8(920 + M, (M, K)).astype(np.int64) & 127).astype(np.int8)
    W = datagen.random_int8(930 + N, (N, K))
    acc = oracle.lut_gemm(A, W, T, 8)
    sa, sw, so = np.float32(0.011), np.float32(0.0037), np.float32(0.045)
    r = datagen.normal(940 + M, 940 + M, (M, N), 0.5)
    y_ref = np.maximum(oracle.dequantize(acc, sa, sw) + r, np.float32(0))
    q_ref = oracle.quantize(y_ref, so, 8)
    lut = ax.Lut(8, T)
    wp = ax.WPack(lut, _t(W), a_nonneg=True)
    y = torch.empty(M, N, device=DEV)
    q = torch.empty(M, N, dtype=torch.int8, device=DEV)
    ws = torch.zeros(ax.axq_workspace_elems(M, N), dtype=torch.int32, device=DEV)
    dsa, dsw, dso = _t(np.array([sa])), _t(np.array([sw])), _t(np.array([so]))
    dr = _t(r)
    ep = ax.make_epilogue(dsa, dsw, y=y, ldy=N, workspace=ws, residual=dr, ldr=N, relu=True,
                          q_out=q, ldq=N, d_scale_out=dso, bits_out=8)
    ax.axq_lut_gemm_wp(_t(A), wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), y_ref)
    np.testing.assert_array_equal(q.cpu().numpy(), q_ref)
