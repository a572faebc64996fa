"""GPU parity of the wide-ACU path (NEXT-2: b = 10, 12 with int16 codes) against
the oracle: int16 quantizer codes, raw int32 LUT-GEMM for delta16 and int32 tables, the fused
epilogue, and the int8 entry points refusing a wide handle."""
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


@pytest.mark.parametrize("bits", [10, 12])
def test_quantize16(ax, bits):
    x = datagen.normal(36, bits, (1000, 77))
    s = oracle.scale(oracle.amax(x), bits)
    ref = oracle.quantize16(x, s, bits)
    q = torch.empty(x.shape, dtype=torch.int16, device=DEV)
    ax.axq_quantize16(_t(x), torch.tensor([s], device=DEV), bits, q)
    np.testing.assert_array_equal(q.cpu().numpy(), ref)


@pytest.mark.parametrize("bits,kind", [(10, "randerr"), (12, "randerr"), (10, "wide32"), (12, "exact")])
@pytest.mark.parametrize("M,N,K", [(300, 37, 129), (1, 1, 1), (513, 16, 64)])
def test_lut_gemm16(ax, bits, kind, M, N, K):
    if kind == "randerr":
        T = datagen.lut_randerr(bits, 9, 2)
    elif kind == "exact":
        T = datagen.lut_exact(bits)
    else:
        T = (datagen.lut_exact(bits).astype(np.int64)
             + np.random.default_rng(7).integers(-100000, 100000, 1 << (2 * bits))).astype(np.int32)
    A = datagen.random_int16(10 + M, (M, K), bits)
    W = datagen.random_int16(20 + N, (N, K), bits)
    ref = oracle.lut_gemm16(A, W, T, bits)
    lut = ax.Lut(bits, T)
    assert lut.repr == ("wide32" if kind == "wide32" else "wide16")
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm16(_t(A), _t(W), lut, None, C)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), ref)


def test_lut_gemm16_fused_and_guards(ax):
    bits = 12
    T = datagen.lut_randerr(bits, 9, 3)
    x = datagen.normal(37, 1, (200, 96))
    w = datagen.normal(37, 2, (48, 96), 0.05)
    b = datagen.normal(37, 3, (48,), 0.01)
    sa, sw = oracle.scale(oracle.amax(x), bits), oracle.scale(oracle.amax(w), bits)
    qa, qw = oracle.quantize16(x, sa, bits), oracle.quantize16(w, sw, bits)
    ref = oracle.dequantize(oracle.lut_gemm16(qa, qw, T, bits), sa, sw, b)
    lut = ax.Lut(bits, T)
    y = torch.empty(200, 48, device=DEV)
    dsa, dsw, db = torch.tensor([sa], device=DEV), torch.tensor([sw], device=DEV), _t(b)
    ep = ax.make_epilogue(dsa, dsw, bias=db, y=y, ldy=48)
    ax.axq_lut_gemm16(_t(qa), _t(qw), lut, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), ref)
    # the int8 entry points refuse a wide handle; the int32 guard holds
    with pytest.raises(ax.AxqError) as e:
        ax.axq_lut_gemm(torch.zeros(4, 8, dtype=torch.int8, device=DEV),
                        torch.zeros(4, 8, dtype=torch.int8, device=DEV), lut,
                        torch.zeros(4, 4, dtype=torch.int32, device=DEV))
    assert e.value.status == ax.AXQ_ERR_UNSUPPORTED
    with pytest.raises(ax.AxqError) as e:
        big = torch.zeros(2, 4096, dtype=torch.int16, device=DEV)
        ax.axq_lut_gemm16(big, big, lut, None, torch.zeros(2, 2, dtype=torch.int32, device=DEV))
    assert e.value.status == ax.AXQ_ERR_OVERFLOW


@pytest.mark.parametrize("bits", [9, 10, 11, 12])
@pytest.mark.parametrize("M,N,K", [(300, 37, 129), (1, 1, 1), (2049, 16, 64), (4100, 9, 300)])
def test_lut_gemm16_packed(ax, bits, M, N, K):
    """NEXT-2 packed (the table tiled by the weights, axq_lut_gemm16_wp) == the oracle, raw int32
    and fused epilogue, ragged M / N / K (K padded to whole stages)."""
    T = datagen.lut_randerr(bits, 9, bits)
    A = datagen.random_int16(30 + M, (M, K), bits)
    W = datagen.random_int16(40 + N, (N, K), bits)
    ref = oracle.lut_gemm16(A, W, T, bits)
    lut = ax.Lut(bits, T)
    assert lut.repr == "wide16"
    wp = ax.WPack16(lut, _t(W))
    C = torch.empty(M, N, dtype=torch.int32, device=DEV)
    ax.axq_lut_gemm16_wp(_t(A), wp, None, C)
    assert ax.axq_last_path()[0] == "widepk"
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), ref)
    sa, sw = np.float32(0.0007), np.float32(0.0011)
    b = datagen.normal(38, bits, (N,), 0.1)
    y = torch.empty(M, N, device=DEV)
    ep = ax.make_epilogue(_t(np.array([sa])), _t(np.array([sw])), bias=_t(b), y=y, ldy=N)
    ax.axq_lut_gemm16_wp(_t(A), wp, ep)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.dequantize(ref, sa, sw, b))


def test_wpack16_refuses_wide32(ax):
    bits = 10
    T = (datagen.lut_exact(bits).astype(np.int64)
         + np.random.default_rng(7).integers(-100000, 100000, 1 << (2 * bits))).astype(np.int32)
    lut = ax.Lut(bits, T)
    with pytest.raises(ax.AxqError) as e:
        ax.WPack16(lut, torch.zeros(4, 8, dtype=torch.int16, device=DEV))
    assert e.value.status == ax.AXQ_ERR_UNSUPPORTED
