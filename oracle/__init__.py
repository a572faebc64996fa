"""CPU oracle for the AdaPT approximate LUT layer -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2203_04071_b200``) never imports it and shares no code with it.

The arithmetic lives in ``axq_oracle.c`` (plain loops, int64 sums, pinned fp32); this module
only compiles it with gcc and marshals numpy arrays through ctypes.  Each wrapper names the
paper passage its C function follows (see the C file for the full citation).

Parity status: every function here is pinned by tests/test_oracle_pins.py against closed
forms, library routines, brute force or the worked examples in tests/golden/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_SRC = [_DIR / "axq_oracle.c", _DIR / "resnet_oracle.c", _DIR / "lstm_oracle.c"]
_LIB = _DIR / "liboracle.so"
_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
           "-std=c11", "-Wall"]


def build(force: bool = False) -> Path:
    srcs = [s for s in _SRC if s.exists()]
    if force or not _LIB.exists() or any(s.stat().st_mtime > _LIB.stat().st_mtime for s in srcs):
        tmp = _LIB.with_suffix(".so.tmp%d" % os.getpid())
        subprocess.check_call(["gcc", *_CFLAGS, *map(str, srcs), "-o", str(tmp), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        i64, i32, f32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_void_p
        L.orc_amax.argtypes = [vp, i64]
        L.orc_amax.restype = f32
        L.orc_scale.argtypes = [f32, i32]
        L.orc_scale.restype = f32
        L.orc_quantize.argtypes = [vp, i64, f32, i32, vp]
        L.orc_quantize.restype = None
        L.orc_lut_gemm.argtypes = [i64, i64, i64, vp, vp, i32, vp, vp]
        L.orc_lut_gemm.restype = i64
        L.orc_lut_conv2d.argtypes = [i64] * 14 + [vp, vp, i32, vp, vp]
        L.orc_lut_conv2d.restype = i64
        L.orc_dequantize.argtypes = [i64, vp, f32, f32, vp, i64, i64, vp]
        L.orc_dequantize.restype = None
        L.orc_amax_rows.argtypes = [vp, i64, i64, vp]
        L.orc_amax_rows.restype = None
        L.orc_quantize_rows.argtypes = [vp, i64, i64, vp, i32, vp]
        L.orc_quantize_rows.restype = None
        L.orc_hist_calib.argtypes = [vp, i64, i32, i64, i64, ctypes.POINTER(f32)]
        L.orc_hist_calib.restype = i64
        L.orc_dequantize_pc.argtypes = [i64, vp, f32, vp, vp, i64, i64, vp]
        L.orc_dequantize_pc.restype = None
        L.orc_quantize16.argtypes = [vp, i64, f32, i32, vp]
        L.orc_quantize16.restype = None
        L.orc_lut_gemm16.argtypes = [i64, i64, i64, vp, vp, i32, vp, vp]
        L.orc_lut_gemm16.restype = i64
        L.orc_set_threads.argtypes = [i32]
        L.orc_set_threads.restype = None
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = i32
        _register_models(L)
        _lib = L
    return _lib


def _register_models(L):
    from . import models  # noqa: F401  (binds the ResNet/LSTM entry points when present)
    models.register(L)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ---- quantizer ----

def amax(x) -> np.float32:
    x = _c(x, np.float32)
    return np.float32(lib().orc_amax(_p(x), x.size))


def scale(amax_v, bits: int) -> np.float32:
    return np.float32(lib().orc_scale(float(np.float32(amax_v)), int(bits)))


def quantize(x, s, bits: int) -> np.ndarray:
    x = _c(x, np.float32)
    q = np.empty(x.shape, np.int8)
    lib().orc_quantize(_p(x), x.size, float(np.float32(s)), int(bits), _p(q))
    return q


def dequantize(acc, s_a, s_w, bias=None, channel_axis: int = -1) -> np.ndarray:
    """y = fl(fl(acc * fl(s_a*s_w)) + bias[ch]) with ch the index along ``channel_axis``."""
    acc = _c(acc, np.int32)
    y = np.empty(acc.shape, np.float32)
    ax = channel_axis % acc.ndim
    nch = acc.shape[ax]
    inner = int(np.prod(acc.shape[ax + 1:], dtype=np.int64))
    b = None if bias is None else _c(bias, np.float32)
    lib().orc_dequantize(acc.size, _p(acc), float(np.float32(s_a)), float(np.float32(s_w)),
                         None if b is None else _p(b), nch, inner, _p(y))
    return y


# ---- LUT GEMM / conv ----

def lut_gemm(A, W, lut, bits: int) -> np.ndarray:
    """A int8 [M][K], W int8 [N][K] -> int32 [M][N]; raises if an exact sum exceeds int32."""
    A = _c(A, np.int8)
    W = _c(W, np.int8)
    T = _c(lut, np.int32)
    assert T.size == 1 << (2 * bits)
    M, K = A.shape
    N, K2 = W.shape
    assert K == K2
    C = np.empty((M, N), np.int32)
    bad = lib().orc_lut_gemm(M, N, K, _p(A), _p(W), int(bits), _p(T), _p(C))
    if bad:
        raise OverflowError("%d outputs exceed int32" % bad)
    return C


def conv_out_hw(H, W, R, S, stride, pad, dil=(1, 1)):
    Ho = (H + 2 * pad[0] - dil[0] * (R - 1) - 1) // stride[0] + 1
    Wo = (W + 2 * pad[1] - dil[1] * (S - 1) - 1) // stride[1] + 1
    return Ho, Wo


def lut_conv2d(X, Wt, lut, bits: int, stride=(1, 1), pad=(0, 0), dil=(1, 1),
               groups: int = 1) -> np.ndarray:
    """X int8 NCHW, Wt int8 (Cout, Cin/groups, R, S) -> int32 NCHW."""
    X = _c(X, np.int8)
    Wt = _c(Wt, np.int8)
    T = _c(lut, np.int32)
    Nb, C, H, Wd = X.shape
    Co, Cg, R, S = Wt.shape
    assert Cg * groups == C and Co % groups == 0
    Ho, Wo = conv_out_hw(H, Wd, R, S, stride, pad, dil)
    Y = np.empty((Nb, Co, Ho, Wo), np.int32)
    bad = lib().orc_lut_conv2d(Nb, C, H, Wd, Co, R, S, stride[0], stride[1], pad[0], pad[1],
                               dil[0], dil[1], groups, _p(X), _p(Wt), int(bits), _p(T), _p(Y))
    if bad:
        raise OverflowError("%d outputs exceed int32" % bad)
    return Y


# ---- composed layers (the steps in the order §8(a) lists them) ----

def quantize_tensor(x, bits: int):
    """Max-calibrated per-tensor quantization: (q, s) (BJ:ns)."""
    s = scale(amax(x), bits)
    return quantize(x, s, bits), s


def linear(x, W, b, lut, bits: int):
    """Approximate Linear y = x W^T + b with every multiply a LUT lookup."""
    qa, sa = quantize_tensor(x, bits)
    qw, sw = quantize_tensor(W, bits)
    acc = lut_gemm(qa, qw, lut, bits)
    return dequantize(acc, sa, sw, b), acc, (qa, sa, qw, sw)


def conv2d(x, W, bias, lut, bits: int, stride=(1, 1), pad=(0, 0)):
    """Approximate Conv2d on fp32 NCHW input; returns fp32 NCHW."""
    qa, sa = quantize_tensor(x, bits)
    qw, sw = quantize_tensor(W, bits)
    acc = lut_conv2d(qa, qw, lut, bits, stride, pad)
    return dequantize(acc, sa, sw, bias, channel_axis=1), acc, (qa, sa, qw, sw)


# ---- NEXT-1: the paper's quantizer -- per-channel weights, 99.9 % histogram activations
#      (readings A30-A32) ----

HIST_BINS = 2048
PERCENTILE = (999, 1000)      # 99.9 %


def amax_rows(W) -> np.ndarray:
    """Per-output-channel max |W| (A31); W [rows][...] flattened per row."""
    W = _c(W, np.float32)
    rows = W.shape[0]
    cols = W.size // rows
    a = np.empty(rows, np.float32)
    lib().orc_amax_rows(_p(W), rows, cols, _p(a))
    return a


def scale_rows(amax_r, bits: int) -> np.ndarray:
    """Per-channel scales: orc_scale of each channel's amax (A4 per channel)."""
    return np.array([scale(a, bits) for a in np.asarray(amax_r, np.float32)], np.float32)


def quantize_rows(W, s_r, bits: int) -> np.ndarray:
    W = _c(W, np.float32)
    rows = W.shape[0]
    cols = W.size // rows
    s = _c(s_r, np.float32)
    assert s.size == rows
    q = np.empty(W.shape, np.int8)
    lib().orc_quantize_rows(_p(W), rows, cols, _p(s), int(bits), _p(q))
    return q


def hist_calib_max(x, bins: int = HIST_BINS, percentile=PERCENTILE):
    """(calib_max, bin index) of the histogram percentile calibrator (A30)."""
    x = _c(x, np.float32)
    cm = ctypes.c_float()
    b = lib().orc_hist_calib(_p(x), x.size, int(bins), int(percentile[0]), int(percentile[1]),
                             ctypes.byref(cm))
    return np.float32(cm.value), int(b)


def dequantize_pc(acc, s_a, s_w, bias=None, channel_axis: int = -1) -> np.ndarray:
    """y = fl(fl(acc * fl(s_a * s_w[ch])) + bias[ch]) (A32)."""
    acc = _c(acc, np.int32)
    y = np.empty(acc.shape, np.float32)
    ax = channel_axis % acc.ndim
    nch = acc.shape[ax]
    inner = int(np.prod(acc.shape[ax + 1:], dtype=np.int64))
    sw = _c(s_w, np.float32)
    assert sw.size == nch
    b = None if bias is None else _c(bias, np.float32)
    lib().orc_dequantize_pc(acc.size, _p(acc), float(np.float32(s_a)), _p(sw),
                            None if b is None else _p(b), nch, inner, _p(y))
    return y


# ---- NEXT-2: wide ACUs (b = 9..12) with int16 operand codes ----

def quantize16(x, s, bits: int) -> np.ndarray:
    x = _c(x, np.float32)
    q = np.empty(x.shape, np.int16)
    lib().orc_quantize16(_p(x), x.size, float(np.float32(s)), int(bits), _p(q))
    return q


def lut_gemm16(A, W, lut, bits: int) -> np.ndarray:
    """A int16 [M][K], W int16 [N][K] codes of b <= 16 bits -> int32 [M][N]."""
    A = _c(A, np.int16)
    W = _c(W, np.int16)
    T = _c(lut, np.int32)
    assert T.size == 1 << (2 * bits)
    M, K = A.shape
    N, K2 = W.shape
    assert K == K2
    C = np.empty((M, N), np.int32)
    bad = lib().orc_lut_gemm16(M, N, K, _p(A), _p(W), int(bits), _p(T), _p(C))
    if bad:
        raise OverflowError("%d outputs exceed int32" % bad)
    return C


# ---- NEXT-4: approximation-aware retraining, the STE backward of an approximate linear layer
#      (§III.A.2; reading A36) ----

def _rows(v, ndim):
    """A per-tensor scalar, or a per-output-channel vector [rows] broadcast along axis 0."""
    v = np.asarray(v, dtype=np.float32)
    return v if v.ndim == 0 else v.reshape((-1,) + (1,) * (ndim - 1))


def fake_quant(q, s) -> np.ndarray:
    """The fake-quantized operand the STE differentiates through: fl32(s * q) ("quantized
    floating point values"); s a scalar or per-row (per-output-channel weight scales, P:95
    "weight ranges are per channel")."""
    q = np.asarray(q)
    return (_rows(s, q.ndim) * q.astype(np.float32)).astype(np.float32)


def ste_linear_backward(gy, qa, s_a, qw, s_w, x=None, clip_a=None, w=None, clip_w=None):
    """Gradients of y = dequant(sum_k LUT[qa][qw]) + b under the straight-through estimator
    (P:107-109): the quantizer and the ACU are the identity in the backward pass, so the layer
    differentiates as y = fq(qa) fq(qw)^T + b, and an input outside its calibrated clip range
    (|v| > clip) gets no gradient.  s_w / clip_w may be per output channel ([N]).  Plain fp64 matrix products of the fp32 operands, one
    rounding to fp32 at the end.  Returns (gx [M][K], gw [N][K], gb [N]) fp32."""
    gy64 = np.asarray(gy, dtype=np.float32).astype(np.float64)
    wf = fake_quant(qw, s_w).astype(np.float64)
    xf = fake_quant(qa, s_a).astype(np.float64)
    gx = gy64 @ wf                      # [M][N] . [N][K]
    gw = gy64.T @ xf                    # [N][M] . [M][K]
    gb = gy64.sum(axis=0)
    if x is not None:
        gx = np.where(np.abs(np.asarray(x, dtype=np.float32)) <= np.float32(clip_a), gx, 0.0)
    if w is not None:
        gw = np.where(np.abs(np.asarray(w, dtype=np.float32)) <= _rows(clip_w, 2), gw, 0.0)
    return gx.astype(np.float32), gw.astype(np.float32), gb.astype(np.float32)


def ste_conv2d_backward(gy, qx, s_a, qw, s_w, stride=(1, 1), pad=(0, 0), x=None, clip_a=None,
                        w=None, clip_w=None):
    """STE backward of an approximate conv (P:107-109 over the conv of P:119; reading A36), NHWC:
    gy [N][Ho][Wo][K], qx [N][H][W][C], qw [K][R][S][C] -> (gx [N][H][W][C], gw [K][R][S][C],
    gb [K]) fp32.  The layer differentiates as the conv of the fake-quantized operands: gw is the
    correlation of the zero-padded fq(x) with gy, gx the transposed conv of gy with fq(w); fp64
    sums, one rounding to fp32; inputs outside their clip get no gradient."""
    gy64 = np.asarray(gy, dtype=np.float32).astype(np.float64)
    xf = fake_quant(qx, s_a).astype(np.float64)
    wf = fake_quant(qw, s_w).astype(np.float64)
    N, H, W, C = xf.shape
    K, R, S, _ = wf.shape
    _, Ho, Wo, _ = gy64.shape
    sh, sw = stride
    ph, pw = pad
    xp = np.zeros((N, H + 2 * ph + sh * R, W + 2 * pw + sw * S, C))
    xp[:, ph:ph + H, pw:pw + W, :] = xf
    gxp = np.zeros_like(xp)
    gw = np.zeros((K, R, S, C))
    for r in range(R):
        for s_ in range(S):
            win = xp[:, r:r + sh * Ho:sh, s_:s_ + sw * Wo:sw, :]          # [N][Ho][Wo][C]
            gw[:, r, s_, :] = np.einsum("nhwk,nhwc->kc", gy64, win)
            gxp[:, r:r + sh * Ho:sh, s_:s_ + sw * Wo:sw, :] += np.einsum("nhwk,kc->nhwc", gy64, wf[:, r, s_, :])
    gx = gxp[:, ph:ph + H, pw:pw + W, :]
    gb = gy64.sum(axis=(0, 1, 2))
    if x is not None:
        gx = np.where(np.abs(np.asarray(x, dtype=np.float32)) <= np.float32(clip_a), gx, 0.0)
    if w is not None:
        gw = np.where(np.abs(np.asarray(w, dtype=np.float32)) <= _rows(clip_w, 4), gw, 0.0)
    return gx.astype(np.float32), gw.astype(np.float32), gb.astype(np.float32)
