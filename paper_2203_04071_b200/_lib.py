"""Thin ctypes binding of libaxq.so (include/axq.h).  Argument marshalling only: every step
of the path runs in the library's CUDA kernels.  Tensors are torch CUDA tensors (PyTorch is
used for device memory and streams only); each wrapper has the C entry point's name.

There is no fallback: if libaxq.so is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libaxq.so"

AXQ_OK, AXQ_ERR_INVALID, AXQ_ERR_OVERFLOW, AXQ_ERR_UNSUPPORTED, AXQ_ERR_CUDA = range(5)
REPR_NAMES = {0: "delta8", 1: "int16", 2: "int32", 3: "wide16", 4: "wide32"}

EXPORTED = [
    "axq_last_cuda_error", "axq_status_string", "axq_version",
    "axq_lut_create", "axq_lut_destroy", "axq_lut_info", "axq_lut_set_i32_resident",
    "axq_amax", "axq_scale", "axq_quantize", "axq_quantize_nchw_to_nhwc",
    "axq_lut_gemm", "axq_lut_gemm_dq",
    "axq_conv2d_out_hw", "axq_lut_conv2d", "axq_lut_conv2d_dq",
    "axq_dequantize", "axq_dequantize_nhwc_to_nchw", "axq_epilogue_apply",
    "axq_maxpool2d_nhwc_i8", "axq_avgpool_nhwc", "axq_lstm_cell",
    "axq_wpack_create", "axq_wpack_destroy", "axq_wpack_info", "axq_lut_gemm_wp",
    "axq_lut_conv2d_wp", "axq_wpack_kernel", "axq_wpack_shapes", "axq_lstm_recurrent",
    "axq_ste_linear_backward", "axq_ste_conv2d_backward",
    "axq_amax_rows", "axq_scale_vec", "axq_quantize_rows", "axq_calib_histogram",
    "axq_calib_percentile", "axq_maxpool2d_nhwc_f32", "axq_quantize16", "axq_lut_gemm16",
    "axq_im2col_nhwc_i8", "axq_wpack_repack", "axq_lut_gemm_xs",
    "axq_last_path", "axq_workspace_elems", "axq_lut_gemm_f32a", "axq_lut_conv2d_f32",
    "axq_wpack16_create", "axq_lut_gemm16_wp", "axq_ste_linear_backward_pc",
    "axq_ste_conv2d_backward_pc", "axq_ste_linear_workspace_elems", "axq_ste_conv2d_workspace_elems",
]

# axq_last_path kernel families (include/axq.h AXQ_PATH_*)
PATH_NAMES = {1: "v1", 2: "p4", 3: "p4w", 4: "gconv", 5: "wide", 6: "lstm_rec", 7: "f32a",
              8: "p4w16", 9: "widepk"}
PATH_SPLITK, PATH_STREAMK, PATH_TMA, PATH_TMA_IM2COL = 0x100, 0x200, 0x400, 0x800


class AxqError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__("%s failed: status %d (%s)" % (fn, status, msg))
        self.status = status


class axq_epilogue(ctypes.Structure):
    _fields_ = [("d_scale_a", ctypes.c_void_p), ("d_scale_w", ctypes.c_void_p),
                ("bias", ctypes.c_void_p), ("y", ctypes.c_void_p), ("ldy", ctypes.c_int64),
                ("workspace", ctypes.c_void_p), ("residual", ctypes.c_void_p),
                ("ldr", ctypes.c_int64), ("relu", ctypes.c_int32), ("y_nhwc", ctypes.c_int32),
                ("q_out", ctypes.c_void_p), ("ldq", ctypes.c_int64),
                ("d_scale_out", ctypes.c_void_p), ("bits_out", ctypes.c_int32),
                ("d_scale_w_ch", ctypes.c_void_p), ("workspace_elems", ctypes.c_int64)]


class axq_conv_desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("N", "H", "W", "C", "K", "R", "S", "stride_h", "stride_w", "pad_h", "pad_w",
                 "dil_h", "dil_w", "groups", "c_valid")]


_lib = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libaxq.so (raises if it has not been built -- there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("AXQ_LIB", LIB_PATH))   # AXQ_LIB: A/B builds
    if not p.exists():
        raise ImportError("libaxq.so not built at %s (run __graft_entry__.build())" % p)
    L = ctypes.CDLL(str(p))
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    sig = {
        "axq_last_cuda_error": ([], i32),
        "axq_status_string": ([i32], ctypes.c_char_p),
        "axq_version": ([], i32),
        "axq_last_path": ([ctypes.POINTER(i32)], i32),
        "axq_workspace_elems": ([i64, i64], i64),
        "axq_ste_linear_workspace_elems": ([i64, i64, i64], i64),
        "axq_ste_conv2d_workspace_elems": ([ctypes.POINTER(axq_conv_desc)], i64),
        "axq_wpack16_create": ([vp, vp, i64, i64, i64, ctypes.POINTER(vp)], i32),
        "axq_lut_gemm16_wp": ([i64, vp, i64, vp, ctypes.POINTER(axq_epilogue), vp, i64, vp], i32),
        "axq_lut_gemm_f32a": ([i64, i64, i64, vp, i64, vp, vp, i64, vp, ctypes.POINTER(axq_epilogue),
                               vp, i64, vp], i32),
        "axq_lut_conv2d_f32": ([ctypes.POINTER(axq_conv_desc), vp, vp, vp, vp,
                                ctypes.POINTER(axq_epilogue), vp, vp], i32),
        "axq_lut_create": ([i32, vp, ctypes.POINTER(vp)], i32),
        "axq_lut_destroy": ([vp], i32),
        "axq_lut_set_i32_resident": ([vp, i32], i32),
        "axq_lut_info": ([vp, ctypes.POINTER(i32), ctypes.POINTER(i32),
                          ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)], i32),
        "axq_amax": ([vp, i64, vp, vp], i32),
        "axq_scale": ([vp, i32, vp, vp], i32),
        "axq_quantize": ([vp, i64, vp, i32, vp, vp], i32),
        "axq_quantize_nchw_to_nhwc": ([vp, i64, i64, i64, i64, i64, vp, i32, vp, vp], i32),
        "axq_lut_gemm": ([i64, i64, i64, vp, i64, vp, i64, vp, vp, i64, vp], i32),
        "axq_lut_gemm_dq": ([i64, i64, i64, vp, i64, vp, i64, vp,
                             ctypes.POINTER(axq_epilogue), vp], i32),
        "axq_conv2d_out_hw": ([ctypes.POINTER(axq_conv_desc), ctypes.POINTER(i64),
                               ctypes.POINTER(i64)], i32),
        "axq_lut_conv2d": ([ctypes.POINTER(axq_conv_desc), vp, vp, vp, vp, vp], i32),
        "axq_lut_conv2d_dq": ([ctypes.POINTER(axq_conv_desc), vp, vp, vp,
                               ctypes.POINTER(axq_epilogue), vp], i32),
        "axq_dequantize": ([i64, i64, vp, i64, vp, vp, vp, vp, i64, vp], i32),
        "axq_dequantize_nhwc_to_nchw": ([i64, i64, i64, vp, vp, vp, vp, vp, vp], i32),
        "axq_epilogue_apply": ([i64, i64, vp, i64, ctypes.POINTER(axq_epilogue), vp], i32),
        "axq_maxpool2d_nhwc_i8": ([vp, i64, i64, i64, i64, i64, i64, i64, i64, vp, vp], i32),
        "axq_avgpool_nhwc": ([vp, i64, i64, i64, vp, vp, vp, i32, vp], i32),
        "axq_lstm_cell": ([i64, i64, vp, vp, vp, vp, vp, vp, i32, vp], i32),
        "axq_wpack_create": ([vp, vp, i64, i64, i64, i32, ctypes.POINTER(vp)], i32),
        "axq_wpack_destroy": ([vp], i32),
        "axq_wpack_kernel": ([i32], i32),
        "axq_wpack_shapes": ([i32, i32, i32], i32),
        "axq_ste_linear_backward": ([i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp], i32),
        "axq_ste_conv2d_backward": ([ctypes.POINTER(axq_conv_desc)] + [vp] * 13 + [i64, vp, vp, i64, vp], i32),
        "axq_ste_linear_backward_pc": ([i64, i64, i64] + [vp] * 15 + [i64, vp], i32),
        "axq_ste_conv2d_backward_pc": ([ctypes.POINTER(axq_conv_desc)] + [vp] * 15 + [i64, vp, vp, i64, vp], i32),
        "axq_amax_rows": ([vp, i64, i64, vp, vp], i32),
        "axq_quantize16": ([vp, i64, vp, i32, vp, vp], i32),
        "axq_im2col_nhwc_i8": ([vp] + [i64] * 11 + [vp, i64, vp], i32),
        "axq_wpack_repack": ([vp, vp, i64, vp], i32),
        "axq_lut_gemm_xs": ([i64, vp, i64, vp, ctypes.POINTER(axq_epilogue), vp, i64, vp], i32),
        "axq_lut_gemm16": ([i64, i64, i64, vp, i64, vp, i64, vp, ctypes.POINTER(axq_epilogue), vp, i64, vp], i32),
        "axq_maxpool2d_nhwc_f32": ([vp, i64, i64, i64, i64, i64, i64, i64, i64, vp, vp], i32),
        "axq_scale_vec": ([vp, i64, i32, vp, vp], i32),
        "axq_quantize_rows": ([vp, i64, i64, vp, i32, vp, vp], i32),
        "axq_calib_histogram": ([vp, i64, vp, i32, vp, vp], i32),
        "axq_calib_percentile": ([vp, i32, i64, vp, i64, i64, i32, vp, vp, vp], i32),
        "axq_lstm_recurrent": ([i64, i64, i64, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp], i32),
        "axq_wpack_info": ([vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "axq_lut_gemm_wp": ([i64, vp, i64, vp, ctypes.POINTER(axq_epilogue), vp, i64, vp], i32),
        "axq_lut_conv2d_wp": ([ctypes.POINTER(axq_conv_desc), vp, vp,
                               ctypes.POINTER(axq_epilogue), vp, vp], i32),
    }
    ab = "AXQ_LIB" in os.environ           # an older A/B build may lack newer entry points
    for name, (args, res) in sig.items():
        if ab and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    v = os.environ.get("AXQ_WPACK_KERNEL")   # measurement switch (include/axq.h axq_wpack_kernel)
    if v:
        if L.axq_wpack_kernel(int(v)) < 0:
            raise ValueError("AXQ_WPACK_KERNEL=%s: unknown packed-table kernel" % v)
    return L


def _check(fn: str, st: int) -> None:
    if st != AXQ_OK:
        L = load()
        msg = L.axq_status_string(st).decode()
        if st == AXQ_ERR_CUDA:
            msg += " (cudaError %d)" % L.axq_last_cuda_error()
        raise AxqError(fn, st, msg)


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------------------------------
# ACU table handle
# ---------------------------------------------------------------------------------------
class Lut:
    """Owns an axq_lut_t (device copy of an ACU table in the chosen representation)."""

    def __init__(self, bits: int, host_table: np.ndarray):
        t = np.ascontiguousarray(host_table, dtype=np.int32)
        if t.size != 1 << (2 * bits):
            raise ValueError("table must have 2^(2*bits) entries")
        h = ctypes.c_void_p()
        _check("axq_lut_create", load().axq_lut_create(int(bits), t.ctypes.data, ctypes.byref(h)))
        self.handle = h
        self.bits = int(bits)
        b, r, lo, hi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int32(), ctypes.c_int32()
        _check("axq_lut_info", load().axq_lut_info(h, ctypes.byref(b), ctypes.byref(r),
                                                   ctypes.byref(lo), ctypes.byref(hi)))
        self.repr = REPR_NAMES[r.value]
        self.tmin, self.tmax = lo.value, hi.value

    def set_i32_resident(self, resident: bool) -> None:
        """int32 tables: SM-resident halves (True) or the L1 gather (False); same results."""
        _check("axq_lut_set_i32_resident", load().axq_lut_set_i32_resident(self.handle, int(resident)))

    def close(self):
        if self.handle is not None and self.handle.value:
            load().axq_lut_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def axq_lut_create(bits: int, host_table: np.ndarray) -> Lut:
    return Lut(bits, host_table)


def _ste_in(t, name, dtype, shape, dev):
    """Read-only STE operand: on the device, of the expected dtype and shape; made contiguous
    (autograd hands out expanded / strided gradients, e.g. stride 0 after y.sum())."""
    import torch
    if t is None:
        return None
    if t.device != dev or t.dtype != dtype or tuple(t.shape) != tuple(shape):
        raise ValueError("%s: expected %s %s on %s, got %s %s on %s"
                         % (name, dtype, tuple(shape), dev, t.dtype, tuple(t.shape), t.device))
    return t if t.is_contiguous() else t.contiguous()


def _ste_out(t, name, shape, dev):
    import torch
    if t is None:
        return None
    if t.device != dev or t.dtype != torch.float32 or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError("%s: expected a contiguous fp32 %s tensor on %s" % (name, tuple(shape), dev))
    return t


def _ste_scalar_or_vec(t, name, n, dev):
    """A device fp32 scale / clip: one element (per tensor) or n (per output channel)."""
    import torch
    if t is None:
        return None, False
    t = _ste_in(t.reshape(-1), name, torch.float32, (t.numel(),), dev)
    if t.numel() not in (1, n):
        raise ValueError("%s: 1 or %d elements, got %d" % (name, n, t.numel()))
    return t, t.numel() == n and n != 1


def axq_ste_linear_backward(gy, qa, d_scale_a, qw, d_scale_w, x=None, d_clip_a=None, w=None,
                            d_clip_w=None, gx=None, gw=None, gb=None, workspace=None,
                            stream=None) -> None:
    """NEXT-4 STE backward of an approximate linear layer (include/axq.h): gy [M][N], qa [M][K],
    qw [N][K] -> gx [M][K], gw [N][K], gb [N] (each optional); workspace: fp32 tensor for
    K-split partial products (optional).  d_scale_w / d_clip_w: 1 element (per tensor) or N
    (per output channel, axq_ste_linear_backward_pc).  Inputs are checked and made contiguous."""
    import torch
    dev = gy.device
    M, N = gy.shape
    K = qa.shape[1] if qa is not None else qw.shape[1]
    gy = _ste_in(gy, "gy", torch.float32, (M, N), dev)
    qa = _ste_in(qa, "qa", torch.int8, (M, K), dev)
    qw = _ste_in(qw, "qw", torch.int8, (N, K), dev)
    x = _ste_in(x, "x", torch.float32, (M, K), dev)
    w = _ste_in(w, "w", torch.float32, (N, K), dev)
    d_scale_a, _ = _ste_scalar_or_vec(d_scale_a, "d_scale_a", 1, dev)
    d_clip_a, _ = _ste_scalar_or_vec(d_clip_a, "d_clip_a", 1, dev)
    sw, sw_vec = _ste_scalar_or_vec(d_scale_w, "d_scale_w", N, dev)
    cw, cw_vec = _ste_scalar_or_vec(d_clip_w, "d_clip_w", N, dev)
    gx, gw, gb = _ste_out(gx, "gx", (M, K), dev), _ste_out(gw, "gw", (N, K), dev), _ste_out(gb, "gb", (N,), dev)
    if workspace is not None and (workspace.dtype != torch.float32 or not workspace.is_contiguous()):
        raise ValueError("workspace: a contiguous fp32 tensor")
    _check("axq_ste_linear_backward_pc", load().axq_ste_linear_backward_pc(
        M, N, K, _ptr(gy), _ptr(qa), _ptr(d_scale_a), _ptr(x), _ptr(d_clip_a), _ptr(qw),
        None if sw_vec else _ptr(sw), _ptr(sw) if sw_vec else None, _ptr(w),
        None if cw_vec else _ptr(cw), _ptr(cw) if cw_vec else None, _ptr(gx), _ptr(gw), _ptr(gb),
        _ptr(workspace), workspace.numel() if workspace is not None else 0, _stream(stream)))


def axq_ste_conv2d_backward(d, gy, qx, d_scale_a, qw, d_scale_w, x=None, d_clip_a=None, w=None,
                            d_clip_w=None, gx=None, gw=None, gb=None, cols=None, gcols=None,
                            workspace=None, stream=None) -> None:
    """NEXT-4 STE backward of an approximate conv (include/axq.h): gy NHWC [N][Ho][Wo][K], qx
    NHWC int8, qw [K][R][S][C] int8 -> gx NHWC, gw [K][R][S][C], gb [K]; cols / gcols are the
    im2col workspaces (allocated here when None).  Shapes are checked against the descriptor
    (the kernel sizes everything from it); d_scale_w / d_clip_w may be per output channel."""
    import torch
    dev = gy.device
    Ho, Wo = axq_conv2d_out_hw(d)
    M, Kc = d.N * Ho * Wo, d.R * d.S * d.C
    gy = _ste_in(gy, "gy", torch.float32, (d.N, Ho, Wo, d.K), dev)
    qx = _ste_in(qx, "qx", torch.int8, (d.N, d.H, d.W, d.C), dev)
    qw = _ste_in(qw, "qw", torch.int8, (d.K, d.R, d.S, d.C), dev)
    x = _ste_in(x, "x", torch.float32, (d.N, d.H, d.W, d.C), dev)
    w = _ste_in(w, "w", torch.float32, (d.K, d.R, d.S, d.C), dev)
    d_scale_a, _ = _ste_scalar_or_vec(d_scale_a, "d_scale_a", 1, dev)
    d_clip_a, _ = _ste_scalar_or_vec(d_clip_a, "d_clip_a", 1, dev)
    sw, sw_vec = _ste_scalar_or_vec(d_scale_w, "d_scale_w", d.K, dev)
    cw, cw_vec = _ste_scalar_or_vec(d_clip_w, "d_clip_w", d.K, dev)
    gx = _ste_out(gx, "gx", (d.N, d.H, d.W, d.C), dev)
    gw = _ste_out(gw, "gw", (d.K, d.R, d.S, d.C), dev)
    gb = _ste_out(gb, "gb", (d.K,), dev)
    if gw is not None and cols is None:
        cols = torch.empty(M, (Kc + 15) // 16 * 16, dtype=torch.int8, device=dev)
    if gx is not None and gcols is None:
        gcols = torch.empty(M, Kc, dtype=torch.float32, device=dev)
    if cols is not None and (cols.dtype != torch.int8 or cols.shape[0] != M or cols.shape[1] < Kc or cols.stride(1) != 1):
        raise ValueError("cols: int8 [M][>= R*S*C] with unit column stride")
    if gcols is not None and (gcols.dtype != torch.float32 or tuple(gcols.shape) != (M, Kc) or not gcols.is_contiguous()):
        raise ValueError("gcols: contiguous fp32 [M][R*S*C]")
    if workspace is not None and (workspace.dtype != torch.float32 or not workspace.is_contiguous()):
        raise ValueError("workspace: a contiguous fp32 tensor")
    _check("axq_ste_conv2d_backward_pc", load().axq_ste_conv2d_backward_pc(
        ctypes.byref(d), _ptr(gy), _ptr(qx), _ptr(d_scale_a), _ptr(x), _ptr(d_clip_a), _ptr(qw),
        None if sw_vec else _ptr(sw), _ptr(sw) if sw_vec else None, _ptr(w),
        None if cw_vec else _ptr(cw), _ptr(cw) if cw_vec else None, _ptr(gx), _ptr(gw), _ptr(gb),
        _ptr(cols), cols.stride(0) if cols is not None else 0, _ptr(gcols), _ptr(workspace),
        workspace.numel() if workspace is not None else 0, _stream(stream)))


def axq_wpack_shapes(main_cw: int = 0, res_cw: int = 0, small_cw: int = 0) -> None:
    """P4W consumer-warp counts (include/axq.h axq_wpack_shapes); 0 leaves a value unchanged."""
    _check("axq_wpack_shapes", load().axq_wpack_shapes(int(main_cw), int(res_cw), int(small_cw)))


def axq_last_path() -> tuple[str, int]:
    """(kernel family, flags) of the calling thread's last LUT launch (include/axq.h)."""
    v = ctypes.c_int()
    _check("axq_last_path", load().axq_last_path(ctypes.byref(v)))
    return PATH_NAMES.get(v.value & 0xff, "none"), v.value & ~0xff


def axq_workspace_elems(M: int, N: int) -> int:
    """Epilogue workspace size (int32 elements) enabling every decomposition for M x N outputs."""
    return int(load().axq_workspace_elems(int(M), int(N)))


def axq_ste_linear_workspace_elems(M: int, N: int, K: int) -> int:
    """STE backward workspace (fp32 elements) for the fastest decomposition (include/axq.h)."""
    return int(load().axq_ste_linear_workspace_elems(int(M), int(N), int(K)))


def axq_ste_conv2d_workspace_elems(d) -> int:
    """STE conv backward workspace (fp32 elements) for the fastest decomposition."""
    return int(load().axq_ste_conv2d_workspace_elems(ctypes.byref(d)))


def axq_wpack_kernel(variant: int) -> int:
    """Select the packed-table kernel (0 default = P4W (P4 for C % 16 != 0 convs), 1 P4, 3 P4W); returns the previous."""
    r = load().axq_wpack_kernel(int(variant))
    if r < 0:
        raise ValueError("unknown packed-table kernel variant %r" % variant)
    return r


def axq_lut_destroy(lut: Lut) -> None:
    lut.close()


# ---------------------------------------------------------------------------------------
# Quantizer
# ---------------------------------------------------------------------------------------
def axq_amax(x, d_amax, stream=None) -> None:
    _check("axq_amax", load().axq_amax(_ptr(x), x.numel(), _ptr(d_amax), _stream(stream)))


def axq_scale(d_amax, bits: int, d_scale, stream=None) -> None:
    _check("axq_scale", load().axq_scale(_ptr(d_amax), int(bits), _ptr(d_scale), _stream(stream)))


def axq_quantize(x, d_scale, bits: int, q, stream=None) -> None:
    assert x.is_contiguous() and q.is_contiguous() and q.numel() == x.numel()
    _check("axq_quantize", load().axq_quantize(_ptr(x), x.numel(), _ptr(d_scale), int(bits),
                                               _ptr(q), _stream(stream)))


def axq_quantize_nchw_to_nhwc(x, d_scale, bits: int, q, stream=None) -> None:
    """x fp32 [N][C][H][W] -> q int8 [N][H][W][Cq] (Cq = q.shape[-1] >= C, pad channels 0)."""
    assert x.is_contiguous() and q.is_contiguous() and x.dim() == 4
    N, C, H, W = x.shape
    _check("axq_quantize_nchw_to_nhwc",
           load().axq_quantize_nchw_to_nhwc(_ptr(x), N, C, H, W, q.shape[-1], _ptr(d_scale),
                                            int(bits), _ptr(q), _stream(stream)))


# ---------------------------------------------------------------------------------------
# LUT GEMM / conv / dequant
# ---------------------------------------------------------------------------------------
def axq_lut_gemm(A, W, lut: Lut, C, stream=None) -> None:
    """A int8 [M][K] (row stride A.stride(0)), W int8 [N][K], C int32 [M][N]."""
    M, K = A.shape
    N = W.shape[0]
    _check("axq_lut_gemm", load().axq_lut_gemm(M, N, K, _ptr(A), A.stride(0), _ptr(W),
                                               W.stride(0), lut.handle, _ptr(C), C.stride(0),
                                               _stream(stream)))


def make_epilogue(d_scale_a, d_scale_w, bias=None, y=None, ldy=0, workspace=None,
                  residual=None, ldr=0, relu=False, y_nhwc=False, q_out=None, ldq=0,
                  d_scale_out=None, bits_out=0, d_scale_w_ch=None) -> axq_epilogue:
    """d_scale_w: the per-tensor weight scale (device scalar); d_scale_w_ch: per-output-channel
    weight scales [N] (NEXT-1), which take precedence when given."""
    if workspace is not None:
        assert workspace.is_cuda and workspace.element_size() == 4 and workspace.is_contiguous()
    ep = axq_epilogue(_ptr(d_scale_a), _ptr(d_scale_w), _ptr(bias), _ptr(y), int(ldy),
                      _ptr(workspace), _ptr(residual), int(ldr), int(bool(relu)),
                      int(bool(y_nhwc)), _ptr(q_out), int(ldq), _ptr(d_scale_out),
                      int(bits_out), _ptr(d_scale_w_ch),
                      int(workspace.numel()) if workspace is not None else 0)
    # the struct holds raw device pointers: keep the tensors alive as long as it lives
    ep._keep = (d_scale_a, d_scale_w, bias, y, workspace, residual, q_out, d_scale_out, d_scale_w_ch)
    return ep


def _epilogue(d_scale_a, d_scale_w, bias, y, ldy, workspace):
    return make_epilogue(d_scale_a, d_scale_w, bias, y, ldy, workspace)


def axq_lut_gemm_dq(A, W, lut: Lut, d_scale_a, d_scale_w, bias, y, workspace=None,
                    stream=None) -> None:
    M, K = A.shape
    N = W.shape[0]
    ep = _epilogue(d_scale_a, d_scale_w, bias, y, y.stride(0), workspace)
    _check("axq_lut_gemm_dq", load().axq_lut_gemm_dq(M, N, K, _ptr(A), A.stride(0), _ptr(W),
                                                     W.stride(0), lut.handle, ctypes.byref(ep),
                                                     _stream(stream)))


def conv_desc(N, H, W, C, K, R, S, stride=(1, 1), pad=(0, 0), dil=(1, 1), groups=1,
              c_valid=0):
    return axq_conv_desc(N, H, W, C, K, R, S, stride[0], stride[1], pad[0], pad[1], dil[0],
                         dil[1], groups, c_valid)


def axq_conv2d_out_hw(desc: axq_conv_desc):
    ho, wo = ctypes.c_int64(), ctypes.c_int64()
    _check("axq_conv2d_out_hw", load().axq_conv2d_out_hw(ctypes.byref(desc), ctypes.byref(ho),
                                                         ctypes.byref(wo)))
    return ho.value, wo.value


def axq_lut_conv2d(desc: axq_conv_desc, X_nhwc, W_krsc, lut: Lut, Y_nhwc, stream=None) -> None:
    _check("axq_lut_conv2d", load().axq_lut_conv2d(ctypes.byref(desc), _ptr(X_nhwc),
                                                   _ptr(W_krsc), lut.handle, _ptr(Y_nhwc),
                                                   _stream(stream)))


def axq_lut_conv2d_dq(desc: axq_conv_desc, X_nhwc, W_krsc, lut: Lut, d_scale_a, d_scale_w,
                      bias, y_nchw, workspace=None, stream=None) -> None:
    ep = _epilogue(d_scale_a, d_scale_w, bias, y_nchw, 0, workspace)
    _check("axq_lut_conv2d_dq", load().axq_lut_conv2d_dq(ctypes.byref(desc), _ptr(X_nhwc),
                                                         _ptr(W_krsc), lut.handle,
                                                         ctypes.byref(ep), _stream(stream)))


def axq_dequantize(acc, d_scale_a, d_scale_w, bias, y, stream=None) -> None:
    M, N = acc.shape
    _check("axq_dequantize", load().axq_dequantize(M, N, _ptr(acc), acc.stride(0),
                                                   _ptr(d_scale_a), _ptr(d_scale_w),
                                                   _ptr(bias), _ptr(y), y.stride(0),
                                                   _stream(stream)))


def axq_dequantize_nhwc_to_nchw(acc_nhwc, d_scale_a, d_scale_w, bias, y_nchw,
                                stream=None) -> None:
    N, H, W, C = acc_nhwc.shape
    _check("axq_dequantize_nhwc_to_nchw",
           load().axq_dequantize_nhwc_to_nchw(N, H * W, C, _ptr(acc_nhwc), _ptr(d_scale_a),
                                              _ptr(d_scale_w), _ptr(bias), _ptr(y_nchw),
                                              _stream(stream)))


def axq_lut_gemm_ep(A, W, lut: Lut, ep: axq_epilogue, stream=None) -> None:
    """axq_lut_gemm_dq with a caller-built epilogue (make_epilogue)."""
    M, K = A.shape
    N = W.shape[0]
    _check("axq_lut_gemm_dq", load().axq_lut_gemm_dq(M, N, K, _ptr(A), A.stride(0), _ptr(W),
                                                     W.stride(0), lut.handle, ctypes.byref(ep),
                                                     _stream(stream)))


def axq_lut_conv2d_ep(desc: axq_conv_desc, X_nhwc, W_krsc, lut: Lut, ep: axq_epilogue,
                      stream=None) -> None:
    _check("axq_lut_conv2d_dq", load().axq_lut_conv2d_dq(ctypes.byref(desc), _ptr(X_nhwc),
                                                         _ptr(W_krsc), lut.handle,
                                                         ctypes.byref(ep), _stream(stream)))


def axq_lut_gemm_f32a(A, d_scale_a, W, lut: Lut, ep: axq_epilogue | None = None, C=None,
                      stream=None) -> None:
    """Quantize-on-load LUT-GEMM: A fp32 [M][K] (row stride A.stride(0)) with its device scale,
    W int8 [N][K]; raw int32 C [M][N] or the fused epilogue."""
    assert A.dtype.is_floating_point and A.element_size() == 4 and A.stride(1) == 1
    M, K = A.shape
    N = W.shape[0]
    _check("axq_lut_gemm_f32a", load().axq_lut_gemm_f32a(
        M, N, K, _ptr(A), A.stride(0), _ptr(d_scale_a), _ptr(W), W.stride(0), lut.handle,
        ctypes.byref(ep) if ep is not None else None, _ptr(C), C.stride(0) if C is not None else 0,
        _stream(stream)))


def axq_lut_conv2d_f32(desc: axq_conv_desc, X_nchw, d_scale_a, W_krsc, lut: Lut,
                       ep: axq_epilogue | None = None, Y_nhwc=None, stream=None) -> None:
    """Quantize-on-load LUT conv: X fp32 NCHW (contiguous) with its device scale."""
    assert X_nchw.is_contiguous() and X_nchw.element_size() == 4
    _check("axq_lut_conv2d_f32", load().axq_lut_conv2d_f32(
        ctypes.byref(desc), _ptr(X_nchw), _ptr(d_scale_a), _ptr(W_krsc), lut.handle,
        ctypes.byref(ep) if ep is not None else None, _ptr(Y_nhwc), _stream(stream)))


def axq_epilogue_apply(acc, ep: axq_epilogue, stream=None) -> None:
    M, N = acc.shape
    _check("axq_epilogue_apply", load().axq_epilogue_apply(M, N, _ptr(acc), acc.stride(0),
                                                           ctypes.byref(ep), _stream(stream)))


def axq_maxpool2d_nhwc_i8(x, R, S, stride, pad, y, stream=None) -> None:
    N, H, W, C = x.shape
    _check("axq_maxpool2d_nhwc_i8", load().axq_maxpool2d_nhwc_i8(
        _ptr(x), N, H, W, C, R, S, stride, pad, _ptr(y), _stream(stream)))


def axq_avgpool_nhwc(x, y=None, q=None, d_scale=None, bits=8, stream=None) -> None:
    """x fp32 [N][H][W][C] (or [N][HW][C]) -> y fp32 [N][C] and/or q int8 [N][C]."""
    N, C = x.shape[0], x.shape[-1]
    HW = x.numel() // (N * C) if N * C else 0
    _check("axq_avgpool_nhwc", load().axq_avgpool_nhwc(_ptr(x), N, HW, C, _ptr(y), _ptr(q),
                                                       _ptr(d_scale), int(bits), _stream(stream)))


def axq_lstm_cell(gates_ih, gates_hh, c, h_out, q_h=None, d_scale_h=None, bits=8,
                  stream=None) -> None:
    B, H4 = gates_hh.shape
    _check("axq_lstm_cell", load().axq_lstm_cell(B, H4 // 4, _ptr(gates_ih), _ptr(gates_hh),
                                                 _ptr(c), _ptr(h_out), _ptr(q_h),
                                                 _ptr(d_scale_h), int(bits), _stream(stream)))


# ---------------------------------------------------------------------------------------
# prepared weights (packed-table kernel)
# ---------------------------------------------------------------------------------------
class WPack:
    """Owns an axq_wpack_t: weight-specialised E tables of a layer (delta8 LUTs only)."""

    def __init__(self, lut: Lut, W, K: int | None = None, a_nonneg: bool = False,
                 activations: bool = False):
        """W: device int8 [N][K] (conv: KRSC flattened).  a_nonneg: every activation code will
        be >= 0 (ReLU outputs) -> half-range tables."""
        N = W.shape[0]
        K = W.numel() // N if K is None else K
        h = ctypes.c_void_p()
        flags = (1 if a_nonneg else 0) | (2 if activations else 0)
        _check("axq_wpack_create", load().axq_wpack_create(lut.handle, _ptr(W), N, K,
                                                           W.stride(0), flags, ctypes.byref(h)))
        self.a_nonneg = bool(a_nonneg)
        self.handle = h
        self.N, self.K = N, K
        nb = ctypes.c_int64()
        load().axq_wpack_info(h, None, None, ctypes.byref(nb))
        self.device_bytes = nb.value

    def close(self):
        if self.handle is not None and self.handle.value:
            load().axq_wpack_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


P4_BM, P4_TN = 1024, 16


def prefer_packed(M: int, N: int, n_sms: int) -> bool:
    """Packed-table kernel from 1024 rows up (it picks 1024- or 512-row tiles and a K split
    itself, axq p4_plan); below that the per-row-gather kernel wastes fewer lanes."""
    return M >= P4_BM


def axq_wpack_create(lut: Lut, W) -> WPack:
    return WPack(lut, W)


def axq_lut_gemm_wp(A, wp: WPack, ep: axq_epilogue | None = None, C=None, stream=None) -> None:
    """A int8 [M][K] (16-byte aligned rows) with prepared weights; ep or raw int32 C."""
    M = A.shape[0]
    _check("axq_lut_gemm_wp", load().axq_lut_gemm_wp(
        M, _ptr(A), A.stride(0), wp.handle, ctypes.byref(ep) if ep is not None else None,
        _ptr(C), C.stride(0) if C is not None else 0, _stream(stream)))


def axq_lut_conv2d_wp(desc: axq_conv_desc, X_nhwc, wp: WPack, ep: axq_epilogue | None = None,
                      Y=None, stream=None) -> None:
    _check("axq_lut_conv2d_wp", load().axq_lut_conv2d_wp(
        ctypes.byref(desc), _ptr(X_nhwc), wp.handle, ctypes.byref(ep) if ep is not None else None,
        _ptr(Y), _stream(stream)))


def axq_lstm_recurrent(gates_ih, qw_hh, d_scale_w_hh, b_hh, d_scale_h, bits: int, lut: Lut, hs, c_out,
                       workspace, stream=None) -> None:
    """The static-scale LSTM recurrence in one persistent launch (include/axq.h).  Raises
    AxqError with status AXQ_ERR_UNSUPPORTED when the shape cannot run co-resident."""
    T, B, H = hs.shape
    _check("axq_lstm_recurrent", load().axq_lstm_recurrent(
        T, B, H, _ptr(gates_ih), _ptr(qw_hh), _ptr(d_scale_w_hh), _ptr(b_hh), _ptr(d_scale_h),
        int(bits), lut.handle, _ptr(hs), _ptr(c_out), _ptr(workspace), _stream(stream)))


# ---- NEXT-1: the paper's quantizer (per-channel weights, 99.9 % histogram calib_max) ----
HIST_BINS = 2048
PERCENTILE = (999, 1000)


def axq_amax_rows(W, d_amax, stream=None) -> None:
    rows = W.shape[0]
    _check("axq_amax_rows", load().axq_amax_rows(_ptr(W), rows, W.numel() // rows, _ptr(d_amax),
                                                 _stream(stream)))


def axq_scale_vec(d_amax, bits: int, d_scale, stream=None) -> None:
    _check("axq_scale_vec", load().axq_scale_vec(_ptr(d_amax), d_amax.numel(), int(bits), _ptr(d_scale),
                                                 _stream(stream)))


def axq_quantize_rows(W, d_scale_rows, bits: int, q, stream=None) -> None:
    rows = W.shape[0]
    _check("axq_quantize_rows", load().axq_quantize_rows(_ptr(W), rows, W.numel() // rows,
                                                         _ptr(d_scale_rows), int(bits), _ptr(q),
                                                         _stream(stream)))


def axq_calib_histogram(x, d_amax, d_hist, stream=None) -> None:
    _check("axq_calib_histogram", load().axq_calib_histogram(_ptr(x), x.numel(), _ptr(d_amax),
                                                             d_hist.numel(), _ptr(d_hist), _stream(stream)))


def axq_calib_percentile(d_hist, n: int, d_amax, bits: int, d_calib_max=None, d_scale=None,
                         percentile=PERCENTILE, stream=None) -> None:
    _check("axq_calib_percentile", load().axq_calib_percentile(
        _ptr(d_hist), d_hist.numel(), int(n), _ptr(d_amax), int(percentile[0]), int(percentile[1]),
        int(bits), _ptr(d_calib_max), _ptr(d_scale), _stream(stream)))


def axq_maxpool2d_nhwc_f32(x, R: int, S: int, stride: int, pad: int, y, stream=None) -> None:
    N, H, W, C = x.shape
    _check("axq_maxpool2d_nhwc_f32", load().axq_maxpool2d_nhwc_f32(
        _ptr(x), N, H, W, C, R, S, stride, pad, _ptr(y), _stream(stream)))


# ---- NEXT-2: wide ACUs (b = 9..12) with int16 codes ----
def axq_quantize16(x, d_scale, bits: int, q, stream=None) -> None:
    assert q.dtype == __import__("torch").int16 and q.numel() == x.numel()
    _check("axq_quantize16", load().axq_quantize16(_ptr(x), x.numel(), _ptr(d_scale), int(bits), _ptr(q),
                                                   _stream(stream)))


def axq_lut_gemm16(A, W, lut: Lut, ep: axq_epilogue | None = None, C=None, stream=None) -> None:
    """A int16 [M][K], W int16 [N][K] codes; raw int32 C [M][N] or the fused epilogue."""
    M, K = A.shape
    N = W.shape[0]
    _check("axq_lut_gemm16", load().axq_lut_gemm16(
        M, N, K, _ptr(A), A.stride(0), _ptr(W), W.stride(0), lut.handle,
        ctypes.byref(ep) if ep is not None else None, _ptr(C), C.stride(0) if C is not None else 0,
        _stream(stream)))


class WPack16:
    """Owns a wide (b = 9..12) weight pack: the table tiled by the weights (axq_wpack16_create)."""

    def __init__(self, lut: Lut, W):
        """W: device int16 codes [N][K] of a WIDE16 handle's bit width."""
        assert W.dtype.itemsize == 2 and W.stride(1) == 1
        N, K = W.shape
        h = ctypes.c_void_p()
        _check("axq_wpack16_create", load().axq_wpack16_create(lut.handle, _ptr(W), N, K, W.stride(0),
                                                               ctypes.byref(h)))
        self.handle = h
        self.N, self.K = N, K

    def close(self):
        if self.handle is not None and self.handle.value:
            load().axq_wpack_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def axq_lut_gemm16_wp(A, wp: WPack16, ep: axq_epilogue | None = None, C=None, stream=None) -> None:
    """A int16 codes [M][K] with a wide weight pack; raw int32 C [M][N] or the fused epilogue."""
    M = A.shape[0]
    _check("axq_lut_gemm16_wp", load().axq_lut_gemm16_wp(
        M, _ptr(A), A.stride(0), wp.handle, ctypes.byref(ep) if ep is not None else None, _ptr(C),
        C.stride(0) if C is not None else 0, _stream(stream)))


def axq_im2col_nhwc_i8(X, c_valid: int, R: int, S: int, stride, pad, A, stream=None) -> None:
    """Explicit im2col of int8 NHWC codes into A [M][lda] (k = (r, s, c), zero padded)."""
    N, H, W, C = X.shape
    _check("axq_im2col_nhwc_i8", load().axq_im2col_nhwc_i8(
        _ptr(X), N, H, W, C, int(c_valid), R, S, stride[0], stride[1], pad[0], pad[1], _ptr(A),
        A.stride(0), _stream(stream)))


def axq_wpack_repack(wp: WPack, W, stream=None) -> None:
    _check("axq_wpack_repack", load().axq_wpack_repack(wp.handle, _ptr(W), W.stride(0), _stream(stream)))


def axq_lut_gemm_xs(W, xp: WPack, ep: axq_epilogue | None = None, C=None, stream=None) -> None:
    """acc[m][n] = sum_k LUT[x[m][k]][W[n][k]] with x packed in xp (activations=True)."""
    N = W.shape[0]
    _check("axq_lut_gemm_xs", load().axq_lut_gemm_xs(
        N, _ptr(W), W.stride(0), xp.handle, ctypes.byref(ep) if ep is not None else None, _ptr(C),
        C.stride(0) if C is not None else 0, _stream(stream)))
