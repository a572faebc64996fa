"""Approximate layers built from the C ABI (the "approximate layer library" of PAPER.md:113-141,
§III.B, reduced to what the hot path needs).  Each forward runs the §8(a) steps in order --
amax -> scale -> quantize -> LUT-GEMM/conv -> dequantize(+bias) -- every one of them a
libaxq kernel on the caller's stream; torch only allocates device memory.

Weight preparation (amax_w, scale_w, quantize, relayout) happens once at construction and is
not part of a timed step (the paper calibrates offline).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as ax


class ApproxLinear:
    """y = x W^T + b with every multiply a LUT lookup."""

    def __init__(self, weight: torch.Tensor, bias: torch.Tensor | None, lut: ax.Lut,
                 device="cuda"):
        self.lut = lut
        self.bits = lut.bits
        w = weight.to(device=device, dtype=torch.float32).contiguous()
        self.N, self.K = w.shape
        self.d_amax_w = torch.empty(1, device=device)
        self.d_scale_w = torch.empty(1, device=device)
        self.qw = torch.empty(self.N, self.K, dtype=torch.int8, device=device)
        ax.axq_amax(w, self.d_amax_w)
        ax.axq_scale(self.d_amax_w, self.bits, self.d_scale_w)
        ax.axq_quantize(w, self.d_scale_w, self.bits, self.qw)
        self.bias = None if bias is None else bias.to(device=device, dtype=torch.float32).contiguous()
        self.d_amax_a = torch.empty(1, device=device)
        self.d_scale_a = torch.empty(1, device=device)
        self._bufs = {}

    # Kernel path by input rows M (xspec: None = automatic, True / False force the
    # activation-specialised path).  Measured (L2 flushed), e.g. K = 1024, N = 1024:
    #   M = 128: per-row gather 54 us = activation-specialised 55 us
    #   M = 256: gather 79, activation-specialised tables (build 17 + 512-row P4W 49) 68 us
    #   M = 512: gather 118, weight-specialised packed tables (512-row P4W) 77 us
    # and at K = 2048, N = 1000 (the ResNet fc): M = 32 gather 48 vs 77; M = 256 gather 132 vs 110.
    xspec = None
    XS_MIN_M, WP_MIN_M = 192, 384

    def _packable(self) -> bool:
        return self.lut.repr == "delta8" and self.K % 16 == 0 and self.K >= 64 and self.N >= 256

    def path(self, M: int) -> str:
        """'gather' (per-row gather kernel), 'xspec' (tables of this call's activations, built
        per call) or 'wpack' (tables of the weights, built once)."""
        if self.xspec is True and self._packable() and M <= 2048:
            return "xspec"
        if self.xspec is False or not self._packable():
            return "gather"
        if self.XS_MIN_M <= M < self.WP_MIN_M and self.N >= 2 * M:
            return "xspec"
        if M >= self.WP_MIN_M:
            return "wpack"
        return "gather"

    def use_xspec(self, M: int) -> bool:
        return self.path(M) == "xspec"

    def buffers(self, M: int, device):
        b = self._bufs.get(M)
        if b is None:
            b = dict(qa=torch.empty(M, self.K, dtype=torch.int8, device=device),
                     ws=torch.zeros(ax.axq_workspace_elems(M, self.N), dtype=torch.int32,
                                            device=device))
            pth = self.path(M)
            if pth == "xspec":
                # per-call activation tables (M x K x 1 KiB / 4 B) and their packed operand tile
                b["xp"] = ax.WPack(self.lut, b["qa"], activations=True)
            elif pth == "wpack" and self._wp is None:
                self._wp = ax.WPack(self.lut, self.qw)          # 256 x K x N bytes, once
            self._bufs[M] = b
        return b

    _wp = None

    def gemm_q(self, qa, d_scale_a, y, stream=None, hook=None):
        """LUT-GEMM + fused dequantize + bias of the quantized input qa [M][K] into y [M][N]."""
        M = qa.shape[0]
        b = self.buffers(M, qa.device)
        pth = self.path(M)
        if hook:
            hook("pre", stream)
        if pth == "xspec":
            ax.axq_wpack_repack(b["xp"], qa, stream)           # tables of this call's activations
            ep = ax.make_epilogue(d_scale_a, self.d_scale_w, bias=self.bias, y=y, ldy=y.stride(0),
                                  workspace=b["ws"])
            ax.axq_lut_gemm_xs(self.qw, b["xp"], ep, stream=stream)
        elif pth == "wpack":
            ep = ax.make_epilogue(d_scale_a, self.d_scale_w, bias=self.bias, y=y, ldy=y.stride(0),
                                  workspace=b["ws"])
            ax.axq_lut_gemm_wp(qa, self._wp, ep, stream=stream)
        else:
            ax.axq_lut_gemm_dq(qa, self.qw, self.lut, d_scale_a, self.d_scale_w, self.bias, y,
                               workspace=b["ws"], stream=stream)
        if hook:
            hook("post", stream)

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None, d_scale_a=None):
        """x fp32 [M][K] -> y fp32 [M][N].  With d_scale_a given (static calibration), the
        amax/scale steps are skipped."""
        M = x.shape[0]
        b = self.buffers(M, x.device)
        if y is None:
            y = torch.empty(M, self.N, dtype=torch.float32, device=x.device)
        if d_scale_a is None:
            ax.axq_amax(x, self.d_amax_a)
            ax.axq_scale(self.d_amax_a, self.bits, self.d_scale_a)
            d_scale_a = self.d_scale_a
        ax.axq_quantize(x, d_scale_a, self.bits, b["qa"])
        self.gemm_q(b["qa"], d_scale_a, y)
        return y

    __call__ = forward


class ApproxConv2d:
    """Conv2d with every multiply a LUT lookup; NCHW fp32 in/out, implicit im2col."""

    def __init__(self, weight: torch.Tensor, bias: torch.Tensor | None, lut: ax.Lut,
                 stride=(1, 1), padding=(0, 0), device="cuda", packed=True, a_nonneg=False, groups=1):
        """a_nonneg: the layer input is non-negative (e.g. a ReLU output), so its codes are >= 0
        and the packed kernel may use half-range tables.  groups (NEXT-3): weight [K][C/G][R][S];
        packed tables when C/G and K/G are multiples of 16, else the grouped resident-table path."""
        self.lut = lut
        self.bits = lut.bits
        w = weight.to(device=device, dtype=torch.float32).contiguous()   # [K][C/G][R][S]
        self.Kout, cg, self.R, self.S = w.shape
        self.groups = int(groups)
        self.C = cg * self.groups
        self.stride, self.padding = tuple(stride), tuple(padding)
        self.d_amax_w = torch.empty(1, device=device)
        self.d_scale_w = torch.empty(1, device=device)
        q = torch.empty(w.shape, dtype=torch.int8, device=device)
        ax.axq_amax(w, self.d_amax_w)
        ax.axq_scale(self.d_amax_w, self.bits, self.d_scale_w)
        ax.axq_quantize(w, self.d_scale_w, self.bits, q)
        self.qw_kcrs = q
        self.qw = q.permute(0, 2, 3, 1).contiguous()                      # KRSC relayout
        self.bias = None if bias is None else bias.to(device=device, dtype=torch.float32).contiguous()
        self.wp = None
        grp_ok = self.groups == 1 or (cg % 16 == 0 and (self.Kout // self.groups) % 16 == 0 and lut.repr == "delta8")
        if packed and grp_ok and self.C % 16 == 0 and cg * self.R * self.S >= 128:
            # delta8 tables: packed int8 E (P4W); other ACUs with |E| < 2^15 and non-negative
            # inputs: packed int16 E (P4W16); otherwise the resident-table kernel
            if lut.repr == "delta8":
                self.wp = ax.WPack(lut, self.qw.reshape(self.Kout, -1), a_nonneg=a_nonneg)
            elif a_nonneg:
                try:
                    self.wp = ax.WPack(lut, self.qw.reshape(self.Kout, -1), a_nonneg=True)
                except ax.AxqError as e:
                    if e.status != ax.AXQ_ERR_UNSUPPORTED:
                        raise
        self.n_sms = torch.cuda.get_device_properties(torch.device(device)).multi_processor_count
        self.d_amax_a = torch.empty(1, device=device)
        self.d_scale_a = torch.empty(1, device=device)
        self._bufs = {}

    def desc(self, N, H, W):
        return ax.conv_desc(N, H, W, self.C, self.Kout, self.R, self.S, self.stride, self.padding,
                            groups=self.groups)

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None, d_scale_a=None):
        N, C, H, W = x.shape
        d = self.desc(N, H, W)
        Ho, Wo = ax.axq_conv2d_out_hw(d)
        key = (N, H, W)
        b = self._bufs.get(key)
        if b is None:
            b = dict(qx=torch.empty(N, H, W, C, dtype=torch.int8, device=x.device))
            self._bufs[key] = b
        if y is None:
            y = torch.empty(N, self.Kout, Ho, Wo, dtype=torch.float32, device=x.device)
        if d_scale_a is None:
            ax.axq_amax(x, self.d_amax_a)
            ax.axq_scale(self.d_amax_a, self.bits, self.d_scale_a)
            d_scale_a = self.d_scale_a
        ax.axq_quantize_nchw_to_nhwc(x, d_scale_a, self.bits, b["qx"])
        self.conv_q(d, b["qx"], d_scale_a, y)
        return y

    def conv_q(self, d, qx, d_scale_a, y, stream=None):
        """LUT conv of int8 NHWC codes with the fused dequant epilogue to fp32 NCHW y (keeps
        every epilogue tensor referenced until the launch)."""
        Ho, Wo = ax.axq_conv2d_out_hw(d)
        if self.wp is not None and ax.prefer_packed(d.N * Ho * Wo, self.Kout, self.n_sms):
            ep = ax.make_epilogue(d_scale_a, self.d_scale_w, bias=self.bias, y=y)
            ax.axq_lut_conv2d_wp(d, qx, self.wp, ep, stream=stream)
        else:
            ax.axq_lut_conv2d_dq(d, qx, self.qw, self.lut, d_scale_a, self.d_scale_w, self.bias, y,
                                 stream=stream)

    __call__ = forward
