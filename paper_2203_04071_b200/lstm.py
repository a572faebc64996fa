"""One-layer LSTM with approximate gate GEMMs on the C ABI (BASELINE.json configs[4]).

"We implemented the feedback loop in the recurrent layer ... mathematically equivalent with
the vanilla Pytorch RNN layer.  It also utilizes our custom Linear layer": the
input projection x_t W_ih^T and the recurrent projection h_{t-1} W_hh^T are two separately
quantized approximate Linears (own input and weight scales, A18), gates in PyTorch order
i, f, g, o.  The input projection of all T steps is hoisted into one LUT-GEMM
(M = T*B); each step runs one LUT-GEMM (M = B) with the bias epilogue and one cell kernel
that applies the pinned sigmoid / tanh, updates c and writes h both in fp32 and as int8 codes
for the next step (static scale).  The static (calibrated) forward runs the whole recurrence
in ONE persistent launch (axq_lstm_recurrent: each CTA owns hidden units, a grid barrier per
step) when the shape fits; the per-step chain remains for calibration and other shapes.  The
static forward can be captured in a CUDA graph.

calibrate(x): every quantization dynamic (per-tensor max of that tensor); s_x = scale of
max|x| over all steps, s_h = scale of max_t max|h_t| (reading A7').
"""
from __future__ import annotations

import torch

from . import _lib as ax


class ApproxLSTM:
    def __init__(self, W_ih, W_hh, b_ih, b_hh, lut: ax.Lut, device="cuda"):
        self.dev = torch.device(device)
        self.lut, self.bits = lut, lut.bits
        f32 = torch.float32

        def prep(w):
            w = torch.as_tensor(w).to(self.dev, f32).contiguous()
            a, s = torch.empty(1, device=self.dev), torch.empty(1, device=self.dev)
            q = torch.empty(w.shape, dtype=torch.int8, device=self.dev)
            ax.axq_amax(w, a)
            ax.axq_scale(a, self.bits, s)
            ax.axq_quantize(w, s, self.bits, q)
            return q, s

        self.qw_ih, self.sw_ih = prep(W_ih)
        self.qw_hh, self.sw_hh = prep(W_hh)
        self.b_ih = torch.as_tensor(b_ih).to(self.dev, f32).contiguous()
        self.b_hh = torch.as_tensor(b_hh).to(self.dev, f32).contiguous()
        self.H4, self.I = self.qw_ih.shape
        self.H = self.H4 // 4
        # prepared weights for the hoisted input projection (large M) on the packed-table kernel
        self.wp_ih = ax.WPack(lut, self.qw_ih) if (lut.repr == "delta8" and self.I % 16 == 0) else None
        self.n_sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.s_x = torch.ones(1, device=self.dev)
        self.s_h = torch.ones(1, device=self.dev)
        self._tmp_amax = torch.zeros(1, device=self.dev)
        self._tmp_scale = torch.ones(1, device=self.dev)
        self._bufs = {}
        self.calibrated = False
        self.timing_hook = None     # optional callable(kind, stream) around every LUT launch
        # static forward: the whole recurrence in one persistent launch (axq_lstm_recurrent)
        # when the shape allows it; "steps" forces one LUT-GEMM + one cell launch per step
        self.recurrent = "auto"
        self._persistent_ok = lut.repr == "delta8"

    def _hook(self, kind, stream):
        if self.timing_hook:
            self.timing_hook(kind, stream)

    def _buffers(self, T, B):
        key = (T, B)
        if key not in self._bufs:
            d, f32, i8 = self.dev, torch.float32, torch.int8
            self._bufs[key] = dict(
                qx=torch.empty(T * B, self.I, dtype=i8, device=d),
                gih=torch.empty(T * B, self.H4, dtype=f32, device=d),
                ghh=torch.empty(B, self.H4, dtype=f32, device=d),
                qh=torch.empty(B, self.H, dtype=i8, device=d),
                hs=torch.empty(T, B, self.H, dtype=f32, device=d),
                h0=torch.zeros(B, self.H, dtype=f32, device=d),
                c=torch.empty(B, self.H, dtype=f32, device=d),
                ws_ih=torch.zeros(ax.axq_workspace_elems(T * B, self.H4), dtype=torch.int32, device=d),
                ws=torch.zeros(ax.axq_workspace_elems(B, self.H4), dtype=torch.int32, device=d),
                ws_rec=torch.empty(2 * B * self.H + 256, dtype=torch.int8, device=d))
        return self._bufs[key]

    def run(self, x: torch.Tensor, calibrate: bool, stream=None):
        """x fp32 [T][B][I] on the device -> (hs fp32 [T][B][H], c_T fp32 [B][H])."""
        if stream is None:
            stream = torch.cuda.current_stream(self.dev)
        T, B, I = x.shape
        b = self._buffers(T, B)
        bits = self.bits
        x2 = x.reshape(T * B, I)
        if calibrate:
            ax.axq_amax(x2, self._tmp_amax, stream)
            ax.axq_scale(self._tmp_amax, bits, self.s_x, stream)
        ax.axq_quantize(x2, self.s_x, bits, b["qx"], stream)
        gih = b["gih"]
        ep = ax.make_epilogue(self.s_x, self.sw_ih, bias=self.b_ih, y=gih, ldy=self.H4,
                              workspace=b["ws_ih"])
        self._hook("pre", stream)
        if self.wp_ih is not None and ax.prefer_packed(T * B, self.H4, self.n_sms):
            ax.axq_lut_gemm_wp(b["qx"], self.wp_ih, ep, stream=stream)
        else:
            ax.axq_lut_gemm_ep(b["qx"], self.qw_ih, self.lut, ep, stream)
        self._hook("post", stream)
        c, qh, ghh, hs = b["c"], b["qh"], b["ghh"], b["hs"]
        if not calibrate and self.recurrent == "auto" and self._persistent_ok:
            self._hook("pre", stream)
            try:
                ax.axq_lstm_recurrent(gih, self.qw_hh, self.sw_hh, self.b_hh, self.s_h, bits,
                                      self.lut, hs, c, b["ws_rec"], stream)
                self._hook("post", stream)
                return hs, c
            except ax.AxqError as e:          # shape not co-resident: per-step launches
                if e.status != ax.AXQ_ERR_UNSUPPORTED:
                    raise
                self._persistent_ok = False
                self._hook("post", stream)
        with torch.cuda.stream(stream):
            c.zero_()
            qh.zero_()
        ep_hh = ax.make_epilogue(self._tmp_scale if calibrate else self.s_h, self.sw_hh,
                                 bias=self.b_hh, y=ghh, ldy=self.H4, workspace=b["ws"])
        for t in range(T):
            if calibrate:
                h_prev = b["h0"] if t == 0 else hs[t - 1]
                ax.axq_amax(h_prev, self._tmp_amax, stream)
                ax.axq_scale(self._tmp_amax, bits, self._tmp_scale, stream)
                ax.axq_quantize(h_prev, self._tmp_scale, bits, qh, stream)
            self._hook("pre", stream)
            ax.axq_lut_gemm_ep(qh, self.qw_hh, self.lut, ep_hh, stream)
            self._hook("post", stream)
            g_t = gih[t * B:(t + 1) * B]
            if calibrate:
                ax.axq_lstm_cell(g_t, ghh, c, hs[t], stream=stream)
            else:
                ax.axq_lstm_cell(g_t, ghh, c, hs[t], q_h=qh, d_scale_h=self.s_h, bits=bits,
                                 stream=stream)
        if calibrate:
            ax.axq_amax(hs, self._tmp_amax, stream)
            ax.axq_scale(self._tmp_amax, bits, self.s_h, stream)
            self.calibrated = True
        return hs, c

    def calibrate(self, x, stream=None):
        return self.run(x, True, stream)

    def forward(self, x, stream=None):
        assert self.calibrated, "calibrate() first (static scales)"
        return self.run(x, False, stream)

    def capture(self, x):
        """Record the static forward on x (a fixed device buffer) as a CUDA graph: the 128
        sequential steps are ~4 short launches each, which the host cannot issue as fast as the
        GPU runs them.  Returns a replay callable (same results as forward(x))."""
        assert self.calibrated, "calibrate() first (static scales)"
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self.run(x, False, side)           # warm-up: kernel attributes, workspaces
        torch.cuda.current_stream(self.dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.run(x, False, torch.cuda.current_stream(self.dev))
        self._graph = g

        def replay():
            g.replay()
            return out
        return replay

    __call__ = forward

    def lookups(self, T, B) -> int:
        return T * B * self.H4 * self.I + T * B * self.H4 * self.H
