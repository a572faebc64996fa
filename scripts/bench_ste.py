"""NEXT-4 measurement: the STE backward of an approximate linear layer (axq_ste_linear_backward:
gx, gw, gb with clip masks) on BJ configs[1]'s shape and the ResNet fc, L2 flushed before each
call.  Prints one JSON object: ms, GFLOP/s (2 GEMMs x 2 M N K flops) and the fraction of the
fp32 FMA peak (148 SMs x 128 lanes x 2 flops x 1.965 GHz = 74.4 TFLOP/s)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

PEAK = 148 * 128 * 2 * 1.965e9
# bf16 dense tensor-core peak (MEASURED_PEAKS.json sustained cuBLAS bf16, when present)
try:
    BF16 = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["bf16_tflops_sustained"] * 1e12
except Exception:
    BF16 = 2.25e15
MMA_TERMS = 3     # the fp32 operand enters as three bf16 terms (hi + mid + lo): 3 MMAs per useful MAC


def run(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(1)
    gy = torch.randn(M, N, device="cuda", generator=g)
    x = torch.randn(M, K, device="cuda", generator=g)
    w = torch.randn(N, K, device="cuda", generator=g) * 0.02
    qa = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda", generator=g)
    qw = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda", generator=g)
    s = torch.tensor([0.01], device="cuda")
    clip = torch.tensor([3.0], device="cuda")
    gx, gw, gb = torch.empty(M, K, device="cuda"), torch.empty(N, K, device="cuda"), torch.empty(N, device="cuda")
    ws = torch.empty(max(1, ax.axq_ste_linear_workspace_elems(M, N, K)), device="cuda")
    flush = torch.empty(64 << 20, device="cuda")
    ts = []
    for i in range(13):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        ax.axq_ste_linear_backward(gy, qa, s, qw, s, x=x, d_clip_a=clip, w=w, d_clip_w=clip,
                                   gx=gx, gw=gw, gb=gb, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    fl = 2 * 2 * M * N * K
    return {"M": M, "N": N, "K": K, "ws_mib": round(ws.numel() * 4 / 2**20, 1), "ms": round(ms, 4), "gflops": round(fl / ms / 1e6, 1),
            "frac_fp32_fma_peak": round(fl / (ms * 1e-3) / PEAK, 3),
            "frac_bf16_peak_useful": round(fl / (ms * 1e-3) / BF16, 4),
            "frac_bf16_peak_executed": round(MMA_TERMS * fl / (ms * 1e-3) / BF16, 4)}


def run_conv(N, C, H, K, R, st):
    pd = R // 2
    Ho = (H + 2 * pd - R) // st + 1
    g = torch.Generator(device="cuda").manual_seed(2)
    gy = torch.randn(N, Ho, Ho, K, device="cuda", generator=g)
    qx = torch.randint(-127, 128, (N, H, H, C), dtype=torch.int8, device="cuda", generator=g)
    qw = torch.randint(-127, 128, (K, R, R, C), dtype=torch.int8, device="cuda", generator=g)
    s = torch.tensor([0.01], device="cuda")
    gx, gw, gb = torch.empty(N, H, H, C, device="cuda"), torch.empty(K, R, R, C, device="cuda"), torch.empty(K, device="cuda")
    M, Kc = N * Ho * Ho, R * R * C
    cols = torch.empty(M, (Kc + 15) // 16 * 16, dtype=torch.int8, device="cuda")
    gcols = torch.empty(M, Kc, device="cuda")
    d = ax.conv_desc(N, H, H, C, K, R, R, (st, st), (pd, pd))
    ws = torch.empty(max(1, ax.axq_ste_conv2d_workspace_elems(d)), device="cuda")
    flush = torch.empty(64 << 20, device="cuda")
    ts = []
    for i in range(8):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        ax.axq_ste_conv2d_backward(d, gy, qx, s, qw, s, gx=gx, gw=gw, gb=gb, cols=cols, gcols=gcols, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    fl = 2 * 2 * M * K * Kc
    return {"conv": [N, C, H, K, R, st], "ws_mib": round(ws.numel() * 4 / 2**20, 1), "ms": round(ms, 4), "gflops": round(fl / ms / 1e6, 1),
            "frac_fp32_fma_peak": round(fl / (ms * 1e-3) / PEAK, 3),
            "frac_bf16_peak_useful": round(fl / (ms * 1e-3) / BF16, 4),
            "frac_bf16_peak_executed": round(MMA_TERMS * fl / (ms * 1e-3) / BF16, 4)}


if __name__ == "__main__":
    out = {"metric": "STE backward (NEXT-4) GFLOP/s", "peak_tflops_fp32_fma": round(PEAK / 1e12, 1),
           "shapes": [run(256, 1024, 1024), run(256, 1000, 2048), run(2048, 4096, 1024)],
           "conv_shapes": [run_conv(32, 64, 56, 64, 3, 1), run_conv(32, 256, 14, 256, 3, 1)]}
    print(json.dumps(out))
