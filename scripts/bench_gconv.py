"""NEXT-3 measurement: a MobileNet-style depthwise 3x3 layer (128 x 256 x 56 x 56, stride 1,
pad 1, fused dequantize + ReLU + requantize, int8 NHWC out) and a ShuffleNet-style grouped 1x1
(G = 4, 256 -> 256), CUDA events after warm-up; lookups/s against the 9.306 T/s smem-lookup
roofline and HBM bytes/s against MEASURED_PEAKS.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
rng = np.random.default_rng(0)
try:
    hbm = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    hbm = 6650.0
for name, (N, C, H, K, R, G) in {"depthwise3x3": (128, 256, 56, 256, 3, 256),
                                  "grouped1x1_G4": (128, 256, 56, 256, 1, 4)}.items():
    x = torch.from_numpy(rng.integers(0, 100, (N, H, H, C)).astype(np.int8)).cuda()
    w = torch.from_numpy(rng.integers(-60, 60, (K, R, R, C // G)).astype(np.int8)).cuda()
    d = ax.conv_desc(N, H, H, C, K, R, R, (1, 1), (R // 2, R // 2), groups=G)
    M = N * H * H
    q = torch.empty(M, K, dtype=torch.int8, device="cuda")
    sa, sw, so = (torch.tensor([v], device="cuda") for v in (0.01, 0.01, 0.05))
    ep = ax.make_epilogue(sa, sw, relu=True, y_nhwc=True, q_out=q, ldq=K, d_scale_out=so, bits_out=8)
    for _ in range(3):
        ax.axq_lut_conv2d_ep(d, x, w, lut, ep)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        ax.axq_lut_conv2d_ep(d, x, w, lut, ep)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    lookups = M * K * R * R * (C // G)
    byts = x.numel() + q.numel()
    print(json.dumps({"layer": name, "ms": round(ms, 4), "G_lookups_s": round(lookups / ms / 1e6, 1),
                      "frac_smem_roofline": round(lookups / ms / 1e6 / 9306.24, 3),
                      "GBps": round(byts / ms / 1e6, 1), "frac_hbm": round(byts / ms / 1e6 / hbm, 3)}))
    if G < C and (C // G) % 16 == 0 and (K // G) % 16 == 0:
        # the same grouped layer on weight-specialised packed tables (axq_lut_conv2d_wp, P4W)
        wp = ax.WPack(lut, w.reshape(K, -1), a_nonneg=True)
        ws = torch.zeros(ax.axq_workspace_elems(M, K), dtype=torch.int32, device="cuda")
        epw = ax.make_epilogue(sa, sw, relu=True, y_nhwc=True, q_out=q, ldq=K, d_scale_out=so, bits_out=8,
                               workspace=ws)
        for _ in range(3):
            ax.axq_lut_conv2d_wp(d, x, wp, epw)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            ax.axq_lut_conv2d_wp(d, x, wp, epw)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"layer": name + "_packed", "ms": round(ms, 4),
                          "G_lookups_s": round(lookups / ms / 1e6, 1),
                          "frac_smem_roofline": round(lookups / ms / 1e6 / 9306.24, 3),
                          "path": ax.axq_last_path()[0]}))
