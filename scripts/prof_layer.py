"""One ResNet-shaped packed-table conv layer with the ResNet epilogue, for ncu captures and
timing: python scripts/prof_layer.py N H W C K R stride [resid] [reps]
(resid = 1: fp32 residual + ReLU + fp32 y + int8 q_out, the block-output epilogue; 0: ReLU + q_out;
2: fp32 y only, the projection shortcut)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

N, H, W, C, K, R, st = (int(v) for v in sys.argv[1:8])
resid = int(sys.argv[8]) if len(sys.argv) > 8 else 1
reps = int(sys.argv[9]) if len(sys.argv) > 9 else 2
pad = R // 2
rng = np.random.default_rng(0)
lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
x = torch.from_numpy(np.minimum(np.abs(rng.standard_normal((N, H, W, C), dtype=np.float32)) * 20, 127)).to(torch.int8).cuda()
w = torch.from_numpy(rng.integers(-60, 60, (K, R, R, C)).astype(np.int8)).cuda()
d = ax.conv_desc(N, H, W, C, K, R, R, (st, st), (pad, pad))
Ho, Wo = ax.axq_conv2d_out_hw(d)
M = N * Ho * Wo
sa = torch.tensor([0.01], device="cuda"); sw = torch.tensor([0.01], device="cuda"); so = torch.tensor([0.05], device="cuda")
q = torch.empty(M, K, dtype=torch.int8, device="cuda")
ws = torch.zeros(M * K, dtype=torch.int32, device="cuda")
if resid == 2:   # projection-shortcut epilogue: fp32 y only
    y = torch.empty(M, K, device="cuda")
    ep = ax.make_epilogue(sa, sw, y=y, ldy=K, workspace=ws, y_nhwc=True)
elif resid:
    y = torch.empty(M, K, device="cuda")
    r = torch.randn(M, K, device="cuda")
    ep = ax.make_epilogue(sa, sw, y=y, ldy=K, workspace=ws, residual=r, ldr=K, relu=True, y_nhwc=True,
                          q_out=q, ldq=K, d_scale_out=so, bits_out=8)
else:
    ep = ax.make_epilogue(sa, sw, workspace=ws, relu=True, y_nhwc=True, q_out=q, ldq=K, d_scale_out=so, bits_out=8)
wp = ax.WPack(lut, w.reshape(K, -1), a_nonneg=True)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
for i in range(reps):
    if i == reps - 1:
        e0.record()
    ax.axq_lut_conv2d_wp(d, x, wp, ep)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e3
print("M=%d N=%d K=%d: %.1f us  %.0f G lookups/s" % (M, K, C * R * R, t, M * K * C * R * R / t / 1e3))
