"""One depthwise 3x3 layer (BJ-style MobileNet shape 128 x 256 x 56 x 56, stride 1, pad 1, fused
ReLU + requantize), for ncu captures of the depthwise kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

N, C, H = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 256, 56)))
lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.integers(0, 100, (N, H, H, C)).astype(np.int8)).cuda()
w = torch.from_numpy(rng.integers(-60, 60, (C, 3, 3, 1)).astype(np.int8)).cuda()
d = ax.conv_desc(N, H, H, C, C, 3, 3, (1, 1), (1, 1), groups=C)
q = torch.empty(N * H * H, C, dtype=torch.int8, device="cuda")
sa, sw, so = (torch.tensor([v], device="cuda") for v in (0.01, 0.01, 0.05))
ep = ax.make_epilogue(sa, sw, relu=True, y_nhwc=True, q_out=q, ldq=C, d_scale_out=so, bits_out=8)
for _ in range(2):
    ax.axq_lut_conv2d_ep(d, x, w, lut, ep)
torch.cuda.synchronize()
print("ok")
