"""c2-shaped P4 (or v1 with argv[1] == 'v1') launches for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen
from paper_2203_04071_b200 import _lib as ax
ax.load()
which = sys.argv[1] if len(sys.argv) > 1 else "p4"
lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
rng = np.random.default_rng(0)
N, H, W, C, K = 128, 56, 56, 64, 64
x = torch.from_numpy(np.maximum(rng.standard_normal((N, H, W, C), dtype=np.float32), 0) * 20).to(torch.int8).cuda()
w = torch.from_numpy(rng.integers(-60, 60, (K, 3, 3, C)).astype(np.int8)).cuda()
d = ax.conv_desc(N, H, W, C, K, 3, 3, (1, 1), (1, 1))
sa = torch.tensor([0.01], device="cuda"); sw = torch.tensor([0.01], device="cuda")
y = torch.empty(N, K, H, W, device="cuda")
ep = ax.make_epilogue(sa, sw, y=y)
wp = ax.WPack(lut, w.reshape(K, -1), a_nonneg=True)
for _ in range(2):
    if which == "p4":
        ax.axq_lut_conv2d_wp(d, x, wp, ep)
    else:
        ax.axq_lut_conv2d_ep(d, x, w, lut, ep)
torch.cuda.synchronize()
print("ok", which)
