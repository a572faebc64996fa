"""Time v1 vs P4 LUT kernels on BJ configs[2] (conv) and a few ResNet shapes (CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen
from paper_2203_04071_b200 import _lib as ax
ax.load()
lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
rng = np.random.default_rng(0)

def bench(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps

shapes = [("c2", 128, 56, 56, 64, 64, 3, 1, 1), ("s0.c1", 256, 56, 56, 256, 64, 1, 1, 0),
          ("s0.c3", 256, 56, 56, 64, 256, 1, 1, 0), ("s1.c2", 256, 28, 28, 128, 128, 3, 1, 1),
          ("s3.c2", 256, 7, 7, 512, 512, 3, 1, 1), ("s2.c1", 256, 14, 14, 1024, 256, 1, 1, 0)]
for name, N, H, W, C, K, R, st, pd in shapes:
    x = torch.from_numpy(np.maximum(rng.standard_normal((N, H, W, C), dtype=np.float32), 0) * 20).to(torch.int8).cuda()
    w = torch.from_numpy(rng.integers(-60, 60, (K, R, R, C)).astype(np.int8)).cuda()
    d = ax.conv_desc(N, H, W, C, K, R, R, (st, st), (pd, pd))
    Ho, Wo = ax.axq_conv2d_out_hw(d)
    sa = torch.tensor([0.01], device="cuda"); sw = torch.tensor([0.01], device="cuda")
    y = torch.empty(N, Ho, Wo, K, device="cuda")
    q = torch.empty(N, Ho, Wo, K, dtype=torch.int8, device="cuda")
    so = torch.tensor([0.05], device="cuda")
    ep = ax.make_epilogue(sa, sw, y=y, ldy=K, y_nhwc=True, relu=True, q_out=q, ldq=K, d_scale_out=so, bits_out=8)
    wp = ax.WPack(lut, w.reshape(K, -1), a_nonneg=True)
    t1 = bench(lambda: ax.axq_lut_conv2d_ep(d, x, w, lut, ep))
    y1 = y.clone()
    t2 = bench(lambda: ax.axq_lut_conv2d_wp(d, x, wp, ep))
    same = torch.equal(y1, y)
    lk = N * Ho * Wo * K * C * R * R
    print("%-6s v1 %8.3f ms (%5.0f Glk/s)  P4 %8.3f ms (%5.0f Glk/s) speedup %.2f same=%s" % (
        name, t1, lk / t1 / 1e6, t2, lk / t2 / 1e6, t1 / t2, same))
