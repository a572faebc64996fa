"""One weight-tiled packed wide LUT-GEMM (axq_lut_gemm16_wp, NEXT-2) at the bench_wide shape, for
ncu captures: argv[1] = bits (10 or 12)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 12
M, N, K = 8192, 256, 256
A = torch.from_numpy(datagen.random_int16(3, (M, K), bits)).cuda()
W = torch.from_numpy(datagen.random_int16(4, (N, K), bits)).cuda()
C = torch.empty(M, N, dtype=torch.int32, device="cuda")
lut = ax.Lut(bits, datagen.lut_randerr(bits, 9, bits))
wpb = ax.WPack16(lut, W)
for _ in range(3):
    ax.axq_lut_gemm16_wp(A, wpb, None, C)
torch.cuda.synchronize()
print("ok")
