"""NEXT-2 measurement: the bitwidth experiment of P:322 on the GPU -- one LUT-GEMM
(M = 8192, N = 256, K = 256, randerr tables) at b = 8 (int8 codes, resident-table v1 kernel and
the packed-table P4W kernel) and b = 10, 12 (int16 codes: L2-resident wide tables gathered per
lookup, and the table tiled by the weights -- axq_lut_gemm16_wp)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

M, N, K = 8192, 256, 256


def timeit(f, reps=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
A8 = torch.from_numpy(datagen.random_int8(1, (M, K))).cuda()
W8 = torch.from_numpy(datagen.random_int8(2, (N, K))).cuda()
C = torch.empty(M, N, dtype=torch.int32, device="cuda")
lut8 = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
out["b8_v1"] = timeit(lambda: ax.axq_lut_gemm(A8, W8, lut8, C))
wp = ax.WPack(lut8, W8)
out["b8_p4w"] = timeit(lambda: ax.axq_lut_gemm_wp(A8, wp, None, C))
for bits in (10, 12):
    A = torch.from_numpy(datagen.random_int16(3, (M, K), bits)).cuda()
    W = torch.from_numpy(datagen.random_int16(4, (N, K), bits)).cuda()
    lut = ax.Lut(bits, datagen.lut_randerr(bits, 9, bits))
    out["b%d_wide" % bits] = timeit(lambda: ax.axq_lut_gemm16(A, W, lut, None, C))
    wpb = ax.WPack16(lut, W)                       # the table tiled by the weights (packed)
    out["b%d_packed" % bits] = timeit(lambda: ax.axq_lut_gemm16_wp(A, wpb, None, C))
    del wpb
res = {k: {"ms": round(v, 4), "G_lookups_s": round(M * N * K / v / 1e6, 1)} for k, v in out.items()}
res["ratio_b10_b8v1"] = round(out["b10_wide"] / out["b8_v1"], 2)
res["ratio_b12_b10"] = round(out["b12_wide"] / out["b10_wide"], 2)
res["packed_ratio_b10_b8p4w"] = round(out["b10_packed"] / out["b8_p4w"], 2)
res["packed_ratio_b12_b10"] = round(out["b12_packed"] / out["b10_packed"], 2)
res["paper"] = "~2.1x per +2 bits on a Xeon with AVX2 (P:322)"
print(json.dumps(res))
