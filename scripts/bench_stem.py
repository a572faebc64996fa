"""The ResNet stem as the bench runs it: explicit-im2col rows [M][160] (K = 147 taps x 3
channels, lda 160) against 64 filters, full-range (signed image) tables, fused ReLU + int8
requantize; times axq_lut_gemm_wp (L2 flushed) for the P4W shape picked by the environment
(AXQ_P4W_CW=16 forces the 512-row shape).  python scripts/bench_stem.py [images]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    M, K, N = n * 112 * 112, 147, 64
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randint(-127, 128, (M, 160), dtype=torch.int8, device="cuda", generator=g)
    W = torch.from_numpy(datagen.random_int8(7, (N, K))).cuda()
    lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
    wp = ax.WPack(lut, W)
    one = torch.ones(1, device="cuda")
    so = torch.tensor([0.05], device="cuda")
    q = torch.empty(M, N, dtype=torch.int8, device="cuda")
    ws = torch.zeros(M * N, dtype=torch.int32, device="cuda")
    ep = ax.make_epilogue(one, one, workspace=ws, relu=True, q_out=q, ldq=N, d_scale_out=so, bits_out=8)
    flush = torch.empty(64 << 20, device="cuda")
    ts = []
    for i in range(8):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        ax.axq_lut_gemm_wp(A[:, :K], wp, ep)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print("stem M=%d N=%d K=%d: %.1f us  %.0f G lookups/s  (AXQ_P4W_CW=%s)" % (
        M, N, K, ms * 1e3, M * N * K / ms / 1e6, os.environ.get("AXQ_P4W_CW", "auto")))


if __name__ == "__main__":
    main()
