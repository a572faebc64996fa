"""Fixed per-launch cost of the P4W kernel: time axq_lut_gemm_wp (fused ReLU + int8 requantize
epilogue, half-range tables) for a few (M, N, K), averaged over back-to-back launches."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402


def run(M, N, K, reps=50):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randint(0, 128, (M, K), dtype=torch.int8, device="cuda", generator=g)
    W = torch.from_numpy(datagen.random_int8(5, (N, K))).cuda()
    lut = ax.Lut(8, datagen.lut_randerr(8, 0, 2))
    wp = ax.WPack(lut, W, a_nonneg=True)
    one = torch.ones(1, device="cuda")
    so = torch.tensor([0.05], device="cuda")
    q = torch.empty(M, N, dtype=torch.int8, device="cuda")
    ws = torch.zeros(M * N, dtype=torch.int32, device="cuda")
    ep = ax.make_epilogue(one, one, workspace=ws, relu=True, q_out=q, ldq=N, d_scale_out=so, bits_out=8)
    for _ in range(3):
        ax.axq_lut_gemm_wp(A, wp, ep)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        ax.axq_lut_gemm_wp(A, wp, ep)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print("M=%7d N=%5d K=%5d  %8.1f us/launch  %7.0f G lookups/s" % (M, N, K, us, M * N * K / us / 1e3))


if __name__ == "__main__":
    for M, N, K in [(896, 16, 32), (896 * 148, 16, 32), (896 * 148, 16, 64), (896 * 148, 16, 576),
                    (896 * 148, 16, 1152), (896 * 148 * 2, 16, 576), (896 * 148 * 3, 16, 576)]:
        run(M, N, K)
