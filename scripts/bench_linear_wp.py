"""BJ configs[1] (approximate linear 256 x 1024 x 1024): per-row gather (axq_lut_gemm_dq) vs
weight-specialised packed tables streamed from HBM (axq_lut_gemm_wp), L2 flushed before every
timed launch.  Prints one JSON line per path; checks the two outputs are bit-identical."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2203_04071_b200 import Lut  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402
from paper_2203_04071_b200.layers import ApproxLinear  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    c = datagen.config1()
    lut = Lut(8, c.lut)
    Ms = [int(v) for v in (sys.argv[1:] or ["256"])]
    W = torch.from_numpy(c.W).to(dev)
    bias = torch.from_numpy(c.b).to(dev)
    if os.environ.get("KN"):   # other layer shapes: KN=K,N (random weights, zero bias)
        K, N = (int(v) for v in os.environ["KN"].split(","))
        W = torch.randn(N, K, generator=torch.Generator().manual_seed(1)).mul_(0.02).to(dev)
        bias = torch.zeros(N, device=dev)
    L = ApproxLinear(W, bias, lut)
    wp = ax.WPack(lut, L.qw)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
    for M in Ms:
        x = torch.randn(M, L.K, generator=torch.Generator().manual_seed(M)).to(dev)
        qa = torch.empty(M, L.K, dtype=torch.int8, device=dev)
        ax.axq_amax(x, L.d_amax_a)
        ax.axq_scale(L.d_amax_a, 8, L.d_scale_a)
        ax.axq_quantize(x, L.d_scale_a, 8, qa)
        ws = torch.zeros(M, L.N, dtype=torch.int32, device=dev)
        y0 = torch.empty(M, L.N, device=dev)
        y1 = torch.empty(M, L.N, device=dev)

        def run_dq():
            ax.axq_lut_gemm_dq(qa, L.qw, lut, L.d_scale_a, L.d_scale_w, L.bias, y0, workspace=ws)

        ep = ax.make_epilogue(L.d_scale_a, L.d_scale_w, bias=L.bias, y=y1, ldy=L.N, workspace=ws)

        def run_wp():
            ax.axq_lut_gemm_wp(qa, wp, ep)

        xp = ax.WPack(lut, qa, activations=True)
        y2 = torch.empty(M, L.N, device=dev)
        ep2 = ax.make_epilogue(L.d_scale_a, L.d_scale_w, bias=L.bias, y=y2, ldy=L.N, workspace=ws)

        def run_xs():
            ax.axq_wpack_repack(xp, qa)
            ax.axq_lut_gemm_xs(L.qw, xp, ep2)

        out = {}
        paths = (("gather", run_dq), ("packed", run_wp), ("xspec", run_xs))
        only = os.environ.get("ONLY")
        for name, fn in paths:
            if only and name != only:
                continue
            for _ in range(3):
                fn()
            ts = []
            for _ in range(20):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            ms = ts[len(ts) // 2]
            out[name] = {"ms": round(ms, 4), "Glookup_s": round(M * L.N * L.K / ms / 1e6, 1)}
        torch.cuda.synchronize()
        if not only:
            out["bit_identical"] = bool(torch.equal(y0, y1)) and bool(torch.equal(y0, y2))
        out["M"] = M
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
