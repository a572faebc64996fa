"""NEXT-1 calibration kernels on a BJ configs[2]-sized tensor (25.7 M fp32 values): amax,
2048-bin histogram, percentile (CUDA events, warm), against the HBM roofline of the two
reads (MEASURED_PEAKS.json hbm_gbs)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

x = torch.from_numpy(datagen.config2().x).cuda()
amax = torch.empty(1, device="cuda")
hist = torch.empty(ax.HIST_BINS, dtype=torch.int32, device="cuda")
s = torch.empty(1, device="cuda")


def once():
    ax.axq_amax(x, amax)
    ax.axq_calib_histogram(x, amax, hist)
    ax.axq_calib_percentile(hist, x.numel(), amax, 8, d_scale=s)


for _ in range(3):
    once()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20):
    once()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 20
try:
    hbm = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    hbm = 6650.0
gbs = 2 * x.numel() * 4 / (ms * 1e-3) / 1e9
print(json.dumps({"what": "amax + histogram + percentile calibration of a c2 input (25.7 M fp32)",
                  "ms": round(ms, 4), "algorithmic_GBps": round(gbs, 1), "hbm_peak_GBps": hbm,
                  "frac": round(gbs / hbm, 3)}))
