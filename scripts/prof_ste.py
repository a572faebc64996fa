"""One STE linear backward call at a given shape (for ncu captures of the STE kernels)."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2203_04071_b200 import _lib as ax  # noqa: E402

M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (2048, 4096, 1024)))
g = torch.Generator(device="cuda").manual_seed(1)
gy = torch.randn(M, N, device="cuda", generator=g)
qa = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda", generator=g)
qw = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda", generator=g)
s = torch.tensor([0.01], device="cuda")
gx, gw = torch.empty(M, K, device="cuda"), torch.empty(N, K, device="cuda")
ws = torch.empty(max(1, ax.axq_ste_linear_workspace_elems(M, N, K)), device="cuda")
for _ in range(2):
    ax.axq_ste_linear_backward(gy, qa, s, qw, s, gx=gx, gw=gw, workspace=ws)
torch.cuda.synchronize()
