"""One calibrated ResNet-50 (c3) forward at a given batch, for ncu launch lists / captures.
Prints the per-layer (name, M, N, K, lookups) plan so launch times can be matched to layers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import Lut  # noqa: E402
from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x_all = datagen.config3_images(max(batch, 8))
net = ApproxResNet(datagen.network_weights(layer_specs(), 3), Lut(8, datagen.lut_randerr(8, 0, 2)))
net.calibrate(torch.from_numpy(x_all[:8]).cuda())
x = torch.from_numpy(x_all[:batch]).cuda()
torch.cuda.synchronize()
for _ in range(reps):
    net.forward(x)
torch.cuda.synchronize()
print("ok batch", batch)
