"""The c3 forward (batch 256, calibrated, one warm-up pass) with the CUDA profiler range
around one more forward only -- for ncu --profile-from-start off -k regex:lut_p4w
--launch-skip i --launch-count 1 captures of single layers on real activations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2203_04071_b200 import Lut  # noqa: E402
from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
x_all = datagen.config3_images(max(batch, 8))
net = ApproxResNet(datagen.network_weights(layer_specs(), 3), Lut(8, datagen.lut_randerr(8, 0, 2)))
net.calibrate(torch.from_numpy(x_all[:8]).cuda())
x = torch.from_numpy(x_all[:batch]).cuda()
net.forward(x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
net.forward(x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
