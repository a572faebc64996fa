"""Per-GPU ResNet-50 (c3) forward time at the per-rank batch of N = 1, 2, 4, 8 GPUs (256/N
images) on one GPU: predicts strong-scaling efficiency before the collective."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2203_04071_b200 import Lut
from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs
x_all = datagen.config3_images(256)
net = ApproxResNet(datagen.network_weights(layer_specs(), 3), Lut(8, datagen.lut_randerr(8, 0, 2)))
net.calibrate(torch.from_numpy(x_all[:8]).cuda())
base = None
for n in (1, 2, 4, 8):
    b = 256 // n
    x = torch.from_numpy(x_all[:b]).cuda()
    for _ in range(2):
        net.forward(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        net.forward(x)
    e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 5
    if base is None:
        base = t
    print("N=%d batch %3d: %8.2f ms/forward  %7.1f img/s/GPU  predicted E(N)=%.3f" % (n, b, t, b / t * 1e3, base / (n * t)))
# the same per-rank batches replayed as CUDA graphs (no launch gaps between the 55 LUT kernels)
base = None
for n in (1, 2, 4, 8):
    b = 256 // n
    x = torch.from_numpy(x_all[:b]).cuda()
    ref = net.forward(x).clone()
    replay = net.capture(x)
    out = replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    for _ in range(2):
        replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        replay()
    e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 5
    if base is None:
        base = t
    print("graph N=%d batch %3d: %8.2f ms/forward  %7.1f img/s/GPU  predicted E(N)=%.3f" % (n, b, t, b / t * 1e3, base / (n * t)))
# do CUDA events recorded inside a captured graph time the replay?
x = torch.from_numpy(x_all[:32]).cuda()
side = torch.cuda.Stream()
ev = [torch.cuda.Event(True), torch.cuda.Event(True)]
g = torch.cuda.CUDAGraph()
net.forward(x)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    ev[0].record()
    net.run(x, False, torch.cuda.current_stream())
    ev[1].record()
g.replay()
torch.cuda.synchronize()
try:
    print("event inside graph: %.3f ms" % ev[0].elapsed_time(ev[1]))
except Exception as e:
    print("event inside graph: unavailable (%s)" % e)
