"""One calibrated LSTM (c4, b=8) forward, for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2203_04071_b200 import Lut
from paper_2203_04071_b200.lstm import ApproxLSTM
c = datagen.config4()
net = ApproxLSTM(c.W_ih, c.W_hh, c.b_ih, c.b_hh, Lut(8, c.luts[8]), "cuda")
x = torch.from_numpy(c.x).cuda()
net.calibrate(x)
torch.cuda.synchronize()
net.forward(x)
torch.cuda.synchronize()
print("ok")
