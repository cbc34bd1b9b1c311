"""Debug: one Tucker ResNet-50 forward (batch 32) for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth.models as sm
from paper_2211_03715_b200 import tdc
arch = sys.argv[1] if len(sys.argv) > 1 else "r50"
ops = sm.tucker_resnet(50) if arch == "r50" else sm.tucker_vgg16()
b = 32 if arch == "r50" else 64
m = tdc.Model(ops, b)
h, w, c = m.output_shape()
x = torch.from_numpy(sm.model_input(b)).cuda()
o = torch.empty((b, h, w, c), device="cuda")
for _ in range(3):
    m.forward(x, o)
torch.cuda.synchronize()
