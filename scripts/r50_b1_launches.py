"""Debug: one Tucker ResNet-50 forward at batch 1 (target of an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth.models as sm
from paper_2211_03715_b200 import tdc
b = int(sys.argv[1]) if len(sys.argv) > 1 else 1
m = tdc.Model(sm.tucker_resnet(50), b)
h, w, c = m.output_shape()
x = torch.from_numpy(sm.model_input(b)).cuda()
o = torch.empty((b, h, w, c), device="cuda")
for _ in range(3):
    m.forward(x, o)
torch.cuda.synchronize()
