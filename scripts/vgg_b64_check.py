"""Debug: one Tucker VGG-16 forward at a given batch with CUDA_LAUNCH_BLOCKING (locate a failing op)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth.models as sm
from paper_2211_03715_b200 import tdc
b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
arch = sys.argv[2] if len(sys.argv) > 2 else "vgg"
ops = sm.tucker_vgg16() if arch == "vgg" else sm.tucker_resnet(50)
m = tdc.Model(ops, b)
h, w, c = m.output_shape()
x = torch.from_numpy(sm.model_input(b)).cuda()
o = torch.empty((b, h, w, c), device="cuda")
m.forward(x, o)
torch.cuda.synchronize()
print("ok", b, arch)
