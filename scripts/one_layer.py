"""Run one R18 layer (batch 32) a few times: target for ncu captures.
Usage: python scripts/one_layer.py <shape idx> [reps] [math]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
math = sys.argv[3] if len(sys.argv) > 3 else "3xbf16"
s = synth.R18_SHAPES[idx][0].with_batch(32)
d = synth.make_layer(s)
plan = tdc.ConvPlan(s, d, math=tdc.MATH_NAMES[math])
print(plan.info().variant_name)
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
for _ in range(reps):
    plan.forward(x, y)
torch.cuda.synchronize()
