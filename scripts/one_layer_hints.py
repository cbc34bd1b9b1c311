"""Run one R18 layer (batch 32) with plan hints a few times: ncu target.
Usage: python scripts/one_layer_hints.py <shape idx> <reps> key=val ..."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx, reps = int(sys.argv[1]), int(sys.argv[2])
hints = {k: int(v) for k, v in (a.split("=") for a in sys.argv[3:])} or None
s = synth.R18_SHAPES[idx][0].with_batch(32)
d = synth.make_layer(s)
plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16, hints=hints)
i = plan.info()
print(i.variant_name, i.gsplit_stage1, i.gsplit_core, i.gsplit_stage3, i.bn_stage1, i.bn_core, i.bn_stage3)
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
for _ in range(reps):
    plan.forward(x, y)
torch.cuda.synchronize()
