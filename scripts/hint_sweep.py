"""Debug: µs per forward of one R18 layer (batch 32, 3xBF16) under planner hint sets.
Usage: python scripts/hint_sweep.py <shape idx> 'k=v,k=v' ['k=v' ...]   ('' = planner)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402

s = synth.R18_SHAPES[int(sys.argv[1])][0].with_batch(32)
d = synth.make_layer(s)
xs = [torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda() for _ in range(4)]
ys = [torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda") for _ in range(4)]
for spec in sys.argv[2:] or [""]:
    hints = {k: int(v) for k, v in (kv.split("=") for kv in spec.split(",") if kv)}
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16, hints=hints or None)
    st = torch.cuda.current_stream()
    for k in range(20):
        plan.forward(xs[k % 4], ys[k % 4])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    e0.record(st)
    for k in range(n):
        plan.forward(xs[k % 4], ys[k % 4])
    e1.record(st)
    torch.cuda.synchronize()
    i = plan.info()
    print(f"{s.name:18s} {spec or 'planner':60s} {e0.elapsed_time(e1) * 1e3 / n:8.2f} us  "
          f"bn {i.bn_stage1}/{i.bn_core}/{i.bn_stage3} gs {i.gsplit_stage1}/{i.gsplit_core}/{i.gsplit_stage3}")
    plan.close()
