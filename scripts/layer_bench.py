"""Debug: mean µs per forward of single R18 layers (back-to-back forwards on one
stream, CUDA events), for quick A/B of planner/env settings.
Usage: python scripts/layer_bench.py <math> [shape idx ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402

math = sys.argv[1] if len(sys.argv) > 1 else "3xbf16"
idx = [int(a) for a in sys.argv[2:]] or list(range(len(synth.R18_SHAPES)))
for i in idx:
    s = synth.R18_SHAPES[i][0].with_batch(32)
    d = synth.make_layer(s)
    plan = tdc.ConvPlan(s, d, math=tdc.MATH_NAMES[math])
    xs = [torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda() for _ in range(4)]
    ys = [torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda") for _ in range(4)]
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
    info = plan.info()
    print(f"{s.name:20s} {e0.elapsed_time(e1) * 1e3 / n:8.2f} us  {info.variant_name}")
    plan.close()
