"""Debug: device time per forward (CUDA-graph replay of 50 forwards) of a tiny TKD layer
through 1 (single-launch layer kernel), 2 (stage 1 + core3) and 3 launches: the per-launch
floor of the persistent tcgen05 kernels in a PDL chain."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from synth import LayerShape
from paper_2211_03715_b200 import tdc

for s in [LayerShape(1, 64, 64, 8, 8, 32, 32), LayerShape(1, 64, 64, 56, 56, 32, 32), LayerShape(8, 64, 64, 56, 56, 32, 32)]:
    d = synth.make_layer(s)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    for label, hints in [("1 launch", None), ("2 launches", {"fused_layer": 0}),
                         ("3 launches", {"fused_layer": 0, "core3": 0})]:
        plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16, hints=hints)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                plan.forward(x, y, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(50):
                plan.forward(x, y, stream=st)
        with torch.cuda.stream(st):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(4):
                g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        print(f"B={s.B} {s.H}x{s.W}: {label:10s} {plan.info().variant_name:20s} {e0.elapsed_time(e1) * 1e3 / 200:7.2f} us",
              flush=True)
        del g
        plan.close()
