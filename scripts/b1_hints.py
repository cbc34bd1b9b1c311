"""Debug: batch-1 µs (CUDA-graph replay of 20 forwards) of the R18 layers / config 1 under
planner hint sets and math modes.  Usage: python scripts/b1_hints.py <idx|c1> 'math:k=v,k=v' ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402

B = int(os.environ.get("LAYER_B", "1"))
s = synth.CONFIG1.with_batch(B) if sys.argv[1] == "c1" else synth.R18_SHAPES[int(sys.argv[1])][0].with_batch(B)
d = synth.make_layer(s)
xs = [torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda() for _ in range(4)]
ys = [torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda") for _ in range(4)]
for spec in sys.argv[2:] or ["3xbf16:"]:
    math, _, kv = spec.partition(":")
    hints = {k: int(v) for k, v in (p.split("=") for p in kv.split(",") if p)}
    try:
        plan = tdc.ConvPlan(s, d, math=tdc.MATH_NAMES[math], hints=hints or None)
    except Exception as e:  # noqa: BLE001
        print(f"{s.name} B={B} {spec:40s} plan failed: {e}")
        continue
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        for k in range(5):
            plan.forward(xs[k % 4], ys[k % 4], stream=gs)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for k in range(20):
            plan.forward(xs[k % 4], ys[k % 4], stream=gs)
    with torch.cuda.stream(gs):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(gs)
    with torch.cuda.stream(gs):
        for _ in range(10):
            g.replay()
    e1.record(gs)
    torch.cuda.synchronize()
    print(f"{s.name} B={B} {spec:40s} {plan.info().variant_name:22s} {e0.elapsed_time(e1) * 1e3 / 200:8.2f} us",
          flush=True)
    del g
    plan.close()
