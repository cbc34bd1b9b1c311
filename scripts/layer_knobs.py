"""Debug: µs per forward of one R18 layer (batch 32) in the single-launch layer kernel
under TDC_LAYER_DBG attribution knobs (knobs build: TDC_LIB=.../libtdc_kn.so).
Usage: python scripts/layer_knobs.py <shape idx> knob [knob ...]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1])
B = int(os.environ.get("LAYER_B", "32"))
s = synth.R18_SHAPES[idx][0].with_batch(B)
if os.environ.get("LAYER_HW"):
    hw = int(os.environ["LAYER_HW"])
    s = synth.LayerShape(B, s.C, s.N, hw, hw, s.D1, s.D2, s.K, s.stride, s.pad, f"{s.name}_{hw}x{hw}")
d = synth.make_layer(s)
xs = [torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda() for _ in range(4)]
ys = [torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda") for _ in range(4)]
for kn in sys.argv[2:]:
    os.environ["TDC_LAYER_DBG"] = kn
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
    st = torch.cuda.current_stream()
    for k in range(10):
        plan.forward(xs[k % 4], ys[k % 4])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 100
    e0.record(st)
    for k in range(n):
        plan.forward(xs[k % 4], ys[k % 4])
    e1.record(st)
    torch.cuda.synchronize()
    t_plain = e0.elapsed_time(e1) * 1e3 / n
    # CUDA-graph replay of 20 forwards: device time without host launch overhead
    gs = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for k in range(20):
            plan.forward(xs[k % 4], ys[k % 4], stream=gs)
    with torch.cuda.stream(gs):
        g.replay()
    torch.cuda.synchronize()
    e0.record(gs)
    with torch.cuda.stream(gs):
        for _ in range(5):
            g.replay()
    e1.record(gs)
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) * 1e3 / 100
    del g
    print(f"{s.name} B={B} {plan.info().variant_name} knobs={kn:>3s}: {t_plain:7.2f} us plain, {t_graph:7.2f} us graph",
          flush=True)
    plan.close()
