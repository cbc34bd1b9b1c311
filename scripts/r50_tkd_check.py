import sys, torch
sys.path.insert(0, '.')
import synth
from synth import LayerShape
from paper_2211_03715_b200 import tdc
for s in [LayerShape(32, 64, 64, 56, 56, 16, 16, 3, 1, 1, "r50_56_D16"), LayerShape(32, 128, 128, 28, 28, 32, 32, 3, 1, 1, "r50_28_D32"),
          LayerShape(32, 64, 64, 56, 56, 32, 32, 3, 1, 1, "r18_56_D32")]:
    d = synth.make_layer(s)
    p = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda(); y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    for _ in range(5): p.forward(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): p.forward(x, y)
    e1.record(); torch.cuda.synchronize()
    i = p.info()
    print(s.name, round(e0.elapsed_time(e1) * 1e3 / 50, 2), "us", i.variant_name, "bn", i.bn_stage1, i.bn_core, i.bn_stage3, "core3", i.core3)
    p.close()
