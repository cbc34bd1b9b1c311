"""Debug: µs per forward of the single-launch layer kernel vs X staging depth."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from synth import LayerShape
from paper_2211_03715_b200 import tdc
for s in [LayerShape(32, 64, 64, 28, 28, 16, 16, 3, 1, 1, "28x28x64_D16"),
          LayerShape(32, 64, 64, 56, 56, 16, 16, 3, 1, 1, "56x56x64_D16"),
          LayerShape(32, 64, 64, 56, 56, 32, 32, 3, 1, 1, "56x56x64_D32")]:
    d = synth.make_layer(s)
    xs = [torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda() for _ in range(4)]
    ys = [torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda") for _ in range(4)]
    for xsd in ("2", "3", "4"):
        os.environ["TDC_LAYER_XS"] = xsd
        plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
        st = torch.cuda.current_stream()
        for k in range(10):
            plan.forward(xs[k % 4], ys[k % 4])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(100):
            plan.forward(xs[k % 4], ys[k % 4])
        e1.record(st)
        torch.cuda.synchronize()
        print(f"{s.name} XS<={xsd} smem={plan.info().smem_bytes_per_cta} {plan.info().variant_name}: "
              f"{e0.elapsed_time(e1) * 10:7.2f} us", flush=True)
        plan.close()
