"""Debug: per-tile pipeline events of one CTA of the single-launch layer kernel
(TDC_TIMELINE build: python paper_2211_03715_b200/build.py --timeline, TDC_LIB=.../libtdc_tl.so)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
shape = synth.R18_SHAPES[idx][0].with_batch(int(os.environ.get("LAYER_B", "32")))
if os.environ.get("LAYER_HW"):  # e.g. LAYER_HW=8 -> the 8x8 variant of the shape
    hw = int(os.environ["LAYER_HW"])
    shape = synth.LayerShape(shape.B, shape.C, shape.N, hw, hw, shape.D1, shape.D2, shape.K, shape.stride, shape.pad)
d = synth.make_layer(shape)
plan = tdc.ConvPlan(shape, d, math=tdc.TDC_MATH_3XBF16)
print(plan.info().variant_name)
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((shape.B, shape.Ho, shape.Wo, shape.N), device="cuda")
n = 32 * 24
buf = (ctypes.c_ulonglong * n)()
tdc.lib.tdc_debug_layer_timeline(buf, n, cta)
for _ in range(3):
    plan.forward(x, y)
torch.cuda.synchronize()
tdc.lib.tdc_debug_layer_timeline(buf, n, cta)
a = np.array(buf, dtype=np.int64).reshape(32, 24)
names = ["prodX", "convD", "S1iss", "S2iss", "S3iss", "E1acc", "E1rdy", "E2acc", "E2done", "E3acc", "E3done",
         "S2wait", "E2zfree", "S1start", "S1acc1", "S1conv", "E2ld0", "E2ld1", "E2xc0", "E2xc1", "entry", "setup", "wloaded"]
rows = a[a[:, 5] > 0]
t0 = a[a > 0].min()
print("tile " + " ".join(f"{nm:>7s}" for nm in names))
for i, r in enumerate(rows[:12]):
    print(f"{i:4d} " + " ".join(f"{(v - t0) / 1000:7.2f}" if v else "    -  " for v in r[:len(names)]))
