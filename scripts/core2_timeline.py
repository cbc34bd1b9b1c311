"""Debug: per-chunk events of the CTA-pair core kernel (TDC_TIMELINE build; TDC_LIB=.../libtdc_tl.so)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 6
shape = synth.R18_SHAPES[idx][0].with_batch(int(os.environ.get("LAYER_B", "32")))
d = synth.make_layer(shape)
plan = tdc.ConvPlan(shape, d, math=tdc.TDC_MATH_3XBF16)
print(plan.info().variant_name)
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((shape.B, shape.Ho, shape.Wo, shape.N), device="cuda")
for _ in range(4):
    plan.forward(x, y)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 512)()
tdc.lib.tdc_debug_core2_timeline(buf, 512)
a = np.array(buf, dtype=np.int64).reshape(64, 8)[:, :5]
a = a[a[:, 1] > 0]
t0 = a[a > 0].min()
print("kc  w_issue(L)  w_seen(L)  w_peer(L)  mma_done(L)  w_issue(P)")
for i, r in enumerate(a):
    print(i, " ".join(f"{(v - t0) / 1000:9.2f}" if v else "      -  " for v in r))
