"""Debug: per-chunk events of CTA 0's first tile in the stage-1 / stage-3 GEMM launches of one
layer (TDC_TIMELINE build; TDC_LIB=.../libtdc_tl.so).  Usage: python scripts/gemm_chunks.py <idx>"""
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
buf = (ctypes.c_ulonglong * (4 * 64 * 4))()
tdc.lib.tdc_debug_bf_chunks(buf, 4 * 64 * 4)
a = np.array(buf, dtype=np.int64).reshape(4, 64, 4)
for seq in range(4):
    t = a[seq]
    t = t[t[:, 3] > 0]
    if not len(t):
        continue
    t0 = t[t > 0].min()
    print(f"--- launch seq {seq}: chunk  A-issue  landed  conv-done  mma-issued (us)")
    for i, r in enumerate(t):
        print(f"{i:3d} " + " ".join(f"{(v - t0) / 1000:8.2f}" if v else "      - " for v in r))
