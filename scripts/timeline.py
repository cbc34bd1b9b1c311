"""Debug: per-tile event timeline of the fused kernel (CTA 0), from the
TDC_TIMELINE build (libtdc_tl.so).  Usage: TDC_LIB=.../libtdc_tl.so python scripts/timeline.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402

EV = ["Xfree", "Wstart", "MMAtile", "Xland", "Wland", "S1iss", "X'rdy", "S2iss", "a3free", "S3iss",
      "e1acc1", "e1done", "e3acc3", "e3done"] + [f"t{i}" for i in range(9)]
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
shape = synth.R18_SHAPES[idx][0].with_batch(32)
d = synth.make_layer(shape)
plan = tdc.ConvPlan(shape, d, math=tdc.TDC_MATH_TF32)
print(plan.info())
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((shape.B, shape.Ho, shape.Wo, shape.N), device="cuda")
for _ in range(3):
    plan.forward(x, y)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 32))()
tdc.lib.tdc_debug_timeline(buf, 64 * 32)
a = np.array(buf, dtype=np.int64).reshape(64, 32)[:, :len(EV)]
t0 = a[0, 0]
ntile = int((a[:, 2] > 0).sum())
print("ns relative to first X issue; tiles:", ntile)
print("tile " + " ".join(f"{e:>8s}" for e in EV))
for i in range(ntile):
    print(f"{i:4d} " + " ".join(f"{(v - t0) if v else -1:8d}" for v in a[i]))
