"""Debug: per-tile events of CTA 0 of the 3xBF16 GEMM launches (TDC_TIMELINE build)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
shape = synth.R18_SHAPES[idx][0].with_batch(32)
d = synth.make_layer(shape)
plan = tdc.ConvPlan(shape, d, math=tdc.TDC_MATH_3XBF16)
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((shape.B, shape.Ho, shape.Wo, shape.N), device="cuda")
for _ in range(4):
    plan.forward(x, y)
torch.cuda.synchronize()
n = 4 * 64 * 8
buf = (ctypes.c_ulonglong * n)()
tdc.lib.tdc_debug_bf_timeline(buf, n)
a = np.array(buf, dtype=np.int64).reshape(4, 64, 8)
for seq in (2, 3):
    t = a[seq]
    rows = t[t[:, 1] > 0]
    t0 = rows[rows > 0].min()
    print(f"--- launch seq {seq} ({'stage 1' if seq % 2 == 0 else 'stage 3'}): tiles {len(rows)}")
    print("tile prod mma_free mma_opnd mma_iss epi_acc epi_done cv_land cv_done")
    for i, r in enumerate(rows[:8]):
        print(i, " ".join(f"{(v - t0) / 1000:7.2f}" if v else "    -  " for v in r))
