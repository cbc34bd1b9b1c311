"""Debug: per-tile events of CTA 0 for the three launches of a 3-launch forward."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
math = sys.argv[2] if len(sys.argv) > 2 else "3xtf32"
os.environ["TDC_DISABLE_FUSED"] = "1"
shape = synth.R18_SHAPES[idx][0].with_batch(32)
d = synth.make_layer(shape)
plan = tdc.ConvPlan(shape, d, math=tdc.MATH_NAMES[math])
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((shape.B, shape.Ho, shape.Wo, shape.N), device="cuda")
for _ in range(4):  # gemm launches: 2 per forward -> seq 0..7; keep the last forward
    plan.forward(x, y)
torch.cuda.synchronize()
n = 4 * 64 * 8
buf = (ctypes.c_ulonglong * n)()
tdc.lib.tdc_debug_tile_timeline(buf, n)
a = np.array(buf, dtype=np.int64).reshape(4, 64, 8)
for seq in (2, 3):  # stage-1 and stage-3 GEMMs of the 2nd forward (seq % 4)
    t = a[seq]
    rows = t[t[:, 1] > 0]
    t0 = rows[:, 0].min() if (rows[:, 0] > 0).any() else rows[:, 1].min()
    print(f"--- gemm launch seq {seq}: tiles {len(rows)}")
    print("tile prod_start mma_free mma_iss epi_acc epi_done conv_land ld0 st0 (us, rel)")
    for i, r in enumerate(rows[:8]):
        print(i, " ".join(f"{(v - t0) / 1000:8.2f}" if v else "     -  " for v in r[:8]))
