"""Debug: per-CTA timeline of the first GEMM launch of a layer (TDC_TIMELINE build)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
math = sys.argv[2] if len(sys.argv) > 2 else "3xtf32"
shape = synth.R18_SHAPES[idx][0].with_batch(32)
d = synth.make_layer(shape)
os.environ["TDC_DISABLE_FUSED"] = "1"
plan = tdc.ConvPlan(shape, d, math=tdc.MATH_NAMES[math])
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((shape.B, shape.Ho, shape.Wo, shape.N), device="cuda")
plan.forward(x, y); torch.cuda.synchronize()
# isolate the stage-3 launch: re-run, last GEMM writes are stage 3 (same table overwritten)
plan.forward(x, y); torch.cuda.synchronize()
n = 4096 * 8
buf = (ctypes.c_ulonglong * n)()
tdc.lib.tdc_debug_gemm_timeline(buf, n)
a = np.array(buf, dtype=np.int64).reshape(4096, 8)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
rel = (a - t0) / 1000.0
print("CTAs", len(a), "span us", (a[:, 6].max() - t0) / 1000)
names = ["start", "setup", "opnd0", "mma_iss", "acc_rdy", "epi_done", "end"]
for k in range(1, 7):
    dtk = (a[:, k] - a[:, k - 1]) / 1000.0
    print(f"{names[k-1]:>8s}->{names[k]:<8s} median {np.median(dtk):7.2f} us  p90 {np.percentile(dtk,90):7.2f}")
starts = np.sort(rel[:, 0])
print("CTA start times (us) quantiles:", np.percentile(starts, [0, 25, 50, 75, 100]).round(2))
print("CTA durations (us) quantiles:", np.percentile(rel[:, 6] - rel[:, 0], [0, 25, 50, 75, 100]).round(2))
