export TDC_LIB=$PWD/paper_2211_03715_b200/libtdc_tl.so
python - <<'PY'
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2211_03715_b200 import tdc
s = synth.CONFIG1
d = synth.make_layer(s)
plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
buf = (ctypes.c_ulonglong * (32 * 24))()
tdc.lib.tdc_debug_layer_timeline(buf, 32 * 24, 0)
for _ in range(3):
    plan.forward(x, y)
torch.cuda.synchronize()
tdc.lib.tdc_debug_layer_timeline(buf, 32 * 24, 0)
a = np.array(buf, dtype=np.int64).reshape(32, 24)
names = ["prodX", "convD", "S1iss", "S2iss", "S3iss", "E1acc", "E1rdy", "E2acc", "E2done", "E3acc", "E3done",
         "S2wait", "-", "S1start", "-", "-", "cv1", "cv2", "cv3", "Xland", "entry", "setup", "-", "wload"]
t0 = a[0, 21]
for i, nm in enumerate(names):
    if a[0, i]: print(f"{nm:8s} {(a[0, i] - t0) / 1000:7.2f}")
PY
