"""Debug: SM clock (NVML, every ~5 ms) while one R18 layer (3xBF16, batch 32) runs back to back
for ~3 s.  Usage: python scripts/clock_probe.py [shape idx]"""
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402

i = int(sys.argv[1]) if len(sys.argv) > 1 else 0
s = synth.R18_SHAPES[i][0].with_batch(32)
d = synth.make_layer(s)
plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
xs = [torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda() for _ in range(4)]
ys = [torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda") for _ in range(4)]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.005)


th = threading.Thread(target=sampler)
th.start()
t0 = time.time()
n = 0
while time.time() - t0 < 3.0:
    for k in range(200):
        plan.forward(xs[k % 4], ys[k % 4])
    torch.cuda.synchronize()
    n += 200
stop.set()
th.join()
el = time.time() - t0
mhz = sorted(x[0] for x in samples[len(samples) // 4:])
pw = sorted(x[1] for x in samples[len(samples) // 4:])
reasons = sorted({x[2] for x in samples})
print(f"{s.name}: {el / n * 1e6:.2f} us/forward over {n} forwards; SM MHz min/median/max "
      f"{mhz[0]}/{mhz[len(mhz) // 2]}/{mhz[-1]}; power median {pw[len(pw) // 2]:.0f} W; "
      f"throttle reason masks {[hex(r) for r in reasons]}; {len(samples)} samples")
