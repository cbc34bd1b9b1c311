"""Debug: per-tile events of CTA 0 of the 3xBF16 GEMM launches (TDC_TIMELINE build)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
shape = synth.R18_SHAPES[idx][0].with_batch(int(os.environ.get("LAYER_B", "32")))
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
    if not (t[:, 1] > 0).any():
        continue
    rows = t[t[:, 1] > 0]
    t0 = rows[rows > 0].min()
    print(f"--- launch seq {seq} ({'stage 1' if seq % 2 == 0 else 'stage 3'}): tiles {len(rows)}")
    print("tile prod mma_free mma_opnd mma_iss epi_acc epi_done cv_land cv_done")
    for i, r in enumerate(rows[:8]):
        print(i, " ".join(f"{(v - t0) / 1000:7.2f}" if v else "    -  " for v in r))
n2 = 64 * 12
buf2 = (ctypes.c_ulonglong * n2)()
tdc.lib.tdc_debug_bfc_timeline(buf2, n2)
c = np.array(buf2, dtype=np.int64).reshape(64, 12)
rows = c[c[:, 1] > 0]
if len(rows):
    t0 = rows[rows > 0].min()
    print(f"--- core kernel (last launch), CTA 0: tiles {len(rows)}")
    print("tile band_iss mma_free band_land S2_iss  E2_acc  E2_done S3_free S3_iss  E3_acc  E3_done")
    for i, r in enumerate(rows[:12]):
        print(i, " ".join(f"{(v - t0) / 1000:7.2f}" if v else "    -  " for v in r[:10]))
buf3 = (ctypes.c_ulonglong * 256)()
tdc.lib.tdc_debug_bfc_taps(buf3, 256)
tp = np.array(buf3, dtype=np.int64).reshape(128, 2)
tp = tp[tp[:, 0] > 0]
if len(tp):
    t0 = tp.min()
    print("--- core kernel CTA 0 tile 0 per (kc, tap): producer-issue  mma-ready (us)")
    for i, r in enumerate(tp[:80]):
        print(i, " ".join(f"{(v - t0) / 1000:7.2f}" for v in r))
bufs = (ctypes.c_ulonglong * 4096)()
tdc.lib.tdc_debug_bfc_span(bufs, 4096)
sp = np.array(bufs, dtype=np.int64).reshape(1024, 4)[:, :3]
sp = sp[sp[:, 0] > 0]
if len(sp):
    t0 = sp[:, 0].min()
    st, pro, en = (sp[:, 0] - t0) / 1e3, (sp[:, 1] - t0) / 1e3, (sp[:, 2] - t0) / 1e3
    print(f"--- core kernel per-CTA spans ({len(sp)} CTAs, us from first start): start max {st.max():.2f}, "
          f"prologue-done min/med/max {pro.min():.2f}/{np.median(pro):.2f}/{pro.max():.2f}, "
          f"end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f}")
    print("   end percentiles 10/50/90/99:", np.percentile(en, [10, 50, 90, 99]).round(2))
bufg = (ctypes.c_ulonglong * (4 * 1024 * 4))()
tdc.lib.tdc_debug_bfg_span(bufg, 4 * 1024 * 4)
gs = np.array(bufg, dtype=np.int64).reshape(4, 1024, 4)[:, :, :3]
for seq in range(4):
    sp = gs[seq]
    sp = sp[sp[:, 0] > 0]
    if not len(sp):
        continue
    t0 = sp[:, 0].min()
    st, pro, en = (sp[:, 0] - t0) / 1e3, (sp[:, 1] - t0) / 1e3, (sp[:, 2] - t0) / 1e3
    print(f"--- gemm launch seq {seq} per-CTA spans ({len(sp)} CTAs): start max {st.max():.2f}, "
          f"prologue-done min/med/max {pro.min():.2f}/{np.median(pro):.2f}/{pro.max():.2f}, "
          f"end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f}")
