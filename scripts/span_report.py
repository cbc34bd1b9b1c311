"""Debug: per-CTA [start, prologue-done, end] spans of the three kernels of one 3xBF16
layer forward (TDC_TIMELINE build, TDC_LIB=.../libtdc_tl.so), on one time axis.
Usage: TDC_LIB=paper_2211_03715_b200/libtdc_tl.so python scripts/span_report.py [shape idx ...]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402


def spans(fn, n):
    buf = (ctypes.c_ulonglong * n)()
    fn(buf, n)
    return np.array(buf, dtype=np.int64)


def show(name, sp, t0):
    sp = sp[sp[:, 0] > 0]
    if not len(sp):
        print(f"  {name}: no CTAs")
        return
    st, pro, en = (sp[:, 0] - t0) / 1e3, (sp[:, 1] - t0) / 1e3, (sp[:, 2] - t0) / 1e3
    print(f"  {name:8s} CTAs {len(sp):4d}  start {st.min():7.2f}..{st.max():7.2f}  "
          f"prologue {np.median(pro):7.2f} (max {pro.max():7.2f})  "
          f"end p10/50/90/max {np.percentile(en, 10):7.2f} {np.median(en):7.2f} "
          f"{np.percentile(en, 90):7.2f} {en.max():7.2f}")


idx = [int(a) for a in sys.argv[1:]] or list(range(len(synth.R18_SHAPES)))
for i in idx:
    s = synth.R18_SHAPES[i][0].with_batch(32)
    d = synth.make_layer(s)
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    for _ in range(6):
        plan.forward(x, y)
    torch.cuda.synchronize()
    info = plan.info()
    g = spans(tdc.lib.tdc_debug_bfg_span, 4 * 1024 * 4).reshape(4, 1024, 4)[:, :, :3]
    c = spans(tdc.lib.tdc_debug_bfc_span, 1024 * 4).reshape(1024, 4)[:, :3]
    # the last forward's launches: the two most recent gemm sequence slots (stage 1, stage 3)
    last = sorted(range(4), key=lambda k: g[k, :, 0].max())[-2:] if 'core3' not in plan.info().variant_name else \
        sorted(range(4), key=lambda k: g[k, :, 0].max())[-1:]
    t0 = min(g[k][g[k][:, 0] > 0][:, 0].min() for k in last)
    print(f"{s.name} ({info.variant_name}):")
    for k in last:
        gk = g[k]
        if gk[:, 0].max() < c[:, 0].max() or len(last) == 1:
            show("stage1", gk, t0)
    show("core", c, t0)
    for k in last:
        gk = g[k]
        if gk[:, 0].max() > c[:, 0].max() and len(last) == 2:
            show("stage3", gk, t0)
    plan.close()
