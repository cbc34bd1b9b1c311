"""Exhaustive planner-hint sweep of the R18 layers at a given batch (default 1): µs per
forward (back-to-back forwards between CUDA events, inputs L2-resident) for every point
of the split-K / N-tile / fusion hint grid.  Output: JSON lines, best point per layer.
Usage: python scripts/b1_sweep.py [batch] [shape idx ...]"""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
idx = [int(a) for a in sys.argv[2:]] or list(range(len(synth.R18_SHAPES)))
GRID = dict(core3=[-1, 0], bn_core=[0, 32, 64], gsplit_core=[1, 2, 4, 8], gsplit_stage1=[1, 2, 4],
            gsplit_stage3=[1, 2, 4])


def measure(plan, x, y, n=50):
    st = torch.cuda.current_stream()
    for _ in range(5):
        plan.forward(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        plan.forward(x, y)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


for i in idx:
    s = synth.R18_SHAPES[i][0].with_batch(B)
    d = synth.make_layer(s)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
    base = measure(plan, x, y)
    plan.close()
    rows = []
    keys = list(GRID)
    for vals in itertools.product(*GRID.values()):
        h = dict(zip(keys, vals))
        try:
            plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16, hints=h)
        except tdc.TdcError:
            continue
        inf = plan.info()
        t = measure(plan, x, y)
        rows.append((t, h, inf.variant_name, (inf.bn_stage1, inf.bn_core, inf.bn_stage3),
                     (inf.gsplit_stage1, inf.gsplit_core, inf.gsplit_stage3)))
        plan.close()
    rows.sort(key=lambda r: r[0])
    print(json.dumps({"layer": s.name, "batch": B, "planner_us": round(base, 2), "points": len(rows),
                      "best": [{"us": round(r[0], 2), "hints": r[1], "variant": r[2], "bn": r[3], "gs": r[4]}
                               for r in rows[:5]]}), flush=True)
