"""Per-stage hint sweep of the three-launch 3xBF16 path on the R18 shapes the fused layer
kernel does not take (batch 32): each stage's N tile x split-K choice with the other
stages on the planner's choice.  Tuning tool, not product.
Usage: python scripts/bf16_stage_sweep.py [out.json]"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2211_03715_b200 import tdc


def time_us(plan, x, y, iters=30):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            plan.forward(x, y, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(iters):
            plan.forward(x, y, stream=st)
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


INFO = ("variant_name", "bn_stage1", "bn_core", "bn_stage3", "ksplit_stage1", "ksplit_core", "ksplit_stage3",
        "gsplit_stage1", "gsplit_core", "gsplit_stage3", "core3", "launches_per_forward")
out = {}
only = os.environ.get("ONLY")
for sh, _ in synth.R18_SHAPES:
    if only and only not in sh.name:
        continue
    s = sh.with_batch(32)
    d = synth.make_layer(s)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    M = tdc.TDC_MATH_3XBF16
    p = tdc.ConvPlan(s, d, math=M)
    i = p.info()
    rows = {"auto": [time_us(p, x, y), {k: (getattr(i, k))
                                         for k in INFO}]}
    del p
    for stage in ("stage1", "core", "stage3"):
        for bn in (0, 64, 128, 256):
            for mode, ks in [("k", 1), ("k", 2), ("k", 4), ("g", 2), ("g", 4), ("g", 8)]:
                h = {"fused_layer": 0, f"bn_{stage}": bn}
                h["ksplit_" + stage] = ks if mode == "k" else 1
                h["gsplit_" + stage] = ks if mode == "g" else 1
                for c3 in ((0, 1) if stage != "stage1" else (-1,)):
                    h["core3"] = c3
                    key = f"{stage}_bn{bn}_{mode}{ks}_c{c3}"
                    try:
                        p = tdc.ConvPlan(s, d, math=M, hints=h)
                        i = p.info()
                        rows[key] = [time_us(p, x, y), {k: getattr(i, k) for k in INFO}]
                        del p
                    except Exception as e:  # noqa: BLE001
                        rows[key] = [None, str(e)[:80]]
    out[s.name] = rows
    ok = [(v[0], k) for k, v in rows.items() if v[0] is not None]
    best = min(ok)
    print(s.name, f"auto {rows['auto'][0]:.1f}", f"best {best[0]:.1f} {best[1]}", rows[best[1]][1], flush=True)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
