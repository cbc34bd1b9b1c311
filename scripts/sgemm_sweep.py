"""Tile / split-K sweep of the fp32 CUDA-core path (variant 6), one stage at a time with
the other two on the planner's choice, at the bench's batch (32).  Tuning tool, not product.
Usage: python scripts/sgemm_sweep.py [out.json]"""
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


out = {}
for sh, _ in synth.R18_SHAPES:
    s = sh.with_batch(32)
    d = synth.make_layer(s)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    os.environ.pop("TDC_SG_TILES", None); os.environ.pop("TDC_SG_KSPLIT", None)
    base = time_us(tdc.ConvPlan(s, d, math=tdc.TDC_MATH_FP32), x, y)
    rows = {"auto": base}
    for stage in range(3):
        for t in range(3):
            for ks in ["x", "1", "2", "4", "8"]:
                tl = ["x", "x", "x"]; kl = ["x", "x", "x"]
                tl[stage] = str(t); kl[stage] = ks
                os.environ["TDC_SG_TILES"] = ",".join(tl); os.environ["TDC_SG_KSPLIT"] = ",".join(kl)
                try:
                    rows[f"s{stage + 1}_t{t}_k{ks}"] = time_us(tdc.ConvPlan(s, d, math=tdc.TDC_MATH_FP32), x, y)
                except Exception as e:  # noqa: BLE001
                    rows[f"s{stage + 1}_t{t}_k{ks}"] = str(e)[:80]
    out[s.name] = rows
    best = {st: min(((v, k) for k, v in rows.items() if k.startswith(st) and isinstance(v, float)), default=None)
            for st in ("s1", "s2", "s3")}
    print(s.name, f"auto {base:.1f}", {k: (round(v[0], 1), v[1]) for k, v in best.items() if v}, flush=True)
os.environ.pop("TDC_SG_TILES", None); os.environ.pop("TDC_SG_KSPLIT", None)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
