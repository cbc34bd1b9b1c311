"""NEXT-3: exhaustive measured search of the 3xBF16 planner's hint space on
the 7 ResNet-18 layer shapes (batch 32) -- the paper's "oracle" -- against (a) the
library's rule planner and (b) the paper's two-stage analytical selection re-fitted to
B200 (paper_2211_03715_b200/tiling_model.py, Part B; kappa and L0 fitted leave-one-
layer-out, so each layer's analytic pick uses constants fitted on the other six).
Writes profiles/<prefix>_tiling_search_r18_b32.json.  Device time per forward from CUDA
graph replay."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2211_03715_b200 import roofline, tdc  # noqa: E402
from paper_2211_03715_b200 import tiling_model as tm  # noqa: E402

PREFIX = sys.argv[1] if len(sys.argv) > 1 else "r02"
B = 32


def measure(s, d, hints, iters=20):
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16, hints=hints)
    info = plan.info()
    xs = [torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda() for _ in range(2)]
    ys = [torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda") for _ in range(2)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k in range(3):
            plan.forward(xs[k % 2], ys[k % 2], stream=st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for k in range(iters):
            plan.forward(xs[k % 2], ys[k % 2], stream=st)
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    del g
    plan.close()
    return us, info.variant_name


t0 = time.time()
points = tm.hint_points()
layers, samples, rows = [], [], []
for shape, count in synth.R18_SHAPES:
    s = shape.with_batch(B)
    d = synth.make_layer(s)
    L = tm.LayerGeom(B, s.C, s.N, s.H, s.W, s.D1, s.D2, s.K, s.stride, s.pad)
    planner_us, planner_var = measure(s, d, None)
    table = []
    for h in points:
        us, var = measure(s, d, h)
        table.append((h, us, var))
        samples.append((s.name, L, h, us * 1e-6))
    best = min(table, key=lambda r: r[1])
    rows.append({"layer": s.name, "count": count, "planner_us": round(planner_us, 3), "planner_variant": planner_var,
                 "best_us": round(best[1], 3), "best_hints": best[0], "best_variant": best[2],
                 "points": len(table), "table": [[r[0], round(r[1], 3), r[2]] for r in table]})
    layers.append((s.name, L, table))
    print(f"{s.name}: planner {planner_us:.2f} us ({planner_var}), best {best[1]:.2f} us {best[0]} ({best[2]})",
          flush=True)

hbm = roofline.measured_peaks()["hbm_gbs"] * 1e9
fit_all = tm.fit_refit([(L, h, t) for _, L, h, t in samples], hbm=hbm)
for r, (name, L, table) in zip(rows, layers):
    fit = tm.fit_refit([(L2, h, t) for n2, L2, h, t in samples if n2 != name], hbm=hbm)  # leave this layer out
    pick = tm.select_hints_analytical(L, fit, [p for p, _, _ in table])
    us = next(u for p, u, _ in table if p == pick)
    r.update({"analytic_hints": pick, "analytic_us": round(us, 3), "fit_loo": {"kappa": fit.kappa, "l0_us": fit.l0 * 1e6},
              "gap_analytic": round(us / r["best_us"] - 1, 4), "gap_planner": round(r["planner_us"] / r["best_us"] - 1, 4),
              "predicted_best_us": round(fit.predict(tm.kernels_of(L, r["best_hints"])) * 1e6, 3)})
    print(f"{name}: analytic {us:.2f} us ({pick}) gap {r['gap_analytic']:+.1%}; planner gap {r['gap_planner']:+.1%}",
          flush=True)
tot = lambda k: sum(r[k] * r["count"] for r in rows)
out = {"batch": B, "math": "3xbf16", "hint_space": tm.HINT_SPACE, "fit_all": {"kappa": fit_all.kappa,
       "l0_us": fit_all.l0 * 1e6, "hbm_gbs": hbm / 1e9},
       "step_us": {"best": round(tot("best_us"), 2), "planner": round(tot("planner_us"), 2),
                   "analytic": round(tot("analytic_us"), 2)},
       "gap_step": {"analytic": round(tot("analytic_us") / tot("best_us") - 1, 4),
                    "planner": round(tot("planner_us") / tot("best_us") - 1, 4)},
       "seconds": round(time.time() - t0, 1), "layers": rows}
path = os.path.join(ROOT, "profiles", f"{PREFIX}_tiling_search_r18_b32.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", os.path.basename(path)), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "layers"}, indent=1))
