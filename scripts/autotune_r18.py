"""Measured autotune of the 3xBF16 planner on the ResNet-18 layers (NEXT-3):
python scripts/autotune_r18.py [--out profiles] -> r01_autotune_r18_b32.json"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2211_03715_b200 import autotune, tdc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    rows = []
    for s, count in synth.R18_SHAPES:
        shape = s.with_batch(32)
        r = autotune.coordinate_descent(lambda h: autotune.measure_hints_us(shape, h, a.iters))
        d = synth.make_layer(shape)
        plan = tdc.ConvPlan(shape, d, math=tdc.TDC_MATH_3XBF16, hints=dict(r.best_hints))
        info = plan.info()
        plan.close()
        chosen = {k: getattr(info, k) for k in ("core3", "bn_stage1", "bn_core", "bn_stage3", "ksplit_stage1",
                                                "ksplit_core", "ksplit_stage3")}
        rows.append({"layer": shape.name, "count": count, "planner_us": round(r.planner_us, 3),
                     "tuned_us": round(r.best_us, 3), "gap": round(r.gap, 4), "hints": r.best_hints,
                     "tuned_plan": chosen, "points_measured": r.measured})
        print(json.dumps(rows[-1]), flush=True)
    tot_p = sum(x["planner_us"] * x["count"] for x in rows)
    tot_t = sum(x["tuned_us"] * x["count"] for x in rows)
    out = {"math": "3xbf16", "batch": 32, "search": "coordinate descent, 2 passes, from the planner default",
           "layers": rows, "step_planner_us": round(tot_p, 2), "step_tuned_us": round(tot_t, 2),
           "step_gap": round(tot_p / tot_t - 1, 4)}
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "r01_autotune_r18_b32.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("step_planner_us", "step_tuned_us", "step_gap")}))


if __name__ == "__main__":
    main()
