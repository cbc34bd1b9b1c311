"""Measure the latency tables that drive hardware-aware rank selection (BASELINE config 5
and the ResNet-18 layer list) on this GPU, then select ranks under the paper's budget.

  python scripts/rank_sweep.py [--math 3xbf16] [--out profiles] [--quick]

Writes <out>/<prefix>_rank_sweep_28x28x256_b{1,32}.json (config 5: D1, D2 in {8..128}),
<out>/<prefix>_rank_tables_r18_b32.json and <out>/<prefix>_rank_plan_r18_b32.json (greedy and
exact selections at B = 0.63, P:L555 / P:L582)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2211_03715_b200 import ranksel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--math", default="3xbf16")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--budget", type=float, default=0.63)
    ap.add_argument("--slack", type=float, default=0.05)
    ap.add_argument("--from-tables", help="re-run only the selection on a saved rank_tables json")
    ap.add_argument("--prefix", default="r02", help="output file prefix (round)")
    a = ap.parse_args()
    if a.from_tables:
        with open(a.from_tables) as f:
            dump = json.load(f)
        layers, tables = [], {}
        for obj in dump:
            l, t = ranksel.table_from_json(obj)
            layers.append(l)
            tables[l.name] = t
        select(layers, tables, a, dump[0]["math"], dump[0]["batch"], 0.0)
        return
    os.makedirs(a.out, exist_ok=True)
    iters = 10 if a.quick else 50
    t0 = time.time()
    # ---- config 5: 28x28x256 -> 256, 3x3, s1, D1, D2 in {8, 16, 32, 64, 128}
    cfg5 = ranksel.LayerSpec("sweep_28_256_256_s1", 28, 28, 256, 256, 3, 1, 1, 1)
    grid5 = [(d1, d2) for d1 in (8, 16, 32, 64, 128) for d2 in (8, 16, 32, 64, 128)]
    for b in (1, 32):
        tab = ranksel.measure_table(cfg5, grid5, b, a.math, iters)
        obj = ranksel.table_to_json(cfg5, tab, b, a.math)
        ranksel.save_json(os.path.join(a.out, f"{a.prefix}_rank_sweep_28x28x256_b{b}.json"), obj)
        print(f"config 5, batch {b}: " + " ".join(f"{k}:{v:.1f}" for k, v in sorted(tab.items())), flush=True)
    # ---- ResNet-18 layer list, grid at multiples of C/8, batch 32
    layers = ranksel.resnet18_layers()
    tables, dump = {}, []
    for l in layers:
        grid = ranksel.default_grid(l.C, l.N, ranksel.HALF_GRID)
        tables[l.name] = ranksel.measure_table(l, grid, 32, a.math, iters)
        dump.append(ranksel.table_to_json(l, tables[l.name], 32, a.math))
        print(f"{l.name}: measured {len(grid)} rank pairs", flush=True)
    ranksel.save_json(os.path.join(a.out, f"{a.prefix}_rank_tables_r18_b32.json"), dump)
    select(layers, tables, a, a.math, 32, time.time() - t0)


def select(layers, tables, a, math, batch, seconds):
    greedy = ranksel.select_ranks(layers, tables, a.budget, a.slack)
    exact = ranksel.select_ranks_exact(layers, tables, a.budget, a.slack)
    paper = {l.name: (l.C // 2, l.N // 2) for l in layers}
    lat_p, tk_p, orig = ranksel._totals(layers, tables, paper)
    out = {"budget": a.budget, "slack": a.slack, "math": math, "batch": batch,
           "greedy": greedy.to_json(), "exact": exact.to_json(),
           "paper_style_C/2": {"ranks": {k: list(v) for k, v in paper.items()}, "latency_us": round(lat_p, 3),
                               "reduction": round(1 - tk_p / orig, 6)},
           "seconds": round(seconds, 1)}
    ranksel.save_json(os.path.join(a.out, f"{a.prefix}_rank_plan_r18_b32.json"), out)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
