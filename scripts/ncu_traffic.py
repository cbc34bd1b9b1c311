"""Map an ncu per-launch list of one bench step onto the 16 TKD layers and write
per-layer DRAM traffic (read+write bytes per forward) to profiles/ncu_traffic.json.
Usage: python scripts/ncu_traffic.py <math> <launches.csv>"""
import json
import os
import statistics
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from scripts.parse_launches import load  # noqa: E402

math, path = sys.argv[1], sys.argv[2]
ks = load(path)
# group launches into layer forwards: 3xBF16 = a stage-1 launch (tdc_bf_gemm_kernel<1>)
# followed by core3, or core + stage-3 gemm; TF32/3xTF32 three-launch = gemm, (core|gemm),
# gemm; fused/simt = 1 launch
groups, i = [], 0
while i < len(ks):
    n = ks[i]["name"]
    if re.search(r"tdc_bf_gemm_kernel<(\(bool\))?(1|true)[,>]", n):
        j = i + 1
        while j < len(ks) and not re.search(r"tdc_bf_gemm_kernel<(\(bool\))?(1|true)[,>]", ks[j]["name"]) and j - i < 3:
            j += 1
        groups.append(ks[i:j])
        i = j
    elif "tc_gemm" in n:
        groups.append(ks[i:i + 3])
        i += 3
    else:
        groups.append(ks[i:i + 1])
        i += 1
names = [s.name for s, c in synth.R18_SHAPES for _ in range(c)]
steps = len(groups) // len(names)
# the first bench step: bench.py times each layer alone after the steps, so the tail of
# the list is the last layer repeated; ncu flushes caches per launch, so any step is as cold
last = groups[:len(names)]
per = {}
for nm, g in zip(names, last):
    b = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in g)
    t = sum(k.get("gpu__time_duration.sum", 0) for k in g)
    per.setdefault(nm, []).append((b, t, [k["name"] for k in g]))
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_traffic.json")
data = json.load(open(out_path)) if os.path.exists(out_path) else {}
data[math] = {nm: int(statistics.mean(b for b, _, _ in v)) for nm, v in per.items()}
data[math + "_ncu_us"] = {nm: round(statistics.mean(t for _, t, _ in v) / 1e3, 2) for nm, v in per.items()}
data[math + "_kernels"] = {nm: v[0][2] for nm, v in per.items()}
data["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per layer forward, from the ncu "
                 "launch list of one bench step (cold-cache, serialised replay); writes that stay in "
                 "the 126 MB L2 past the kernel's end are not counted, so this is mostly read "
                 "traffic; ncu_us is the ncu duration of the same launches (not a bench number)")
json.dump(data, open(out_path, "w"), indent=1)
print(json.dumps({k: data[k] for k in (math, math + "_ncu_us")}, indent=1))
print("steps seen:", steps, "groups:", len(groups))
