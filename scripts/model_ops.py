"""Map the last Tucker ResNet-50 forward of an ncu launch list (scripts/model_profile.py)
to its ops and print each op's kernel time next to its HBM-ideal time (fp32 activations
in/out + residual, at the measured HBM peak).  Usage: python scripts/model_ops.py launches.csv [r50|vgg16]"""
import csv
import io
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth.models as sm  # noqa: E402

txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
ks = {}
for r in rows:
    e = ks.setdefault(r["ID"], {"name": r["Kernel Name"], "t": 0.0})
    if r["Metric Name"] == "gpu__time_duration.sum":
        e["t"] = float(r["Metric Value"].replace(",", "")) / 1e3
ks = list(ks.values())
start = max(i for i, k in enumerate(ks) if "stem" in k["name"] or "direct_conv" in k["name"])
ks = ks[start:]
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6553.0
arch = sys.argv[2] if len(sys.argv) > 2 else "r50"
B = 32 if arch == "r50" else 64
ops = sm.tucker_resnet(50) if arch == "r50" else sm.tucker_vgg16()
i = 0
tot = tot_ideal = 0.0
agg = {}
for oi, o in enumerate(ops):
    kind = o["kind"]
    H, W, C, N, K, s = o["height"], o["width"], o["c_in"], o["c_out"], o["kernel"], o["stride"]
    Ho = (H + 2 * o["pad"] - K) // s + 1 if kind in (0, 1, 2) else 1
    Wo = (W + 2 * o["pad"] - K) // s + 1 if kind in (0, 1, 2) else 1
    if kind == 0:
        n = 1 if (C <= 4 or (K == 1 and s == 1 and o["pad"] == 0)) else 2
    elif kind == 1:
        n = 2 if re.search(r"core_kernel<(\(bool\))?(1|true)[,>]", ks[i + 1]["name"]) else 3
    else:
        n = 1
    t = sum(k["t"] for k in ks[i:i + n])
    i += n
    if kind == 4:
        byts = B * (C + N) * 4 + C * N * 4
    else:
        byts = B * (H * W * C + Ho * Wo * (N if kind in (0, 1) else C)) * 4 + (B * Ho * Wo * N * 4 if o["res"] >= 0 else 0)
    ideal = byts / (peak * 1e3)
    label = ["conv", "tkd", "maxpool", "avgpool", "fc"][kind]
    agg[label] = agg.get(label, 0) + t
    tot += t
    tot_ideal += ideal
    print(f"op{oi:2d} {label:7s} C{C:4d} N{N:4d} K{K} s{s} H{H:3d} res{int(o['res'] >= 0)} {t:8.1f} us  "
          f"ideal {ideal:6.1f} us  x{t / ideal:5.1f}")
print(f"total {tot:.1f} us, HBM-ideal {tot_ideal:.1f} us;", {k: round(v, 1) for k, v in agg.items()})
