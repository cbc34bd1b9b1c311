"""Per-layer ncu evidence from the launch list of one bench step (VERDICT r1 'next' 1e):
DRAM read bytes, bytes written by the SMs into L2 (lts__t_sectors_srcunit_tex_op_write x 32
-- ncu closes each replayed kernel before its writes leave the 126 MB L2, so
dram__bytes_write undercounts; every written byte eventually goes to DRAM), tensor-pipe
and SM-active share of the elapsed cycles, mapped to the 16 Tucker-ResNet-18 layers.
Usage: python scripts/ncu_step_r02.py <launches.csv> <out prefix>"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2211_03715_b200 import roofline as rl  # noqa: E402

path, prefix = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
iid, iname, imet, ival = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ks = {}
for r in rows[1:]:
    k = ks.setdefault(int(r[iid]), {"name": r[iname]})
    try:
        k[r[imet]] = float(r[ival].replace(",", ""))
    except ValueError:
        pass
ks = [ks[i] for i in sorted(ks)]
short = lambda n: re.sub(r"\(.*", "", n).replace("void ", "").replace("tdc::", "")
# a layer forward starts at a stage-1 gemm or a single-launch layer kernel
starts = [i for i, k in enumerate(ks) if "tdc_bf_layer_" in k["name"] or
          re.search(r"tdc_bf_gemm_kernel<(\(bool\))?(1|true)[,>]", k["name"])]
groups = [ks[a:b] for a, b in zip(starts, starts[1:] + [len(ks)])]
names = [s for s, c in synth.R18_SHAPES for _ in range(c)]
groups = groups[:len(names)]
out, lines = {}, []
for shape, g in zip(names, groups):
    s = shape.with_batch(32)
    alg = rl.tkd_bytes(s)
    rd = sum(k.get("dram__bytes_read.sum", 0) for k in g)
    wr_dram = sum(k.get("dram__bytes_write.sum", 0) for k in g)
    wr_l2 = sum(k.get("lts__t_sectors_srcunit_tex_op_write.sum", 0) for k in g) * 32
    t = sum(k.get("gpu__time_duration.sum", 0) for k in g)
    per_k = [{"kernel": short(k["name"]), "us": round(k.get("gpu__time_duration.sum", 0) / 1e3, 2),
              "dram_read_MB": round(k.get("dram__bytes_read.sum", 0) / 1e6, 2),
              "l2_write_MB": round(k.get("lts__t_sectors_srcunit_tex_op_write.sum", 0) * 32 / 1e6, 2),
              "tensor_pct": round(k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0), 1),
              "sm_active_pct": round(100 * k.get("sm__cycles_active.avg", 0) / max(1, k.get("gpc__cycles_elapsed.max", 1)), 1)}
             for k in g]
    e = out.setdefault(s.name, {"alg_bytes": alg, "samples": []})
    e["samples"].append({"dram_read": int(rd), "dram_write": int(wr_dram), "l2_write": int(wr_l2),
                         "traffic": int(rd + wr_l2), "ratio_to_alg": round((rd + wr_l2) / alg, 3),
                         "ncu_us": round(t / 1e3, 2), "kernels": per_k})
for name, e in out.items():
    smp = e["samples"][0]
    lines.append(f"{name}: alg {e['alg_bytes'] / 1e6:.1f} MB, read {smp['dram_read'] / 1e6:.1f} + L2-write "
                 f"{smp['l2_write'] / 1e6:.1f} = {smp['traffic'] / 1e6:.1f} MB ({smp['ratio_to_alg']:.2f}x alg), "
                 f"ncu {smp['ncu_us']} us")
    for k in smp["kernels"]:
        lines.append(f"    {k['kernel']:<40s} {k['us']:7.2f} us  rd {k['dram_read_MB']:6.2f} MB  L2wr "
                     f"{k['l2_write_MB']:6.2f} MB  tensor {k['tensor_pct']:5.1f}%  SM active {k['sm_active_pct']:5.1f}%")
txt = "\n".join(lines)
print(txt)
with open(os.path.join(ROOT, "profiles", f"{prefix}_ncu_step_3xbf16.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\n"
            "#   lts__t_sectors_srcunit_tex_op_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\n"
            "#   sm__cycles_active.avg,gpc__cycles_elapsed.max --clock-control none, first bench step (cold, serialised)\n"
            + txt + "\n")
traffic = {name: e["samples"][0]["traffic"] for name, e in out.items()}
with open(os.path.join(ROOT, "profiles", f"{prefix}_ncu_traffic.json"), "w") as f:
    json.dump({"3xbf16": traffic, "detail": out,
               "_note": "traffic = dram__bytes_read.sum + 32 * lts__t_sectors_srcunit_tex_op_write.sum per layer "
                        "forward (bytes read from DRAM + bytes the SMs wrote, which reach DRAM when evicted); "
                        "first bench step of the launch list"}, f, indent=1)
