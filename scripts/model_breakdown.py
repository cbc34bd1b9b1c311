"""Map an ncu launch list of one Tucker ResNet-50 forward (scripts/model_profile.py) to ops."""
import re
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.parse_launches import load
import synth.models as sm
ks = load(sys.argv[1])
ops = sm.tucker_resnet(50)
nl_of = []
for o in ops:
    k = o["kind"]
    if k == 0:
        if o["c_in"] <= 4:
            nl_of.append(1)
        else:
            nl_of.append(1 if (o["kernel"] == 1 and o["stride"] == 1 and o["pad"] == 0) else 2)
    elif k == 1:
        nl_of.append(None)
    else:
        nl_of.append(1)
# total launches per forward
def count(start):
    i = start; n = 0
    for o, nl in zip(ops, nl_of):
        if nl is None:
            nl = 2 if re.search(r"core_kernel<(\(bool\))?(1|true)[,>]", ks[i + 1]["name"]) else 3
        i += nl; n += nl
    return n
n = count(len(ks) - 200 if len(ks) > 200 else 0)
last = ks[-n:]
i = 0; rows = []
for oi, (o, nl) in enumerate(zip(ops, nl_of)):
    if nl is None:
        nl = 2 if re.search(r"core_kernel<(\(bool\))?(1|true)[,>]", last[i + 1]["name"]) else 3
    t = sum(x.get("gpu__time_duration.sum", 0) for x in last[i:i + nl]) / 1e3
    rows.append((t, oi, o["kind"], o["c_in"], o["c_out"], o["kernel"], o["stride"], o["height"], nl))
    i += nl
tot = sum(r[0] for r in rows)
print("launches", n, "total us", round(tot, 1))
agg = {}
for r in rows:
    agg[r[2]] = agg.get(r[2], 0) + r[0]
print({["conv", "tkd", "maxpool", "avgpool", "fc"][k]: round(v, 1) for k, v in agg.items()})
for r in sorted(rows, reverse=True)[:12]:
    print("%7.1f us op%2d kind%d C%4d N%4d K%d s%d H%3d launches%d" % r)
