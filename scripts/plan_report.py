"""Print the 3xBF16 planner's choices (variant, N tiles, split-K pieces) for the R18
layers at a batch (default 32).  Usage: python scripts/plan_report.py [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2211_03715_b200 import tdc  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
for s, _ in synth.R18_SHAPES:
    s = s.with_batch(b)
    plan = tdc.ConvPlan(s, synth.make_layer(s), math=tdc.TDC_MATH_3XBF16)
    i = plan.info()
    print(f"{s.name:20s} {i.variant_name:18s} bn {i.bn_stage1:3d}/{i.bn_core:3d}/{i.bn_stage3:3d} "
          f"gsplit {i.gsplit_stage1}/{i.gsplit_core}/{i.gsplit_stage3} ws {i.workspace_bytes / 1e6:.1f} MB")
    plan.close()
