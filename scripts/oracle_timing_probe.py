"""Why did two oracle timings on one box differ 2.6x?  Time one image
through the 16 R18 layers with and without torch imported first, and with
OMP_WAIT_POLICY active/passive (run as separate processes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "torch":
    import torch  # noqa: F401
import bench  # noqa: E402
import oracle  # noqa: E402

insts = bench.layer_instances(32)
ts = []
for _ in range(4):
    _, _, t = bench.run_oracle_sample(insts, 0.0)
    ts.append(t)
print(sys.argv[1:], os.environ.get("OMP_WAIT_POLICY"), oracle.max_threads(), [round(t * 1e3, 1) for t in ts], "ms/image")
