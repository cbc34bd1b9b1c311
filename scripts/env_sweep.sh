#!/bin/bash
# A/B sweep of planner env knobs on one layer: scripts/env_sweep.sh <shape idx> "ENV=.. ENV2=.." ...
idx=$1; shift
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 120 python scripts/layer_knobs.py $idx 0 2>&1 | tail -1
done
