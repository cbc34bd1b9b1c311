#!/bin/bash
# A/B of the headline step: layer kernel off / on (tap pairs off / on), 3 repeats each
for i in 1 2 3; do
  for cfg in "TDC_NO_LAYER=1" "TDC_LAYER_TN=0" "TDC_LAYER_TN=1"; do
    env $cfg python bench.py --no-model --no-e2e --no-cpu --no-b1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['layers'][0]['us'], d['layers'][0]['variant'])"
  done
done
