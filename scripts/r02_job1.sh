#!/bin/bash
# Round-2 GPU job: re-measure rank tables (graph-replayed), rank-selected model tests,
# fused-vs-unfused step A/B, full bench.
set -x
python scripts/rank_sweep.py --prefix r02 > gpurun_out/rank_sweep_r02.log 2>&1
cp profiles/r02_rank_* gpurun_out/ 2>/dev/null
timeout 900 python -m pytest tests/test_model.py -m gpu -q -k "selected or small" > gpurun_out/model_tests.log 2>&1
TDC_NO_LAYER=1 python bench.py --no-model --no-e2e --no-cpu --no-b1 > gpurun_out/bench_nolayer.json 2>/dev/null
python bench.py --no-model --no-e2e --no-cpu --no-b1 > gpurun_out/bench_layer.json 2>/dev/null
python bench.py --no-model-sweep > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
