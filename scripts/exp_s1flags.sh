mkdir -p gpurun_out/g16
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "core3 or r18_shapes_batch32 or deterministic or partial_batch or forward_host" > gpurun_out/g16/tests.txt 2>&1
tail -1 gpurun_out/g16/tests.txt
timeout 200 python scripts/layer_bench.py 3xbf16 0 2 > gpurun_out/g16/layers.txt 2>&1
TDC_NO_S1FLAGS=1 timeout 200 python scripts/layer_bench.py 3xbf16 0 2 >> gpurun_out/g16/layers.txt 2>&1
timeout 300 python -m pytest tests/test_model.py -q -x -m gpu > gpurun_out/g16/tests_model.txt 2>&1
timeout 200 python scripts/model_time.py > gpurun_out/g16/model_time.txt 2>&1
