mkdir -p gpurun_out/g28
timeout 400 python -m pytest tests/test_parity_gpu.py -q -x -k "core3 or integer or r18_shapes_batch1 or three_launch" > gpurun_out/g28/tests.txt 2>&1
tail -n 1 gpurun_out/g28/tests.txt
timeout 200 python scripts/layer_bench.py 3xbf16 > gpurun_out/g28/layers.txt 2>&1
timeout 200 python scripts/model_time.py > gpurun_out/g28/model_time.txt 2>&1
