mkdir -p gpurun_out/g6
timeout 900 python -m pytest tests/test_model.py tests/test_parity_gpu.py -q -x -m gpu -k "model or three_launch or l2_split or forward_host or residual or epilogue or ex" > gpurun_out/g6/tests.txt 2>&1
tail -3 gpurun_out/g6/tests.txt
python scripts/model_time.py > gpurun_out/g6/model_time.txt 2>&1
python scripts/layer_bench.py 3xbf16 > gpurun_out/g6/layers.txt 2>&1
