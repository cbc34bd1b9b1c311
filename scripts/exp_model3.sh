mkdir -p gpurun_out/g10
timeout 900 python -m pytest tests/test_model.py tests/test_parity_gpu.py -q -x -m gpu -k "model or three_launch or core3 or integer or ragged" > gpurun_out/g10/tests.txt 2>&1
tail -1 gpurun_out/g10/tests.txt
python scripts/model_time.py > gpurun_out/g10/model_time.txt 2>&1
python scripts/layer_bench.py 3xbf16 > gpurun_out/g10/layers.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g10/r50.csv python scripts/model_profile.py r50 > /dev/null 2>&1
python scripts/parse_launches.py gpurun_out/g10/r50.csv > gpurun_out/g10/r50_launches.txt 2>&1
