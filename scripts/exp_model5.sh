mkdir -p gpurun_out/g12
timeout 900 python -m pytest tests/test_model.py tests/test_parity_gpu.py -q -x -m gpu > gpurun_out/g12/tests.txt 2>&1
tail -1 gpurun_out/g12/tests.txt
o=gpurun_out/g12/model_time.txt
for cfg in "" "TDC_DENSE_RING=4"; do echo "cfg $cfg" >> $o; env $cfg python scripts/model_time.py >> $o 2>&1; done
python scripts/layer_bench.py 3xbf16 > gpurun_out/g12/layers.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g12/r50.csv python scripts/model_profile.py r50 > /dev/null 2>&1
python scripts/model_ops.py gpurun_out/g12/r50.csv > gpurun_out/g12/r50_ops.txt 2>&1
