mkdir -p gpurun_out/g21
timeout 600 python -m pytest tests/test_model.py -q -x -m gpu > gpurun_out/g21/tests.txt 2>&1
tail -n 1 gpurun_out/g21/tests.txt
timeout 200 python scripts/model_time.py > gpurun_out/g21/model_time.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g21/r50.csv python scripts/model_profile.py r50 > /dev/null 2>&1
python scripts/model_ops.py gpurun_out/g21/r50.csv r50 > gpurun_out/g21/r50_ops.txt 2>&1
