mkdir -p gpurun_out/g18
timeout 400 python -m pytest tests/test_model.py -q -x -m gpu > gpurun_out/g18/tests.txt 2>&1
tail -n 1 gpurun_out/g18/tests.txt
timeout 200 python scripts/model_time.py > gpurun_out/g18/model_time.txt 2>&1
TDC_DENSE_NO_GSPLIT=1 timeout 200 python scripts/model_time.py >> gpurun_out/g18/model_time.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g18/vgg.csv python scripts/model_profile.py vgg16 > /dev/null 2>&1
python scripts/model_ops.py gpurun_out/g18/vgg.csv vgg16 > gpurun_out/g18/vgg_ops.txt 2>&1
