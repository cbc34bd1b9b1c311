mkdir -p gpurun_out/g7
timeout 900 python -m pytest tests/test_model.py -q -x -m gpu > gpurun_out/g7/tests.txt 2>&1
tail -3 gpurun_out/g7/tests.txt
python scripts/model_time.py > gpurun_out/g7/model_time.txt 2>&1
TDC_NO_STEM=1 python scripts/model_time.py >> gpurun_out/g7/model_time.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g7/r50.csv python scripts/model_profile.py r50 > /dev/null 2>&1
python scripts/parse_launches.py gpurun_out/g7/r50.csv > gpurun_out/g7/r50_launches.txt 2>&1
