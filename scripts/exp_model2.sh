mkdir -p gpurun_out/g8
timeout 900 python -m pytest tests/test_model.py -q -x -m gpu > gpurun_out/g8/tests.txt 2>&1
tail -1 gpurun_out/g8/tests.txt
echo default >> gpurun_out/g8/model_time.txt; python scripts/model_time.py >> gpurun_out/g8/model_time.txt 2>&1
echo BN64 >> gpurun_out/g8/model_time.txt; TDC_DENSE_BN=64 python scripts/model_time.py >> gpurun_out/g8/model_time.txt 2>&1
echo ring2 >> gpurun_out/g8/model_time.txt; TDC_DENSE_RING=2 python scripts/model_time.py >> gpurun_out/g8/model_time.txt 2>&1
echo BN64ring2 >> gpurun_out/g8/model_time.txt; TDC_DENSE_RING=2 TDC_DENSE_BN=64 python scripts/model_time.py >> gpurun_out/g8/model_time.txt 2>&1
TDC_DENSE_BN=64 timeout 600 python -m pytest tests/test_model.py -q -x -m gpu > gpurun_out/g8/tests_bn64.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g8/r50.csv python scripts/model_profile.py r50 > /dev/null 2>&1
python scripts/parse_launches.py gpurun_out/g8/r50.csv > gpurun_out/g8/r50_launches.txt 2>&1
