mkdir -p gpurun_out/exp1
for cfg in "0 4" "3 6" "3 8" "1 16" "1 24" "9 2"; do set -- $cfg; echo "TG=$1 WS=$2" >> gpurun_out/exp1/out.txt; TDC_CORE_TG=$1 TDC_CORE_WS=$2 python scripts/layer_bench.py 3xbf16 1 3 4 5 6 >> gpurun_out/exp1/out.txt 2>&1; done
