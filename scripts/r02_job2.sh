#!/bin/bash
# Round-2 GPU job 2: exhaustive tiling search (NEXT-3), ncu launch list of one bench step with
# L2-write and tensor-pipe metrics, ncu --set full of the single-launch layer kernel.
python scripts/tiling_search_r18.py r02 > gpurun_out/tiling_search.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg,gpc__cycles_elapsed.max \
    --clock-control none -c 45 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-model --no-e2e --no-cpu --no-b1 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tdc_bf_layer -c 1 -s 2 -o gpurun_out/layer_full_r02 \
    python scripts/one_layer.py 0 4 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tdc_bf_core -c 1 -s 2 -o gpurun_out/core_full_r02 \
    python scripts/one_layer.py 6 4 > gpurun_out/ncu_full2.log 2>&1
