#!/bin/bash
# Round-2 GPU job 3 (after the TMEM-operand layer kernel): GPU tests, smoke, default bench,
# ncu launch list of one bench step (traffic, tensor pipe), ncu --set full of the layer kernel
# and of the 7x7 core kernel.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err; echo "bench rc=$?" >> gpurun_out/bench_r02j.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg,gpc__cycles_elapsed.max \
    --clock-control none -c 45 --csv --log-file gpurun_out/launches_r02j.csv \
    python bench.py --steps 2 --warmup 3 --no-model --no-e2e --no-cpu --no-b1 --no-math-steps > gpurun_out/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launch_list_r02j.csv \
    python bench.py --steps 2 --warmup 3 --no-model --no-e2e --no-cpu --no-b1 --no-math-steps > gpurun_out/ncu_bench2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tdc_bf_layer -c 1 -s 2 -o gpurun_out/layer_full_r02j \
    python scripts/one_layer.py 0 4 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tdc_bf_core -c 1 -s 2 -o gpurun_out/core_full_r02j \
    python scripts/one_layer.py 6 4 > gpurun_out/ncu_full2.log 2>&1
