# Round-end evidence run (one B200): full GPU tests, benches, ncu launch list and full captures.
set -x
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.log 2>&1; tail -3 gpurun_out/final/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -3 gpurun_out/final/smoke.log
python bench.py > gpurun_out/final/bench_3xbf16.json 2> gpurun_out/final/bench_3xbf16.err
for m in tf32 3xtf32; do python bench.py --math $m --no-cpu --no-model > gpurun_out/final/bench_$m.json 2> gpurun_out/final/bench_$m.err; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/launches_3xbf16.csv python bench.py --math 3xbf16 --steps 2 --warmup 3 --no-e2e --no-cpu --no-model --no-graph > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tdc_bf --launch-count 2 -o gpurun_out/final/prof_bf16_56 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-model --no-graph > gpurun_out/final/ncu_full.log 2>&1
ls -la gpurun_out/final
