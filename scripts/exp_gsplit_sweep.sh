mkdir -p gpurun_out/g2
off="gsplit_stage1=1,gsplit_core=1,gsplit_stage3=1"
python scripts/hint_sweep.py 6 "$off" \
 "gsplit_stage1=2,gsplit_core=1,gsplit_stage3=1" "gsplit_stage1=4,gsplit_core=1,gsplit_stage3=1" \
 "gsplit_stage1=1,gsplit_core=2,gsplit_stage3=1" "gsplit_stage1=1,gsplit_core=4,gsplit_stage3=1" "gsplit_stage1=1,gsplit_core=8,gsplit_stage3=1" \
 "bn_core=128,gsplit_stage1=1,gsplit_core=1,gsplit_stage3=1" "bn_core=128,gsplit_stage1=1,gsplit_core=3,gsplit_stage3=1" \
 "gsplit_stage1=1,gsplit_core=1,gsplit_stage3=2" "bn_stage3=128,gsplit_stage1=1,gsplit_core=1,gsplit_stage3=2" > gpurun_out/g2/sweep6.txt 2>&1
python scripts/hint_sweep.py 5 "$off" "gsplit_stage1=1,gsplit_core=2,gsplit_stage3=1" "gsplit_stage1=2,gsplit_core=1,gsplit_stage3=1" "gsplit_stage1=1,gsplit_core=1,gsplit_stage3=2" > gpurun_out/g2/sweep5.txt 2>&1
python scripts/hint_sweep.py 4 "$off" "gsplit_stage1=2,gsplit_core=1,gsplit_stage3=1" "gsplit_stage1=1,gsplit_core=2,gsplit_stage3=1" "gsplit_stage1=1,gsplit_core=1,gsplit_stage3=2" > gpurun_out/g2/sweep4.txt 2>&1
