# A/B of core3 epilogue knobs on the two core3 layers (56x56 s1, 28x28 s1)
# debug knobs (TDC_*_DBG, TDC_Y_DIRECT) exist only in the debug/timeline build
export TDC_LIB=paper_2211_03715_b200/libtdc_tl.so  # python paper_2211_03715_b200/build.py --timeline
mkdir -p gpurun_out/g3
o=gpurun_out/g3/knobs.txt
echo base >> $o; python scripts/layer_bench.py 3xbf16 0 2 >> $o 2>&1
echo Y_DIRECT >> $o; TDC_Y_DIRECT=1 python scripts/layer_bench.py 3xbf16 0 2 >> $o 2>&1
echo NO_NCAT3 >> $o; TDC_NO_NCAT3=1 python scripts/layer_bench.py 3xbf16 0 2 >> $o 2>&1
echo NO_NCAT3+Y_DIRECT >> $o; TDC_NO_NCAT3=1 TDC_Y_DIRECT=1 python scripts/layer_bench.py 3xbf16 0 2 >> $o 2>&1
echo DBG1_noYstore >> $o; TDC_CORE_DBG=1 python scripts/layer_bench.py 3xbf16 0 2 >> $o 2>&1
echo DBG8_noS3 >> $o; TDC_CORE_DBG=8 python scripts/layer_bench.py 3xbf16 0 2 >> $o 2>&1
echo DBG9 >> $o; TDC_CORE_DBG=9 python scripts/layer_bench.py 3xbf16 0 2 >> $o 2>&1
echo gsplit_test >> $o; timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "l2_split or small_layers_planned" >> $o 2>&1
