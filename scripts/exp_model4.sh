mkdir -p gpurun_out/g11
# debug knobs (TDC_*_DBG, TDC_Y_DIRECT) exist only in the debug/timeline build
export TDC_LIB=paper_2211_03715_b200/libtdc_tl.so  # python paper_2211_03715_b200/build.py --timeline
o=gpurun_out/g11/model_time.txt
for cfg in "" "TDC_DENSE_BN=64" "TDC_GEMM_DBG=1" "TDC_GEMM_DBG=2" "TDC_NO_STEM=1"; do echo "cfg $cfg" >> $o; env $cfg python scripts/model_time.py >> $o 2>&1; done
