# core3 (56x56 s1 layer) time with parts of the kernel switched off (TDC_CORE_DBG bits, wrong results):
# debug knobs (TDC_*_DBG, TDC_Y_DIRECT) exist only in the debug/timeline build
export TDC_LIB=paper_2211_03715_b200/libtdc_tl.so  # python paper_2211_03715_b200/build.py --timeline
# 1 no Y stores, 2 no Z smem writes, 4 no band reloads after tile 1, 8 no S3 MMAs, 16 no acc2-free wait,
# 32 no E2 TMEM loads
mkdir -p gpurun_out/g23
for d in 0 1 2 4 8 32 5 13 45 47; do echo "DBG=$d $(TDC_CORE_DBG=$d python scripts/layer_bench.py 3xbf16 0 2>&1 | tail -1)" >> gpurun_out/g23/dbg.txt; done
