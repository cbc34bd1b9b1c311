export TDC_LIB=$PWD/paper_2211_03715_b200/libtdc_kn.so
for k in 0 256; do
  echo "knob=$k"
  TDC_LAYER_DBG=$k python scripts/b1_hints.py c1 "3xbf16:"
  TDC_LAYER_DBG=$k python scripts/b1_hints.py 0 "3xbf16:"
  TDC_LAYER_DBG=$k LAYER_B=32 python scripts/b1_hints.py 0 "3xbf16:"
done
