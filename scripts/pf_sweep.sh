for pf in 0 2 4 6 8 12; do TDC_LAYER_PF=$pf TDC_LIB=$PWD/paper_2211_03715_b200/libtdc_kn.so python scripts/layer_knobs.py 0 0 15 2>&1 | sed "s/^/pf=$pf /"; done
