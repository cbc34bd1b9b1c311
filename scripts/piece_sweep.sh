for lib in libtdc.so libtdc_p4096.so libtdc_p8192.so libtdc_p32768.so; do
  echo "== $lib"
  for i in 1 2 3 4 5 6; do TDC_LIB=$PWD/paper_2211_03715_b200/$lib LAYER_B=32 python scripts/b1_hints.py $i "3xbf16:"; done
done
