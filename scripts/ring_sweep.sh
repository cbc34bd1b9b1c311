# A/B of ring depths (shared-memory footprint) on the three-launch layers
for cfg in "" "TDC_GEMM_SX=4" "TDC_GEMM_SX=3" "TDC_CORE2_AS=2" "TDC_CORE2_WS=3" "TDC_GEMM_SX=3 TDC_CORE2_AS=2 TDC_CORE2_WS=3"; do
  echo "== $cfg"
  for i in 1 2 3 4 5 6; do env $cfg LAYER_B=32 python scripts/b1_hints.py $i "3xbf16:"; done
done
