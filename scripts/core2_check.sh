# CTA-pair core: variants, parity at batch 32 (full images), timing with and without it
for i in 1 2 3 4 5 6; do LAYER_B=32 timeout 60 python scripts/b1_hints.py $i "3xbf16:"; LAYER_B=32 TDC_CORE2=0 timeout 60 python scripts/b1_hints.py $i "3xbf16:"; done
timeout 600 python -m pytest tests/test_headline_gpu.py -x -q 2>&1 | tail -3
