for i in c1 0 1 2 3 4 5 6; do python scripts/b1_hints.py $i "3xbf16:"; done
for i in 0 1 2 3 4 5 6; do LAYER_B=32 python scripts/b1_hints.py $i "3xbf16:"; done
