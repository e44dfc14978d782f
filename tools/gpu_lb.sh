for lb in 5; do for k in "KS_DYN_MIN_ROUNDS=3" "KS_DYN_MIN_ROUNDS=3,KS_SPLIT_PARTS=4" "KS_DYN_MIN_ROUNDS=3,KS_SPLIT_PARTS=4,KS_DYN_ROUNDS=1" "KS_DYN_MIN_ROUNDS=3,KS_SPLIT_PARTS=8,KS_DYN_ROUNDS=1"; do echo "== lb=$lb $k"; KS_TILE_LB=$lb python tools/exp_b2b.py 3 $k 2>&1 | grep '"round": 1'; done; done
python tools/exp_b2b.py 3 base 2>&1 | grep '"round": 1'
