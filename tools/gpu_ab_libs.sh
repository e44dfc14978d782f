# A/B of variant libraries (gpurun): for each lib in base + $VARIANTS (built
# beforehand into paper_1509_01506_b200/_lib_<name>/), time the scan kernel on
# each config in $CONFIGS with tools/exp_env.py (counts checksum printed, so
# variants can be compared with the base library's).
#   VARIANTS="pair" CONFIGS="3 4" bash tools/gpu_ab_libs.sh > gpurun_out/ab.log
LIB=paper_1509_01506_b200/_lib/libkmerscan_b200.so
cp $LIB /tmp/base.so
for round in 1 2; do
for v in base ${VARIANTS}; do
  if [ $v = base ]; then cp /tmp/base.so $LIB; else cp paper_1509_01506_b200/_lib_$v/libkmerscan_b200.so $LIB; fi
  for c in ${CONFIGS:-3}; do
    echo "== $v C$c round $round"
    python tools/exp_env.py --config $c --reps 9 base 2>&1 | grep '"round": 1'
  done
done
done
cp /tmp/base.so $LIB
