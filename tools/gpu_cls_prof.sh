# ncu --set full of the C3 count kernel: class table (default and $VARIANT
# library) vs the ring kernel; KS_KTIME phase stamps of each (gpurun).
TAG=${1:-clsp}
mkdir -p gpurun_out
CMD="python tools/exp_env.py --config 3 --reps 3"
for v in base KS_NO_CLS=1; do
  KS_KTIME=1 $CMD $v 2>&1 | tail -4 > gpurun_out/ktime_${TAG}_$v.log
  ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 4 -c 1 -o gpurun_out/prof_${TAG}_$v $CMD $v > gpurun_out/ncu_${TAG}_$v.log 2>&1
  ncu -i gpurun_out/prof_${TAG}_$v.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_$v.csv 2>/dev/null
  ncu -i gpurun_out/prof_${TAG}_$v.ncu-rep --page source --csv > gpurun_out/src_${TAG}_$v.csv 2>/dev/null
  echo "ncu $v rc=$?"
done
if [ -n "$VARIANT" ]; then
  cp paper_1509_01506_b200/_lib_$VARIANT/libkmerscan_b200.so paper_1509_01506_b200/_lib/libkmerscan_b200.so
  KS_KTIME=1 $CMD base 2>&1 | tail -4 > gpurun_out/ktime_${TAG}_$VARIANT.log
  ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 4 -c 1 -o gpurun_out/prof_${TAG}_$VARIANT $CMD base > gpurun_out/ncu_${TAG}_$VARIANT.log 2>&1
  ncu -i gpurun_out/prof_${TAG}_$VARIANT.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_$VARIANT.csv 2>/dev/null
  ncu -i gpurun_out/prof_${TAG}_$VARIANT.ncu-rep --page source --csv > gpurun_out/src_${TAG}_$VARIANT.csv 2>/dev/null
  echo "ncu $VARIANT rc=$?"
fi
