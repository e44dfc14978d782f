# Pair-queue class kernel A/B (gpurun): back-to-back time per call of the
# in-tree library and the variant libraries in $VARIANTS, work-split knobs,
# KS_KTIME end spreads, one ncu --set full capture of the in-tree kernel.
TAG=${1:-pair}
mkdir -p gpurun_out
LIB=paper_1509_01506_b200/_lib/libkmerscan_b200.so
cp $LIB /tmp/base.so
for v in base ${VARIANTS}; do
  if [ $v = base ]; then cp /tmp/base.so $LIB; else cp paper_1509_01506_b200/_lib_$v/libkmerscan_b200.so $LIB; fi
  echo "== $v"
  python tools/exp_b2b.py 3 base ${KNOBS} 2>&1 | grep '"round": 1'
  KS_KTIME=1 python tools/exp_env.py --config 3 --reps 3 base 2>&1 | grep ktime | tail -1
done
cp /tmp/base.so $LIB
for lb in ${LBS}; do
  echo "== KS_TILE_LB=$lb"
  KS_TILE_LB=$lb python tools/exp_b2b.py 3 base ${KNOBS} 2>&1 | grep '"round": 1'
done
if [ -n "$NCU" ]; then
CMD="python tools/exp_env.py --config 3 --reps 3 base"
ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 4 -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv > gpurun_out/src_${TAG}.csv 2>/dev/null
echo "ncu rc=$?"
fi
