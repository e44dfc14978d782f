LIB=paper_1509_01506_b200/_lib/libkmerscan_b200.so
cp $LIB /tmp/base.so
for c in 3 4 2 5; do
 for v in base pdl base pdl; do
  if [ $v = base ]; then cp /tmp/base.so $LIB; else cp paper_1509_01506_b200/_lib_pdl/libkmerscan_b200.so $LIB; fi
  KS_ASYNC_NO_EVENTS=1 python bench.py --no-cpu-baseline --e2e-steps 1 --config $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c', '$v', round(d['value']), round(d['ms_per_step']*1000,1))"
 done
done
cp /tmp/base.so $LIB
