# Build-variant A/B (gpurun): bench C$CONFIG with the in-tree library and with
# each variant library paper_1509_01506_b200/_lib_<name>/ built beforehand by
#   make -C paper_1509_01506_b200/csrc OUT=../_lib_<name> EXTRA=-D...
# usage: VARIANTS="chk6 chk8" CONFIG=3 bash tools/gpu_exp_lib.sh
mkdir -p gpurun_out
LIB=paper_1509_01506_b200/_lib/libkmerscan_b200.so
cp $LIB /tmp/base.so
for v in base ${VARIANTS} base; do
  if [ $v = base ]; then cp /tmp/base.so $LIB; else cp paper_1509_01506_b200/_lib_$v/libkmerscan_b200.so $LIB; fi
  python bench.py --no-cpu-baseline --e2e-steps 1 --config ${CONFIG:-3} 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['roofline']['kernel_ms'],4))"
done
cp /tmp/base.so $LIB
