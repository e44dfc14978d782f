# Plain-item loop in every count / map kernel vs the class count only (gpurun):
# GPU tests with the in-tree library, then back-to-back times per config.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_plain.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_plain.log
LIB=paper_1509_01506_b200/_lib/libkmerscan_b200.so
cp $LIB /tmp/base.so
for v in base ${VARIANTS}; do
  if [ $v = base ]; then cp /tmp/base.so $LIB; else cp paper_1509_01506_b200/_lib_$v/libkmerscan_b200.so $LIB; fi
  echo "== $v"
  python tools/exp_b2b.py 3,4,5,2,1 base 2>&1 | grep '"round": 1'
done
cp /tmp/base.so $LIB
