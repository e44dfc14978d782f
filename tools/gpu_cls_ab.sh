# Class-table A/B (gpurun): GPU tests with the default library, then the
# class kernel vs the ring kernel (KS_NO_CLS=1) on C3, then the class-buffer
# variant libraries (built into paper_1509_01506_b200/_lib_<name>/).
#   VARIANTS="r2c1 r3c2" bash tools/gpu_cls_ab.sh TAG
TAG=${1:-cls}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
python tools/exp_env.py --config 3 --reps 9 base KS_NO_CLS=1 > gpurun_out/ab_$TAG.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_$TAG.log
VARIANTS="${VARIANTS}" CONFIGS=3 bash tools/gpu_ab_libs.sh > gpurun_out/ablibs_$TAG.log 2>&1; cat gpurun_out/ablibs_$TAG.log
