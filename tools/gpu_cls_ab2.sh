# Class-table tests + A/B (gpurun): the class-table tests, the C3 parity
# tests, then the default library (class vs ring) and variant libraries.
TAG=${1:-cls}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "class_table or full_size or config_cases or lean_blocks or dynamic or back_to_back" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
KS_KTIME=1 python tools/exp_env.py --config 3 --reps 3 base 2>&1 | tail -2
python tools/exp_env.py --config 3 --reps 9 base KS_NO_CLS=1 > gpurun_out/ab_$TAG.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_$TAG.log
VARIANTS="${VARIANTS}" CONFIGS=3 bash tools/gpu_ab_libs.sh > gpurun_out/ablibs_$TAG.log 2>&1; cat gpurun_out/ablibs_$TAG.log
