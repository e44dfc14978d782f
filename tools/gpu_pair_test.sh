# Class-kernel tests, then tools/gpu_pair_ab.sh (gpurun).
TAG=${1:-pair}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "${KEXPR:-class_table or full_size or config_cases or lean_blocks or dynamic or back_to_back or stream or fasta or shard or multi}" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
bash tools/gpu_pair_ab.sh $TAG
