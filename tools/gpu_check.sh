# Quick GPU pass (run under gpurun):  bash tools/gpu_check.sh TAG
#   build, smoke, pytest -m gpu (incl. the full-size parity tests), default bench,
#   a gloo dry run of the 2-rank path (both ranks on the one GPU, small strong leg)
TAG=${1:-chk}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -20 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc=$?"
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --e2e-steps 1 --strong-bases 400000000 > gpurun_out/gloo2_$TAG.json 2> gpurun_out/gloo2_$TAG.log; echo "gloo2 rc=$?"
tail -c 1500 gpurun_out/bench_$TAG.json
