# usage: bash tools/gpu_round.sh [tag]   (run on the GPU box via gpurun)
TAG=${1:-r}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc=$?"
for c in 1 2 4 5; do python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_c$c.json 2>> gpurun_out/bench_$TAG.log; done
