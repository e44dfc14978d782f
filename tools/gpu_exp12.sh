python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke12.log 2>&1; tail -1 gpurun_out/smoke12.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp12.log 2>&1; tail -3 gpurun_out/pytest_exp12.log
python bench.py --no-cpu-baseline > gpurun_out/bench_exp12.json 2> gpurun_out/bench_exp12.log; echo "bench rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --bases 268435456 > gpurun_out/bench_dist2.json 2> gpurun_out/bench_dist2.log; echo "rc=$?"
