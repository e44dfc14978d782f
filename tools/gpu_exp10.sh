python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke10.log 2>&1; tail -1 gpurun_out/smoke10.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp10.log 2>&1; tail -3 gpurun_out/pytest_exp10.log
python bench.py --no-cpu-baseline > gpurun_out/bench_exp10.json 2> gpurun_out/bench_exp10.log
echo done
