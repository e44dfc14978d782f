# C5 launch list (gpurun): plain run first, then ncu per-kernel durations, cold and warm L2
mkdir -p gpurun_out
python bench.py --no-cpu-baseline --e2e-steps 1 --config ${CFG:-5} --steps 2 --warmup 3 > gpurun_out/c5plain.json 2>&1; echo rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c5launches.csv python bench.py --no-cpu-baseline --e2e-steps 1 --config ${CFG:-5} --steps 2 --warmup 3 > gpurun_out/c5ncu.log 2>&1; echo ncu=$?
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv --log-file gpurun_out/c5launches_warm.csv python bench.py --no-cpu-baseline --e2e-steps 1 --config ${CFG:-5} --steps 2 --warmup 3 > gpurun_out/c5ncu2.log 2>&1; echo ncu=$?
