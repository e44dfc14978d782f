mkdir -p gpurun_out
python bench.py --no-cpu-baseline --e2e-steps 1 --config 5 --steps 2 --warmup 3 > gpurun_out/c5plain.json 2>&1; echo rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c5launches.csv python bench.py --no-cpu-baseline --e2e-steps 1 --config 5 --steps 2 --warmup 3 > gpurun_out/c5ncu.log 2>&1; echo ncu=$?
