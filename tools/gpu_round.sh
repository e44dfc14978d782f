set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.log; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.log && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu rc=$?"
