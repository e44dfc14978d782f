# Full measurement pass (run on the GPU box via gpurun):  bash tools/gpu_round.sh TAG
#   smoke, pytest -m gpu, bench (C3 default + C1/C2/C4/C5), the reference arm,
#   the ncu launch list of the default bench command, one ncu --set full
#   capture of the scan kernel per config (3, 4, 5), raw csv exports.
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc=$?"
for c in 1 2 4 5; do python bench.py --config $c --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_${TAG}_c$c.json 2>> gpurun_out/bench_$TAG.log; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_$TAG.log
python tools/exp_fasta.py > gpurun_out/fasta_$TAG.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1_$TAG.log 2>&1
echo "ncu launches rc=$?"
for c in 3 4 5; do
  $CMD --config $c > gpurun_out/plain_${TAG}_c$c.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 3 -c 1 -o gpurun_out/prof_${TAG}_c$c $CMD --config $c > gpurun_out/ncu2_${TAG}_c$c.log 2>&1 && \
  ncu -i gpurun_out/prof_${TAG}_c$c.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_c$c.csv 2>/dev/null
  echo "ncu full c$c rc=$?"
done
