# Full measurement pass (run on the GPU box via gpurun):  bash tools/gpu_round.sh TAG
#   smoke, pytest -m gpu, the default bench (C3 + parity + others C1/C2/C4/C5),
#   the reference arm on the same config, a gloo dry run of the 2-rank path,
#   the ncu launch list of the default bench command, one ncu --set full
#   capture of the scan kernel per config (C3, C4, C5, C2) and of the wide
#   (> 32767 states) count kernel, raw csv exports.
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_$TAG.log; echo "ref rc=$?"
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/gloo2_$TAG.json 2> gpurun_out/gloo2_$TAG.log; echo "gloo2 rc=$?"
python tools/exp_fasta.py > gpurun_out/fasta_$TAG.log 2>&1
python tools/exp_bigdfa.py > gpurun_out/bigdfa_$TAG.log 2>&1; python tools/exp_bigdfa.py wide >> gpurun_out/bigdfa_$TAG.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity"
$CMD --no-others > gpurun_out/plain_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD --no-others > gpurun_out/ncu1_$TAG.log 2>&1
echo "ncu launches rc=$?"
for c in 3 4 5 2; do
  $CMD --no-others --config $c > gpurun_out/plain_${TAG}_c$c.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 3 -c 1 -o gpurun_out/prof_${TAG}_c$c $CMD --no-others --config $c > gpurun_out/ncu2_${TAG}_c$c.log 2>&1 && \
  ncu -i gpurun_out/prof_${TAG}_c$c.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_c$c.csv 2>/dev/null
  echo "ncu full c$c rc=$?"
done
python tools/exp_wide_one.py 4000 14 > gpurun_out/wide_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_wide -s 2 -c 1 -o gpurun_out/prof_${TAG}_wide python tools/exp_wide_one.py 4000 14 > /dev/null 2>&1 && \
ncu -i gpurun_out/prof_${TAG}_wide.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_wide.csv 2>/dev/null
echo "ncu wide rc=$?"
