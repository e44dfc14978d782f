# one ncu --set full capture of the C3 count kernel (gpurun); TAG as $1
TAG=${1:-p}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 3 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu2_$TAG.log 2>&1
echo "ncu rc=$?"
