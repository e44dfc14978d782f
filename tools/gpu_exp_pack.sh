# host-pack e2e check (gpurun)
mkdir -p gpurun_out
g++ -O3 -std=c++17 -Ipaper_1509_01506_b200/csrc -I/usr/local/cuda/include tools/pack_bench.cpp paper_1509_01506_b200/_lib/obj/host_pack.o -lpthread -o /tmp/pack_bench && /tmp/pack_bench > gpurun_out/pack_bench.txt 2>&1
grep -o -E "avx512[a-z_0-9]*" /proc/cpuinfo | sort -u | tr '\n' ' ' >> gpurun_out/pack_bench.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "host_ascii" > gpurun_out/pytest_pack.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pack.log
python bench.py --no-cpu-baseline > gpurun_out/bench_pack.json 2> gpurun_out/bench_pack.log; echo "bench rc=$?"
for t in 8 12; do KS_HOST_THREADS=$t python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_pack_t$t.json 2>> gpurun_out/bench_pack.log; done
