mkdir -p gpurun_out
for mb in 64 32 16 8; do for nt in 1 0; do
KS_PIECE_MB=$mb KS_PACK_NT=$nt python bench.py --no-cpu-baseline --steps 3 --e2e-steps 5 > gpurun_out/bench_p${mb}_nt$nt.json 2>> gpurun_out/bench_pack.log
done; done
