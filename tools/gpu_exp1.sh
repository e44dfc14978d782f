python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/exp_scan.py --config 3 --n 268435456 --variants default,generic,chunk2k,chunk16k > gpurun_out/exp1_c3.txt 2>&1
python tools/exp_scan.py --config 4 --n 268435456 --variants default,generic,chunk2k > gpurun_out/exp1_c4.txt 2>&1
CMD="python tools/exp_scan.py --config 3 --n 67108864 --reps 1"
$CMD > gpurun_out/exp1_plain.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 1 -c 1 -o gpurun_out/prof_fast_c3 $CMD > gpurun_out/ncu_exp1.log 2>&1
echo done
