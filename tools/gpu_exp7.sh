python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python tools/exp_scan.py --config 3 --n 1073741824 --reps 1 --variants ring"
$CMD > gpurun_out/exp7_plain.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 1 -c 1 -o gpurun_out/prof_tiled_c3 $CMD > gpurun_out/ncu_exp7.log 2>&1
CMD="python tools/exp_scan.py --config 4 --n 1073741824 --reps 1 --variants ring"
$CMD > gpurun_out/exp7_plain4.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 1 -c 1 -o gpurun_out/prof_tiled_c4 $CMD > gpurun_out/ncu_exp7b.log 2>&1
echo done
