python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/exp_scan.py --config 3 --n 1073741824 --variants ring,direct > gpurun_out/exp4_c3.txt 2>&1
python tools/exp_scan.py --config 2 --n 268435456 --variants ring,direct > gpurun_out/exp4_c2.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp4.log 2>&1; tail -2 gpurun_out/pytest_exp4.log
CMD="python tools/exp_scan.py --config 3 --n 268435456 --reps 1 --variants direct"
$CMD > gpurun_out/exp4_plain.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:scan_fast -s 1 -c 1 -o gpurun_out/prof_direct_c3 $CMD > gpurun_out/ncu_exp4.log 2>&1
echo done
