python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/exp_scan.py --config 3 --n 268435456 --variants default,chunk64,chunk128,chunk256,chunk512 > gpurun_out/exp3_c3.txt 2>&1
python tools/exp_scan.py --config 4 --n 268435456 --variants default,chunk64,chunk128,chunk256,chunk512 > gpurun_out/exp3_c4.txt 2>&1
echo done
