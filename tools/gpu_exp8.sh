python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke8.log 2>&1; tail -1 gpurun_out/smoke8.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp8.log 2>&1; tail -3 gpurun_out/pytest_exp8.log
python tools/exp_scan.py --config 3 --n 1073741824 --variants ring,direct > gpurun_out/exp8_c3.txt 2>&1
python tools/exp_scan.py --config 4 --n 1073741824 --variants ring > gpurun_out/exp8_c4.txt 2>&1
python tools/exp_scan.py --config 2 --n 67108864 --variants ring > gpurun_out/exp8_c2.txt 2>&1
echo done
