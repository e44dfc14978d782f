python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke9.log 2>&1; tail -1 gpurun_out/smoke9.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp9.log 2>&1; tail -3 gpurun_out/pytest_exp9.log
python tools/exp_scan.py --config 3 --n 1073741824 --variants ring > gpurun_out/exp9_c3.txt 2>&1
python tools/exp_scan.py --config 4 --n 1073741824 --variants ring > gpurun_out/exp9_c4.txt 2>&1
python tools/exp_scan.py --config 2 --n 268435456 --variants ring > gpurun_out/exp9_c2.txt 2>&1
python tools/exp_scan.py --config 5 --n 268435456 --variants ring > gpurun_out/exp9_c5.txt 2>&1
echo done
