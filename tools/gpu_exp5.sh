python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/exp_scan.py --config 3 --n 1073741824 --variants ring,chunk64,chunk128,chunk256,chunk512,chunk2k > gpurun_out/exp5_c3.txt 2>&1
python tools/exp_scan.py --config 4 --n 1073741824 --variants ring,chunk64,chunk128,chunk256 > gpurun_out/exp5_c4.txt 2>&1
echo done
