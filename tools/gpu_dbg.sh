for n in 1000 20000 100000 400000; do echo "== n=$n"; python tools/dbg_seed.py 20261036 $n 2>&1 | grep -v '^  ' | tail -5; done
