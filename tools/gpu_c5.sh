# C5 / C2 / C4 back-to-back under env knobs (gpurun)
python tools/exp_b2b.py 5 base KS_LEAN=1 2>&1 | grep '"round": 1'
python tools/exp_b2b.py 2 base KS_LEAN=0 2>&1 | grep '"round": 1'
python tools/exp_b2b.py 4 base 2>&1 | grep '"round": 1'
KS_PHASE_TRACE=1 python tools/exp_env.py --config 5 --reps 2 base 2>&1 | tail -12
