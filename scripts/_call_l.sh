(timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gputest_l.log 2>&1; tail -3 gpurun_out/gputest_l.log
timeout 900 python scripts/irka_prof.py --sweeps 6 2>&1 | tail -1 | cut -c1-1500
MPG_NO_IL_PAIRS=1 timeout 900 python scripts/irka_prof.py --sweeps 6 2>&1 | tail -1 | cut -c1-1500
