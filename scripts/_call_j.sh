timeout 900 python scripts/irka_prof.py --sweeps 6 2>&1 | tail -1 | cut -c1-1500
timeout 600 python scripts/step_probe.py --reps 2 2>&1 | tail -1 | cut -c1-700
(timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gputest_j.log 2>&1; tail -3 gpurun_out/gputest_j.log
