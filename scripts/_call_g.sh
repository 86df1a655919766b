timeout 600 python scripts/step_probe.py --reps 2 2>&1 | tail -1
MPG_GF_MBFULL=9 timeout 600 python scripts/step_probe.py --reps 2 2>&1 | tail -1
MPG_GF_MBFULL=3 timeout 600 python scripts/step_probe.py --reps 2 2>&1 | tail -1
(timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gputest_g.log 2>&1; tail -3 gpurun_out/gputest_g.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step_r02d.csv python scripts/step_probe.py --reps 0 > gpurun_out/ncu_launch_d.log 2>&1; gzip -f gpurun_out/launches_step_r02d.csv
