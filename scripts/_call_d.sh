timeout 600 python scripts/step_probe.py --reps 2 > gpurun_out/step_d.json 2>&1; tail -c 900 gpurun_out/step_d.json; echo
(timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gputest_d.log 2>&1; tail -3 gpurun_out/gputest_d.log
timeout 400 python scripts/c5_probe.py > gpurun_out/c5_probe_bins2.json 2>&1; tail -c 1200 gpurun_out/c5_probe_bins2.json; echo
MPG_SPAI_PHASES=1 timeout 400 python scripts/spai_time.py c5 --n 500000 --update > gpurun_out/spai_c5_phases.json 2>&1; cat gpurun_out/spai_c5_phases.json
MPG_SPAI_PHASES=1 timeout 400 python scripts/spai_time.py c3 --update > gpurun_out/spai_c3_phases.json 2>&1; cat gpurun_out/spai_c3_phases.json
