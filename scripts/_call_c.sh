(timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_kernels.py "tests/test_golden_large.py::test_gpu_c5_sweep_matches_golden" -m gpu -q) > gpurun_out/gputest_c.log 2>&1; tail -3 gpurun_out/gputest_c.log
timeout 300 python scripts/spai_time.py c3 --update > gpurun_out/spai_c3.json 2>&1; cat gpurun_out/spai_c3.json
for w in 0 8 4; do if [ $w = 0 ]; then timeout 400 python scripts/spai_time.py c5 --update > gpurun_out/spai_c5_w$w.json 2>&1; else MPG_SPAI_WPS=$w timeout 400 python scripts/spai_time.py c5 --update > gpurun_out/spai_c5_w$w.json 2>&1; fi; cat gpurun_out/spai_c5_w$w.json; done
timeout 400 python scripts/c5_probe.py > gpurun_out/c5_probe_bins.json 2>&1; tail -c 1500 gpurun_out/c5_probe_bins.json
MPG_ROW_BINS=0 timeout 400 python scripts/c5_probe.py > gpurun_out/c5_probe_nobins.json 2>&1; tail -c 1500 gpurun_out/c5_probe_nobins.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step_r02b.csv python scripts/step_probe.py --reps 0 > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log | head -c 300; gzip -f gpurun_out/launches_step_r02b.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gs_tmxf --launch-skip 300 --launch-count 1 -o gpurun_out/tmxf300_r02 -f python scripts/step_probe.py --reps 0 > gpurun_out/ncu_tmxf300.log 2>&1; tail -2 gpurun_out/ncu_tmxf300.log | head -c 300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gs_tmxf --launch-skip 150 --launch-count 1 -o gpurun_out/tmxf150_r02 -f python scripts/step_probe.py --reps 0 > gpurun_out/ncu_tmxf150.log 2>&1; tail -2 gpurun_out/ncu_tmxf150.log | head -c 300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_sell8t --launch-skip 800 --launch-count 4 -o gpurun_out/sell8t_r02 -f python scripts/step_probe.py --reps 0 > gpurun_out/ncu_sell8t.log 2>&1; tail -2 gpurun_out/ncu_sell8t.log | head -c 300
ls -la gpurun_out
