(timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gputest_r.log 2>&1; tail -2 gpurun_out/gputest_r.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v3.json 2> gpurun_out/bench_ref_v3.err; tail -c 300 gpurun_out/bench_ref_v3.json
python bench.py --steps 8 --warmup 3 > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err; tail -c 200 gpurun_out/bench_v5.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 1 --warmup 1 > gpurun_out/ncu_bench.log 2>&1; gzip -f gpurun_out/launches_bench_r02.csv
