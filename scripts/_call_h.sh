for sp in 64 48 32; do MPG_GS_DOT_SPLIT=$sp timeout 600 python scripts/step_probe.py --reps 2 2>&1 | tail -1 | cut -c1-700; done
python bench.py --steps 8 --warmup 3 > gpurun_out/bench_v3.json 2> gpurun_out/bench_v3.err; tail -c 600 gpurun_out/bench_v3.json
