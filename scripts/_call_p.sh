(timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gputest_p.log 2>&1; tail -3 gpurun_out/gputest_p.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py --steps 8 --warmup 3 > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err; tail -c 300 gpurun_out/bench_v4.json
