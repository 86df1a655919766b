(timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gputest_final.log 2>&1; tail -2 gpurun_out/gputest_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 8 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 150 gpurun_out/bench_final.json
