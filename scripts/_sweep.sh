MPG_GS_CLUSTER_DOT=1 timeout 300 python scripts/kprof.py 106 8 2>&1 | grep -E "graph|gs_"
MPG_GS_CLUSTER_DOT=4 timeout 300 python scripts/kprof.py 106 8 2>&1 | grep -E "graph|gs_dot"
ncu --set full --import-source on --clock-control none -k regex:"k_gs_clu" --launch-skip 400 --launch-count 2 -o gpurun_out/gs_cm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-irka > gpurun_out/ncu_gscm.log 2>&1; tail -1 gpurun_out/ncu_gscm.log | cut -c1-50
