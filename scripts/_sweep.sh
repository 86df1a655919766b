timeout 900 python -m pytest tests/test_gpu_gmres.py -q -x 2>&1 | tail -2
timeout 300 python scripts/kprof.py 106 8 2>&1 | grep -E "graph|gs_"
timeout 1500 python scripts/irka_run.py c4 --max-iter 2000 2>&1 | tail -1
