timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_irka.py -q -x 2>&1 | tail -2
timeout 300 python scripts/kprof.py 106 8 2>&1
