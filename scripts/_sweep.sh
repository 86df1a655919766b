timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -3
timeout 300 python scripts/kprof.py 106 8 2>&1
timeout 300 python scripts/kprof.py 106 16 2>&1 | head -7
MPG_GS_CLUSTER_DOT=4 timeout 300 python scripts/kprof.py 106 8 2>&1 | grep -E "gs_dot|graph"
