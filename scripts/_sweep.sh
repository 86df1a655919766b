for w in 16 24 28; do MPG_SPAI_WPS=$w timeout 300 python scripts/spai_prof.py 106 2>&1 | tail -1; done
