run() { echo "== $*"; env "$@" timeout 300 python scripts/kprof.py 106 8 2>&1 | grep -E "graph|spmv" ; }
run A=1
run MPG_L1MAX=1
run MPG_IL2=1
run MPG_IL2=1 MPG_L1MAX=1
MPG_IL2=1 timeout 600 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_irka.py -q -x 2>&1 | tail -2
