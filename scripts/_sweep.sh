for c in 2 4; do
echo "== upd cluster $c"
MPG_GS_CLUSTER_UPD=$c timeout 600 python -m pytest tests/test_gpu_gmres.py -q -x 2>&1 | tail -2
MPG_GS_CLUSTER_UPD=$c timeout 300 python scripts/kprof.py 106 8 2>&1 | grep -E "graph|gs_"
done
