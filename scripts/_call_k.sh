T="tests/test_golden_large.py::test_gpu_c2_irka_from_baseline_seed"
echo "== default"; timeout 300 python -m pytest "$T" -m gpu -q 2>&1 | tail -3
echo "== split 96"; MPG_GS_DOT_SPLIT=96 timeout 300 python -m pytest "$T" -m gpu -q 2>&1 | tail -3
echo "== no il pairs"; MPG_NO_IL_PAIRS=1 timeout 300 python -m pytest "$T" -m gpu -q 2>&1 | tail -3
echo "== no il pairs, split 96"; MPG_NO_IL_PAIRS=1 MPG_GS_DOT_SPLIT=96 timeout 300 python -m pytest "$T" -m gpu -q 2>&1 | tail -3
timeout 900 python scripts/irka_prof.py --sweeps 6 2>&1 | tail -1 | cut -c1-1500
(timeout 1500 python -m pytest tests -m gpu -q) > gpurun_out/gputest_k.log 2>&1; tail -6 gpurun_out/gputest_k.log
