"""Sharded (2 ranks on one GPU) vs single-rank IRKA on C1(40): sweeps and shift
difference (diagnostic for tests/test_dist.py)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

if __name__ == "__main__":
    import test_dist as T
    outs = T._spawn(T._irka_worker, 2)
    (_, lam0, sw0, conv0, rows0, ref), (_, lam1, sw1, conv1, rows1, _) = outs
    print("sharded sweeps", sw0, sw1, "ref sweeps", ref[1], "lam rel diff",
          np.max(np.abs(lam0 - ref[0]) / np.abs(ref[0])))
