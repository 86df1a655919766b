"""SPAI build time on one config (tuning aid): python scripts/spai_time.py c3|c5 [--n N] [--update]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c3", "c5"])
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--update", action="store_true")
a = ap.parse_args()
s = gen.config3(a.n or 106) if a.config == "c3" else gen.config5(a.n or 2_000_000, max_len=2000)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
ec = s.e_csr() if a.config == "c5" else s.e
op = mpg.ShiftedOperator(dev(s.a), dev(ec))
sig = [1.0, 1.2] if a.config == "c5" else [float(s.shifts[0]), float(s.shifts[1])]
m0 = op.explicit(sig[0])
mpg.lib.mpg_synchronize(0)
out = {"config": a.config, "n": int(s.n), "env": {k: v for k, v in os.environ.items() if k.startswith("MPG_")}}
t0 = time.perf_counter(); P = mpg.spai_build(m0); mpg.lib.mpg_synchronize(0)
out["spai_build_s"] = round(time.perf_counter() - t0, 3)
out["fallbacks"] = P.fallback_count
out["nnz_P"] = int(P.p.nnz())
if a.update:
    m1 = op.explicit(sig[1])
    t0 = time.perf_counter(); Q = mpg.update_build(m0, m1); mpg.lib.mpg_synchronize(0)
    out["update_build_s"] = round(time.perf_counter() - t0, 3)
    out["min_residual"] = Q.min_residual
print(json.dumps(out), flush=True)
