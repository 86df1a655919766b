"""C5 grouped-solve probe (tuning aid): 8 shifts sharing one frozen SPAI in one gmres_batch (the FROZEN sweep's
unit of work), per-kernel-class profile. python scripts/c5_group_probe.py [--n 2000000] [--lo 0.05 --hi 5]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--lo", type=float, default=0.05)
ap.add_argument("--hi", type=float, default=5.0)
a = ap.parse_args()
s = gen.config5(a.n, max_len=2000)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e_csr()))
sig = [float(x) for x in np.logspace(np.log10(a.lo), np.log10(a.hi), 8)]
P = mpg.PrecondChain(mpg.spai_build(op.explicit(sig[0])).p)
cfg = mpg.GmresConfig(1e-8, 1000)
bs = [s.b[:, 0]] * 8
mpg.gmres_batch(op, sig, bs, chains=[P] * 8, cfg=cfg)
mpg.profile_enable(True)
res = mpg.gmres_batch(op, sig, bs, chains=[P] * 8, cfg=cfg)
prof = mpg.profile_read()
mpg.profile_enable(False)
tot = sum(v["ms"] for v in prof.values())
print(json.dumps({"n": int(s.n), "its": [r.report.iterations for r in res], "total_ms": round(tot, 1),
                  "kernels": {k: [v["launches"], round(v["ms"], 1), round(v["ms"] / tot, 3)] for k, v in prof.items() if v["launches"]}}))
