"""Per-kernel-class profile of the first sweeps of the C3 IRKA (tuning aid):
python scripts/irka_prof.py [--sweeps 6]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
ap = argparse.ArgumentParser()
ap.add_argument("--sweeps", type=int, default=6)
ap.add_argument("--nodes", type=int, default=106)
a = ap.parse_args()
s = gen.config3(a.nodes)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
cfg = mpg.IrkaConfig(r=s.r, tol=1e-6, max_sweeps=a.sweeps, seed=1, gmres=mpg.GmresConfig(1e-8, 1000), mirror_unstable=True)
mpg.lib.mpg_synchronize(0)
t0 = time.perf_counter()
st, rep = mpg.irka_reduce(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=s.shifts)
wall = time.perf_counter() - t0
mpg.profile_enable(True)
t0 = time.perf_counter()
st, rep = mpg.irka_reduce(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=s.shifts)
pw = time.perf_counter() - t0
prof = mpg.profile_read()
mpg.profile_enable(False)
tot = sum(v["ms"] for v in prof.values())
rows = rep.rows
print(json.dumps({"sweeps": rep.sweeps, "wall_s": round(wall, 2), "profiled_wall_s": round(pw, 2),
                  "lam": [[round(z.real, 3), round(z.imag, 3)] for z in st.lam],
                  "iters_by_sweep": {str(k): [r.gmres_iterations for r in rows if r.sweep == k] for k in sorted({r.sweep for r in rows})},
                  "kernels_ms": {k: [round(v["ms"], 1), round(v["ms"] / tot, 3)] for k, v in prof.items() if v["launches"]}}))
