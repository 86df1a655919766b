"""Full IRKA on one of the BASELINE configs (IRKA wall time; not the bench).

python scripts/irka_run.py c3 [--nodes N] [--mode frozen|chain|fresh|none] [--tol 1e-6] [--max-sweeps 50]
Prints one JSON line: wall seconds, sweeps, converged shifts, solves, GMRES iterations.
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c1", "c2", "c3", "c4"])
ap.add_argument("--size", type=int, default=0)
ap.add_argument("--mode", default="")
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--gtol", type=float, default=1e-8)
ap.add_argument("--max-sweeps", type=int, default=50)
ap.add_argument("--max-iter", type=int, default=1000)
ap.add_argument("--mirror", type=int, default=-1)
a = ap.parse_args()
t0 = time.perf_counter()
sysm = {"c1": lambda: gen.config1(a.size or 100), "c2": lambda: gen.config2(a.size or 64),
        "c3": lambda: gen.config3(a.size or 106), "c4": lambda: gen.config4(a.size or 106)}[a.config]()
tgen = time.perf_counter() - t0
default_mode = {"c1": "chain"}.get(a.config, "frozen")
mode = {"frozen": mpg.PrecondMode.REUSE_FROZEN, "chain": mpg.PrecondMode.REUSE_CHAIN,
        "fresh": mpg.PrecondMode.FRESH_SPAI, "none": mpg.PrecondMode.NONE}[a.mode or default_mode]
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
ec = sysm.e_csr()
op = mpg.ShiftedOperator(dev(sysm.a), dev(ec) if ec is not None else None)
cfg = mpg.IrkaConfig(r=sysm.r, tol=a.tol, max_sweeps=a.max_sweeps, seed=1,
                     gmres=mpg.GmresConfig(a.gtol, a.max_iter),
                     mirror_unstable=(a.config != 'c1') if a.mirror < 0 else bool(a.mirror))
mpg.lib.mpg_synchronize(0)
t0 = time.perf_counter()
st, rep = mpg.irka_reduce(op, sysm.b, sysm.c, cfg, mode, init_shifts=sysm.shifts)
wall = time.perf_counter() - t0
tot = rep.totals()
print(json.dumps({"config": a.config, "n": int(sysm.n), "nnz": int(sysm.a.nnz), "r": int(sysm.r),
                  "mode": a.mode or default_mode, "irka_wall_s": round(wall, 3), "gen_s": round(tgen, 2),
                  "sweeps": rep.sweeps, "converged": rep.converged,
                  "shifts": sorted([float(-x.real) for x in st.lam]),
                  "shifts_im": [float(x.imag) for x in st.lam],
                  "solves": tot["solves"], "gmres_iterations": tot["gmres_iterations"],
                  "precond_build_s": round(tot["precond_build_seconds"], 3),
                  "max_its_per_solve": max(r.gmres_iterations for r in rep.rows),
                  "gmres_s_sum": round(sum(r.gmres_seconds for r in rep.rows), 3),
                  "solves_per_s": round(tot["solves"] / wall, 3)}), flush=True)
