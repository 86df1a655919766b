"""C5 load-imbalance sweep (BASELINE.json configs[4]): 64 log-spaced shifts in
[1e-3, 1e3] on the n = 2M Zipf matrix, each solve to 1e-8 (run_spai_bench,
bench.cpp:159-249). Prints one JSON line (tuning / reporting aid, not the bench).

python scripts/c5_run.py [--n 2000000] [--mode frozen|chain|fresh|none] [--shifts 64]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--max-len", type=int, default=2000)
ap.add_argument("--mode", default="frozen")
ap.add_argument("--shifts", type=int, default=64)
ap.add_argument("--tol", type=float, default=1e-8)
a = ap.parse_args()
t0 = time.perf_counter()
s = gen.config5(a.n, nshifts=a.shifts, max_len=a.max_len)
tgen = time.perf_counter() - t0
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
ec = s.e_csr()
op = mpg.ShiftedOperator(dev(s.a), dev(ec) if ec is not None else None)
mode = {"frozen": mpg.PrecondMode.REUSE_FROZEN, "chain": mpg.PrecondMode.REUSE_CHAIN,
        "fresh": mpg.PrecondMode.FRESH_SPAI, "none": mpg.PrecondMode.NONE}[a.mode]
pts = [float(x) for x in s.shifts]
b = s.b[:, 0]
mpg.lib.mpg_synchronize(0)
t0 = time.perf_counter()
res = mpg.run_spai_bench(op, b, pts, gmres=mpg.GmresConfig(a.tol, 1000), mode=mode)
wall = time.perf_counter() - t0
rows = res.report.rows
rl = np.diff(s.a.rowptr)
print(json.dumps({"config": "c5", "n": int(s.n), "nnz": int(s.a.nnz), "row_len_max": int(rl.max()),
                  "row_len_mean": float(rl.mean()), "mode": a.mode, "shifts": len(pts), "wall_s": round(wall, 3),
                  "gen_s": round(tgen, 2), "failed": res.failed_solves,
                  "solves_per_s": round(len(pts) / wall, 3),
                  "build_s": round(sum(r.precond_build_seconds for r in rows), 3),
                  "gmres_s": round(sum(r.gmres_seconds for r in rows), 3),
                  "iterations": [r.gmres_iterations for r in rows]}), flush=True)
