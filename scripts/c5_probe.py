"""C5 kernel probe (tuning / evidence aid, not the bench): the Zipf-row matrix,
one fresh SPAI at a mid-range shift, then one preconditioned solve with the
per-kernel-class profile (event-bracketed launches). MPG_ROW_BINS=0 gives the fixed-width kernels.

python scripts/c5_probe.py [--n 2000000] [--sigma 1.0] [--reps 50]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--max-len", type=int, default=2000)
ap.add_argument("--sigma", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--no-solve", action="store_true")
a = ap.parse_args()
s = gen.config5(a.n, max_len=a.max_len)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
A = dev(s.a)
op = mpg.ShiftedOperator(A, dev(s.e_csr()))
n, nnz = int(s.n), int(s.a.nnz)
rl = np.diff(s.a.rowptr)
out = {"config": "c5", "n": n, "nnz": nnz, "row_len_max": int(rl.max()), "row_len_mean": float(rl.mean()),
       "row_bins": os.environ.get("MPG_ROW_BINS", "auto"),
       "rows_by_bin": [int(((rl > lo) & (rl <= hi)).sum()) for lo, hi in ((0, 5), (5, 32), (32, 64), (64, 128), (128, 1 << 30))],
       "nnz_by_bin": [int(rl[(rl > lo) & (rl <= hi)].sum()) for lo, hi in ((0, 5), (5, 32), (32, 64), (64, 128), (128, 1 << 30))]}
t0 = time.perf_counter()
P = mpg.spai_build(op.explicit(a.sigma))
mpg.lib.mpg_synchronize(0)
out["spai_build_s"] = round(time.perf_counter() - t0, 3)
out["spai_nnz"] = int(P.p.nnz())
if not a.no_solve:
    chain = mpg.PrecondChain(P.p)
    cfg = mpg.GmresConfig(1e-8, 1000)
    b = s.b[:, 0]
    mpg.gmres_batch(op, [a.sigma], [b], chains=[chain], cfg=cfg)
    t0 = time.perf_counter()
    res = mpg.gmres_batch(op, [a.sigma], [b], chains=[chain], cfg=cfg)
    out["solve_s"] = round(time.perf_counter() - t0, 4)
    out["iterations"] = res[0].report.iterations
    mpg.profile_enable(True)
    mpg.gmres_batch(op, [a.sigma], [b], chains=[chain], cfg=cfg)
    prof = mpg.profile_read()
    mpg.profile_enable(False)
    tot = sum(v["ms"] for v in prof.values())
    out["profile"] = {k: {"launches": v["launches"], "ms": round(v["ms"], 2), "share": round(v["ms"] / tot, 4),
                          "us_per_launch": round(1e3 * v["ms"] / v["launches"], 1),
                          "GBps": round(v["bytes"] / v["ms"] / 1e6, 1) if v["ms"] > 0 and v["bytes"] > 0 else None}
                      for k, v in prof.items() if v["launches"]}
    # algorithmic bytes of one operator / one chain SpMV (12 B per entry + row pointers + vectors)
    it = max(1, out["iterations"])
    for k, nz in (("shifted_spmv", nnz), ("chain_spmv", out["spai_nnz"] or nnz)):
        if k in out["profile"]:
            byts = 12.0 * nz + 4.0 * (n + 1) + 24.0 * n
            us = out["profile"][k]["us_per_launch"]
            out["profile"][k]["spmv_algorithmic_GBps"] = round(byts / us / 1e3, 1)
print(json.dumps(out), flush=True)
