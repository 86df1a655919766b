"""C3-type system (E = consistent mass) in REUSE_CHAIN mode: GPU vs oracle at
a small grid, sweep by sweep iteration counts (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
import oracle as orc
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s = gen.config3(N)
cfg = mpg.IrkaConfig(r=s.r, tol=1e-6, max_sweeps=12, seed=1, gmres=mpg.GmresConfig(1e-8, 1000), mirror_unstable=True)
t = time.perf_counter()
try:
    dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
    op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
    st, rep = mpg.irka_reduce(op, s.b, s.c, cfg, mode, init_shifts=s.shifts)
    print("gpu", rep.sweeps, rep.converged, f"{time.perf_counter()-t:.2f}s")
    for r in rep.rows: print("  gpu", r.sweep, r.point, r.kind, r.gmres_iterations, f"{r.min_residual:.3e}", f"{r.matrix_change:.3e}")
except Exception as e:
    print("gpu failed:", e)
oc = orc.IrkaConfig(r=s.r, tol=1e-6, max_sweeps=12, seed=1, gmres=orc.GmresConfig(1e-8, 1000, False), decoupled=True,
                    mirror_unstable=True, explicit_nnz_cap=10**12)
t = time.perf_counter()
try:
    res = orc.irka_reduce(orc.Csr.of(s.a), orc.Csr.of(s.e), s.b, s.c, oc, mode, init_shifts=s.shifts)
    print("oracle", res.sweeps, res.converged, f"{time.perf_counter()-t:.2f}s")
    for r in res.rows: print("  orc", r.sweep, r.point, r.kind, r.iterations, f"{r.min_residual:.3e}", f"{r.matrix_change:.3e}")
except Exception as e:
    print("oracle failed:", e)
