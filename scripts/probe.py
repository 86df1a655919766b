"""Exploratory timing of the configs on one GPU (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen

def dev(h):
    return mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t = time.time()
if which == "c3":
    s = gen.config3(N or 106)
elif which == "c2":
    s = gen.config2(N or 64)
elif which == "c1":
    s = gen.config1(N or 100)
else:
    s = gen.config5(N or 2_000_000)
print("gen", time.time() - t, "n", s.n, "nnz", s.a.nnz, flush=True)
t = time.time()
A = dev(s.a); ec = s.e_csr(); E = dev(ec) if ec is not None else None
op = mpg.ShiftedOperator(A, E)
print("upload+op", time.time() - t, flush=True)
sig = float(s.shifts[0])
t = time.time(); M = op.explicit(sig); print("explicit", time.time() - t, M.nnz(), flush=True)
t = time.time(); sp = mpg.spai_build(M); print("spai", time.time() - t, sp.build_seconds, "nnzP", sp.p.nnz(), "fb", sp.fallback_count, "res mean", float(np.mean(sp.column_residuals)), flush=True)
ch = mpg.PrecondChain(sp.p)
b = s.b[:, 0]
for mi in (300, 1000):
    cfg = mpg.GmresConfig(1e-8, mi)
    t = time.time()
    r = mpg.gmres_shifted(op, sig, b, ch, False, cfg)
    print("gmres P", mi, r.report.iterations, r.report.converged, r.report.final_residual / r.report.rhs_norm, time.time() - t, flush=True)
    if r.report.converged: break
cfg = mpg.GmresConfig(1e-8, 1000)
sigs = list(s.shifts[:8])
t = time.time()
rs = mpg.gmres_batch(op, sigs, [b] * len(sigs), chains=[ch] * len(sigs), cfg=cfg)
el = time.time() - t
print("batch", len(sigs), [x.report.iterations for x in rs], [x.report.converged for x in rs], el, flush=True)
