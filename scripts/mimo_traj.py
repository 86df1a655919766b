"""Sweep-by-sweep divergence of GPU vs oracle MIMO IRKA (C4 type): N m r log10(lo) log10(hi)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as orc
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
N, m, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
lo_, hi_ = float(sys.argv[4]), float(sys.argv[5])
s = gen.config4(N)
b, c = np.asfortranarray(s.b[:, :m]), np.asfortranarray(s.c[:, :m])
sh = np.logspace(lo_, hi_, r)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
for k in range(1, 7):
    cfg = mpg.IrkaConfig(r=r, tol=1e-14, max_sweeps=k, seed=1, gmres=mpg.GmresConfig(1e-10, 1000))
    st, rep = mpg.irka_reduce(op, b, c, cfg, 3, init_shifts=sh)
    ocfg = orc.IrkaConfig(r=r, tol=1e-14, max_sweeps=k, seed=1, gmres=orc.GmresConfig(1e-10, 1000),
                          explicit_nnz_cap=10**12, decoupled=True)
    o = orc.irka_reduce(orc.Csr.of(s.a), orc.Csr.of(s.e), b, c, ocfg, mode=3, init_shifts=sh)
    lg, lo = np.sort_complex(st.lam), np.sort_complex(o.lam)
    print(k, np.max(np.abs(lg - lo) / np.abs(lo)), lo[-3:], lg[-3:], flush=True)
