import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
import oracle as O
N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
s = gen.config3(N)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
sig = float(s.shifts[0])
P = mpg.spai_build(op.explicit(sig)).p
r = mpg.gmres_shifted(op, sig, s.b[:, 0], mpg.PrecondChain(P), cfg=mpg.GmresConfig(1e-8, 1000))
print("gpu its", r.report.iterations, "reorth", r.report.reorth_passes, flush=True)
Ao, Eo = O.Csr.of(s.a), O.Csr.of(s.e)
Mo = O.kron_assemble(O.shifted(sig), Ao, Eo, cap=10**12)
Po = O.spai_build(Mo, O.SpaiConfig(threads=8))[0]
t = time.time()
x, ro = O.gmres_kron(O.shifted(sig), Ao, Eo, O.Chain(Po), s.b[:, 0], O.GmresConfig(1e-8, 1000))
print("oracle its", ro.iterations, "reorth", ro.reorth_passes, "rel x diff", np.linalg.norm(x - r.x) / np.linalg.norm(x), time.time() - t, flush=True)
