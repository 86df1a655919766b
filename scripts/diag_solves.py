"""Diagnostic: true residuals of a batch of shifted solves (real and pair units,
both sides) at a tight GMRES tolerance, on the BASELINE C2 or C3 pencil.
python scripts/diag_solves.py c2 [--gtol 1e-10]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c1", "c2", "c3"])
ap.add_argument("--gtol", type=float, default=1e-10)
ap.add_argument("--size", type=int, default=0)
a = ap.parse_args()
s = {"c1": lambda: gen.config1(a.size or 100), "c2": lambda: gen.config2(a.size or 64), "c3": lambda: gen.config3(a.size or 106)}[a.config]()
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
ec = s.e_csr()
op = mpg.ShiftedOperator(dev(s.a), dev(ec) if ec is not None else None)
n = s.n
rng = np.random.default_rng(5)
sig = [complex(x) for x in s.shifts[: s.r]]
# pair units spread over the spectrum of the converged C2 reduced model
sig += [6615.6 + 901.3j, 382.5 + 330.5j, 265.3 + 147.5j, 30280.9 + 0j, 244.46 + 0j, 2.3e5 + 0j]
chains = {}
for tr in (False, True):
    P = mpg.spai_build(op.explicit(sig[0], transpose=tr)).p
    chains[tr] = mpg.PrecondChain(P)
sigmas, bs, chs, trs = [], [], [], []
for tr in (False, True):
    col = (s.c if tr else s.b)[:, 0]
    for z in sig:
        b = np.concatenate([col, 0.37 * col]) if z.imag != 0 else col.copy()
        sigmas.append(z); bs.append(b); chs.append(chains[tr]); trs.append(tr)
cfg = mpg.GmresConfig(a.gtol, 1000)
for lo in range(0, len(sigmas), 8):
    hi = min(len(sigmas), lo + 8)
    res = mpg.gmres_batch(op, sigmas[lo:hi], bs[lo:hi], chs[lo:hi], trs[lo:hi], cfg)
    for i, r in enumerate(res):
        j = lo + i
        rt = bs[j] - op.apply(sigmas[j], r.x, transpose=trs[j])
        print(f"{str(sigmas[j]):>28} T={int(trs[j])} its={r.report.iterations:4d} conv={int(r.report.converged)} "
              f"reported={r.report.final_residual / r.report.rhs_norm:.3e} true={np.linalg.norm(rt) / np.linalg.norm(bs[j]):.3e}", flush=True)
