"""Run-mode SpMV kernel classes on C3 (or --nodes N): one 16-solve step's worth
(8 primal + 8 dual solves sharing the frozen SPAI) capped at --its iterations,
per-class CUDA-event times from the engine's profiler. MPG_SPMV_CSR=1 forces the
CSR kernels; MPG_HALO_DEBUG=1 prints the halo layout statistics."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen

ap = argparse.ArgumentParser()
ap.add_argument("--nodes", type=int, default=106)
ap.add_argument("--its", type=int, default=60)
a = ap.parse_args()
s = gen.config3(a.nodes)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
sh = [float(x) for x in s.shifts[:8]]
pv = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], False)).p)
pw = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], True)).p)
sig, trs, ch = sh + sh, [0] * 8 + [1] * 8, [pv] * 8 + [pw] * 8
bs = [s.b[:, 0]] * 8 + [s.c[:, 0]] * 8
cfg = mpg.GmresConfig(1e-30, a.its)
mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
mpg.profile_enable(True)
mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
prof = mpg.profile_read()
mpg.profile_enable(False)
out = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
           "us_per_launch": round(1e3 * v["ms"] / max(v["launches"], 1), 1)} for k, v in prof.items() if v["launches"]}
print(json.dumps({"csr": bool(os.environ.get("MPG_SPMV_CSR")), "its": a.its, "kernels": out}))
