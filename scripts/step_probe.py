"""One bench step (C3: 8 shifts x primal + dual = 16 solves to 1e-8 with the
frozen SPAI) timed twice: once with CUDA events around the whole step, once
profiled per kernel class. Env knobs of the engine (MPG_DCGS2, MPG_GS_DOT_SPLIT,
MPG_SPMV_HALO, ...) select the variants being compared."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ctypes as C
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen, _lib as L

ap = argparse.ArgumentParser()
ap.add_argument("--nodes", type=int, default=106)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
s = gen.config3(a.nodes)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
sh = [float(x) for x in s.shifts[:8]]
pv = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], False)).p)
pw = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], True)).p)
sig, trs, ch = sh + sh, [0] * 8 + [1] * 8, [pv] * 8 + [pw] * 8
bs = [torch.from_numpy(np.ascontiguousarray(s.b[:, 0])).cuda()] * 8 + [torch.from_numpy(np.ascontiguousarray(s.c[:, 0])).cuda()] * 8
cfg = mpg.GmresConfig(1e-8, 1000)
res = mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
sp = C.c_void_p()
L.check(L.lib.mpg_stream(0, C.byref(sp)))
stream = torch.cuda.ExternalStream(sp.value, device="cuda:0")
ms = []
for _ in range(a.reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
    e1.record(stream)
    e1.synchronize()
    ms.append(e0.elapsed_time(e1))
mpg.profile_enable(True)
mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
prof = mpg.profile_read()
mpg.profile_enable(False)
its = [r.report.iterations for r in res]
worst = max(r.report.final_residual / r.report.rhs_norm for r in res)
env = {k: v for k, v in os.environ.items() if k.startswith("MPG_")}
print(json.dumps({"env": env, "step_ms": [round(x, 1) for x in ms], "iterations": its, "max_rel_res": worst,
                  "all_converged": all(r.report.converged for r in res),
                  "kernels_ms": {k: round(v["ms"], 1) for k, v in prof.items() if v["launches"]}}))
