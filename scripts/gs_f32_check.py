"""A/B of the float-shadow projection pass (MPG_GS_F32) on C3 solves: iterations, true residuals,
difference of the solutions, wall time. python scripts/gs_f32_check.py [--tol 1e-8] [--nodes 106]"""
import argparse, json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--nodes", type=int, default=106)
ap.add_argument("--child", default="")
a = ap.parse_args()
if not a.child:
    outs = {}
    for mode in ("0", "1"):
        env = dict(os.environ, MPG_GS_F32=mode)
        path = f"/tmp/gsf32_{mode}.npz"
        subprocess.run([sys.executable, __file__, "--tol", str(a.tol), "--nodes", str(a.nodes), "--child", path], env=env, check=True)
        outs[mode] = np.load(path)
    x0, x1 = outs["0"]["x"], outs["1"]["x"]
    print("iterations fp64:", outs["0"]["its"].tolist())
    print("iterations f32 :", outs["1"]["its"].tolist())
    print("true rel residual fp64 max:", float(outs["0"]["res"].max()), " f32 max:", float(outs["1"]["res"].max()))
    print("max rel diff of x:", float(max(np.linalg.norm(x0[i] - x1[i]) / np.linalg.norm(x0[i]) for i in range(x0.shape[0]))))
    print("reorth passes fp64:", outs["0"]["ro"].tolist(), " f32:", outs["1"]["ro"].tolist())
    print("seconds fp64: %.3f  f32: %.3f" % (float(outs["0"]["t"]), float(outs["1"]["t"])))
    sys.exit(0)
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
s = gen.config3(a.nodes)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
sig = [complex(x) for x in s.shifts[:8]]
P = {tr: mpg.PrecondChain(mpg.spai_build(op.explicit(sig[0], transpose=tr)).p) for tr in (False, True)}
sigmas = sig + sig
trs = [False] * 8 + [True] * 8
bs = [s.b[:, 0]] * 8 + [s.c[:, 0]] * 8
chs = [P[t] for t in trs]
cfg = mpg.GmresConfig(a.tol, 1000)
mpg.gmres_batch(op, sigmas[:2], bs[:2], chs[:2], trs[:2], mpg.GmresConfig(1e-2, 50))  # warm-up
mpg.lib.mpg_synchronize(0)
t0 = time.perf_counter()
res = mpg.gmres_batch(op, sigmas, bs, chs, trs, cfg)
mpg.lib.mpg_synchronize(0)
t = time.perf_counter() - t0
rr = [np.linalg.norm(bs[i] - op.apply(sigmas[i], res[i].x, transpose=trs[i])) / np.linalg.norm(bs[i]) for i in range(16)]
np.savez(a.child, x=np.array([r.x for r in res]), its=np.array([r.report.iterations for r in res]), res=np.array(rr),
         ro=np.array([getattr(r.report, "reorth_passes", -1) for r in res]), t=t)
