"""C4's MIMO tangential IRKA (m = q = 4, r = 16, the C4 initial shifts) on the CPU
oracle at reduced sizes (8^3, 10^3 nodes): does the fixed-point iteration settle?
Writes profiles/r02/c4_oracle_nonconvergence.json (the evidence that the
non-convergence seen at full size on the GPU is a property of the iteration)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle as orc
from oracle import gen

out = []
for N in (8, 10):
    s = gen.config4(N)
    for mirror in (False, True):
        t0 = time.time()
        cfg = orc.IrkaConfig(r=16, tol=1e-6, max_sweeps=150, seed=1, gmres=orc.GmresConfig(1e-10, 1000),
                             explicit_nnz_cap=10 ** 12, decoupled=True, mirror_unstable=mirror)
        try:
            r = orc.irka_reduce(orc.Csr.of(s.a), orc.Csr.of(s.e), s.b, s.c, cfg, mode=3, init_shifts=s.shifts[:16])
            rec = {"nodes": N, "n": int(s.n), "mirror_unstable": mirror, "sweeps": r.sweeps, "converged": r.converged,
                   "final_shifts": sorted([[float(-z.real), float(-z.imag)] for z in r.lam])}
        except Exception as e:
            rec = {"nodes": N, "n": int(s.n), "mirror_unstable": mirror, "error": str(e)}
        rec["oracle_s"] = round(time.time() - t0, 1)
        print(json.dumps(rec), flush=True)
        out.append(rec)
json.dump({"config": "C4 type: Q1 FEM + consistent mass, B, C ~ N(0,1) seed 3, m = q = 4, r = 16, init shifts "
                     "logspace(1e-4, 1e1, 16), FROZEN SPAI (oracle mode 3), GMRES 1e-10, IRKA tol 1e-6, 150 sweeps",
           "runs": out}, open(os.path.join(ROOT, "profiles", "r02", "c4_oracle_nonconvergence.json"), "w"), indent=1)
