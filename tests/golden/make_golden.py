"""Generates the golden fixtures of tests/golden/ with the CPU oracle (test
infrastructure; run here, committed, read by tests/test_gpu_golden.py on the
GPU box where the oracle's long runs would not fit the test budget).

c1_irka.json: BASELINE.json configs[0] at full size -- C1, 100 x 100 cells
(n = 10 000), r = 4, the reference's default preconditioner and reuse rule
(PatternOfA SPAI, ReuseChain, <= 16 factors), GMRES tol 1e-8, IRKA stop at a
relative shift change < 1e-6 or 50 sweeps; decoupled per-unit solves (the
GPU path's form). Stored: converged shifts, sweeps, H_r(i w) on
logspace(-4, 4, 200).
c1_solves.npz: three preconditioned shifted solves of C1 (sigma = 1e-2, 1, 1e1;
fresh SPAI of sigma E - A; tol 1e-10): solutions and iteration counts.

Usage: python tests/golden/make_golden.py   (about two minutes on one core)
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

if __name__ == "__main__":
    import oracle as O
    from paper_2003_12759_b200 import gen
    s = gen.config1()
    a, e = O.Csr.of(s.a), O.Csr.of(s.e_csr())
    t0 = time.time()
    cfg = O.IrkaConfig(r=4, tol=1e-6, max_sweeps=50, seed=1, gmres=O.GmresConfig(1e-8, 1000),
                       explicit_nnz_cap=10 ** 12, decoupled=True)
    res = O.irka_reduce(a, e, s.b, s.c, cfg, mode=2, init_shifts=s.shifts)
    grid = np.logspace(-4, 4, 200)
    hr = np.array([res.transfer(1j * w)[0, 0] for w in grid])
    lam = np.sort_complex(res.lam)
    out = {"config": "C1 N=100 (n=10000), r=4, ReuseChain SPAI, gmres tol 1e-8, irka tol 1e-6, decoupled",
           "converged": res.converged, "sweeps": res.sweeps,
           "shifts_re": [-float(z.real) for z in lam], "shifts_im": [-float(z.imag) for z in lam],
           "grid": grid.tolist(), "hr_re": hr.real.tolist(), "hr_im": hr.imag.tolist(),
           "oracle_seconds": round(time.time() - t0, 1)}
    with open(os.path.join(HERE, "c1_irka.json"), "w") as f:
        json.dump(out, f)
    xs, its = [], []
    for sigma in (1e-2, 1.0, 1e1):
        m = O.kron_assemble(O.shifted(sigma), a, e, cap=10 ** 12)
        x, rep = O.gmres_kron(O.shifted(sigma), a, e, O.Chain(O.spai_build(m)[0]), s.b[:, 0], O.GmresConfig(1e-10, 1000))
        xs.append(x)
        its.append(rep.iterations)
    np.savez_compressed(os.path.join(HERE, "c1_solves.npz"), sigma=np.array([1e-2, 1.0, 1e1]), x=np.array(xs),
                        iterations=np.array(its))
    print("done", out["sweeps"], out["converged"], its, out["oracle_seconds"])
