"""QB-IHOMM on the GPU path at C3 scale: D = the C3
consistent mass, K = the C3 operator A, N and H drawn by generate_qb_toy's
rules at the same n, F = the normalised x = 0 face indicator, C = the block
average. Prints wall time, solves, GMRES iterations and the report rows."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import paper_2003_12759_b200 as mpg
    from paper_2003_12759_b200 import gen
    nodes = int(sys.argv[1]) if len(sys.argv) > 1 else 106
    mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    sig = [float(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0.1, 0.2, 0.4, 0.8]
    s = gen.config3(nodes)
    toy = gen.qb_toy(s.n, 7)
    dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
    sys_ = mpg.QbSystem.create(dev(s.e), dev(s.a), dev(toy.n_op), toy.h, s.b[:, 0], s.c[:, 0])
    cfg = mpg.QbConfig(sigmas=sig, p_moments=1, q_moments=1, gmres=mpg.GmresConfig(1e-8, 1000))
    t0 = time.perf_counter()
    red, rep = mpg.qbihomm_reduce(sys_, cfg, mode)
    wall = time.perf_counter() - t0
    tot = rep.totals()
    out = {"n": s.n, "mode": mode, "sigmas": sig, "order": red.order(), "wall_s": round(wall, 3),
           "solves": tot["solves"], "gmres_iterations": tot["gmres_iterations"],
           "precond_build_s": round(tot["precond_build_seconds"], 3),
           "rows": [(r.sweep, r.point, r.kind, r.solves, r.gmres_iterations, round(r.precond_build_seconds, 3))
                    for r in rep.rows],
           "orth": float(np.linalg.norm(red.basis.T @ red.basis - np.eye(red.order())))}
    print(json.dumps(out))
