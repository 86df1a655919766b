"""Time coupled BIRKA variants on the bilinear toy (n=400, m=2, r=3) to split the per-sweep cost."""
import time
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen

if __name__ == "__main__":
    kh, nh, f, c = gen.bilinear_toy_n(400, 2, 4)
    dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val, 0)
    k, ns = dev(kh), [dev(x) for x in nh]
    for mode, srd, ms in [(2, 5000, 200), (2, 0, 200), (0, 0, 200), (2, 0, 1)]:
        cfg = mpg.IrkaConfig(r=3, tol=1e-9, max_sweeps=ms, seed=4, gmres=mpg.GmresConfig(1e-11, 1000),
                             explicit_nnz_cap=10**9, standard_residual_max_dim=srd)
        t0 = time.perf_counter()
        st, rep = mpg.birka_reduce(k, ns, f, c, cfg, mode)
        w = time.perf_counter() - t0
        tot = rep.totals()
        print(mode, srd, ms, round(w, 3), rep.sweeps, tot["gmres_iterations"], round(tot["gmres_seconds"], 3),
              round(tot["precond_build_seconds"], 3), flush=True)
