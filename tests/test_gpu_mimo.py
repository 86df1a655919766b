"""MIMO tangential IRKA on the GPU path against the CPU oracle (config C4 type:
Q1 FEM with the consistent mass, B, C ~ N(0,1), m = q = 2..4, r = 8..16).

The tangential right-hand sides are B f2 and C c2 with f2 = fr^T R^{-T},
c2 = cr^T R (birka.cpp:182-183, :199). For SISO a wrong R-transform only
rescales each unit's right-hand side, so only m, q > 1 pins it.
North-star tolerances: converged shifts within 1e-6 relative, H_r(i w) on a
fixed 200-point log grid within 1e-6 relative (norm-wise per point)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRID = np.logspace(-4, 4, 200)


def _m(mpg, h):
    return mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)


def _hr_oracle(res, r):
    return [res.cr.T @ np.linalg.solve(1j * w * np.eye(r) - res.kr, res.fr) for w in GRID]


def _run(mpg, orc, N, m, r, mode, tol, max_sweeps):
    from paper_2003_12759_b200 import gen
    s = gen.config4(N)
    b, c = np.asfortranarray(s.b[:, :m]), np.asfortranarray(s.c[:, :m])
    shifts = np.logspace(-4, 1, r)
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e))
    cfg = mpg.IrkaConfig(r=r, tol=tol, max_sweeps=max_sweeps, seed=1, gmres=mpg.GmresConfig(1e-10, 1000))
    st, rep = mpg.irka_reduce(op, b, c, cfg, mode, init_shifts=shifts)
    # The fixed point does not depend on the preconditioner: the oracle runs
    # with its frozen SPAI (mode 3; its reference-faithful chain is slow here).
    ocfg = orc.IrkaConfig(r=r, tol=tol, max_sweeps=max_sweeps, seed=1, gmres=orc.GmresConfig(1e-10, 1000),
                          explicit_nnz_cap=10**12, decoupled=True)
    ores = orc.irka_reduce(orc.Csr.of(s.a), orc.Csr.of(s.e), b, c, ocfg, mode=3, init_shifts=shifts)
    return st, rep, ores


@pytest.mark.parametrize("N,m,r", [(8, 3, 8), (8, 4, 8), (10, 2, 16), (10, 3, 16)])
@pytest.mark.parametrize("mode", [2, 3])
def test_mimo_irka_converged_matches_oracle(mpg, orc, N, m, r, mode):
    st, rep, ores = _run(mpg, orc, N, m, r, mode, tol=1e-9, max_sweeps=150)
    assert ores.converged and rep.converged, (ores.sweeps, rep.sweeps)
    lg, lo = np.sort_complex(st.lam), np.sort_complex(ores.lam)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-6
    ho = _hr_oracle(ores, r)
    for w, h in zip(GRID, ho):
        hg = st.transfer(1j * w)
        assert hg.shape == (m, m)
        assert np.linalg.norm(hg - h) <= 1e-6 * np.linalg.norm(h), w


def test_mimo_irka_trajectory_matches_oracle_unconverged(mpg, orc):
    """N = 8, m = q = 4, r = 16 does not settle within 150 sweeps on the oracle
    either; the first 8 sweeps of the fixed-point map agree."""
    st, rep, ores = _run(mpg, orc, 8, 4, 16, 3, tol=1e-12, max_sweeps=8)
    assert rep.sweeps == ores.sweeps == 8
    lg, lo = np.sort_complex(st.lam), np.sort_complex(ores.lam)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-6
