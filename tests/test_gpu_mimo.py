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


# FROZEN (3) on every case; the vertical chain (2) where it stays a usable
# preconditioner (in the other cases a slot whose shift jumps to an unstable,
# unmirrored value gets an update factor too poor for GMRES to reach 1e-10).
@pytest.mark.parametrize("N,m,r,mode", [(8, 3, 8, 3), (8, 4, 8, 3), (10, 2, 16, 3), (10, 3, 16, 3), (8, 4, 8, 2)])
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


@pytest.mark.parametrize("N,r,lo,hi,sweeps", [(8, 16, 0.0, 3.0, 3), (10, 16, 0.0, 3.0, 3), (8, 8, -1.0, 2.0, 4)])
def test_mimo_irka_trajectory_matches_oracle(mpg, orc, gen, N, r, lo, hi, sweeps):
    """m = q = 4 with r = 16 does not settle within 150 sweeps on the oracle
    either (N = 8, 10), so the fixed-point map itself is compared: from
    well-separated initial shifts the first sweeps agree to 1e-9 (measured;
    the map is expansive, so later sweeps drift apart at rounding level x 10-100
    per sweep). From sweep 2 on, R is non-orthogonal, which pins the
    tangential directions f2 = fr^T R^{-T}, c2 = cr^T R (birka.cpp:182-183)."""
    s = gen.config4(N)
    shifts = np.logspace(lo, hi, r)
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e))
    cfg = mpg.IrkaConfig(r=r, tol=1e-14, max_sweeps=sweeps, seed=1, gmres=mpg.GmresConfig(1e-10, 1000))
    st, rep = mpg.irka_reduce(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=shifts)
    ocfg = orc.IrkaConfig(r=r, tol=1e-14, max_sweeps=sweeps, seed=1, gmres=orc.GmresConfig(1e-10, 1000),
                          explicit_nnz_cap=10**12, decoupled=True)
    ores = orc.irka_reduce(orc.Csr.of(s.a), orc.Csr.of(s.e), s.b, s.c, ocfg, mode=3, init_shifts=shifts)
    assert rep.sweeps == ores.sweeps == sweeps
    lg, lo_ = np.sort_complex(st.lam), np.sort_complex(ores.lam)
    assert np.max(np.abs(lg - lo_) / np.abs(lo_)) <= 1e-6
