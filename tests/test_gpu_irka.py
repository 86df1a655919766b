"""GPU IRKA parity (north-star tolerances): converged shifts within 1e-6
relative and H_r(i w) on a fixed 200-point log grid within 1e-6 relative of
the CPU oracle on the same seeded inputs; plus the reference's oracle-free
checks (interpolation, projection identities; test_birka.cpp:51-132)."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

GRID = np.logspace(-4, 4, 200)


def _m(mpg, h):
    return mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)


def _hr_grid(state):
    return np.array([state.transfer(1j * w) for w in GRID])


def _run_both(mpg, orc, sysm, r, mode, tol=1e-8, gtol=1e-10, max_sweeps=60):
    ecsr = sysm.e_csr()
    op = mpg.ShiftedOperator(_m(mpg, sysm.a), _m(mpg, ecsr) if ecsr is not None else None)
    cfg = mpg.IrkaConfig(r=r, tol=tol, max_sweeps=max_sweeps, seed=1, gmres=mpg.GmresConfig(gtol, 1000))
    st, rep = mpg.irka_reduce(op, sysm.b, sysm.c, cfg, mode, init_shifts=sysm.shifts[:r], want_bases=True)
    ocfg = orc.IrkaConfig(r=r, tol=tol, max_sweeps=max_sweeps, seed=1, gmres=orc.GmresConfig(gtol, 1000),
                          explicit_nnz_cap=10**12, decoupled=True)
    ores = orc.irka_reduce(orc.Csr.of(sysm.a), orc.Csr.of(ecsr) if ecsr is not None else None, sysm.b, sysm.c, ocfg,
                           mode=min(mode, 2), init_shifts=sysm.shifts[:r])
    return op, st, rep, ores


@pytest.mark.parametrize("mode", [0, 2, 3])
def test_irka_config1_small_matches_oracle(mpg, orc, gen, mode):
    sysm = gen.config1(N=16)
    op, st, rep, ores = _run_both(mpg, orc, sysm, 4, mode)
    assert rep.converged and ores.converged
    lam, lamo = np.sort_complex(st.lam), np.sort_complex(ores.lam)
    assert rel(lam, lamo) <= 1e-6
    hg, ho = _hr_grid(st), _hr_grid(ores)
    assert np.max(np.abs(hg - ho) / np.maximum(np.abs(ho), 1e-300)) <= 1e-6


def test_irka_interpolates_at_converged_shifts(mpg, orc, gen):
    sysm = gen.config1(N=12)
    op, st, rep, _ = _run_both(mpg, orc, sysm, 4, 2, tol=1e-12, gtol=1e-13, max_sweeps=200)
    assert rep.converged
    a = sysm.a.to_dense()
    e = np.diag(sysm.e_diag)
    for lam in st.lam:
        s = -lam
        h = sysm.c[:, 0] @ np.linalg.solve(s * e - a, sysm.b[:, 0])
        # H_r(s) = c_r^T (s I - K_r)^{-1} f_r with K_r = E_r^{-1} A_r
        assert abs(h - st.transfer(s)[0, 0]) <= 1e-7 * abs(h)


def test_irka_projection_identities(mpg, orc, gen):
    sysm = gen.config1(N=12)
    op, st, rep, _ = _run_both(mpg, orc, sysm, 4, 2)
    v, w = st.v, st.w
    assert np.linalg.norm(v.T @ v - np.eye(4)) <= 1e-12
    assert np.linalg.norm(w.T @ w - np.eye(4)) <= 1e-12
    a = sysm.a.to_dense()
    e = np.diag(sysm.e_diag)
    er = w.T @ e @ v
    assert np.linalg.norm(np.linalg.solve(er, w.T @ a @ v) - st.kr) <= 1e-10 * (1 + np.linalg.norm(st.kr))
    assert np.linalg.norm(np.linalg.solve(er, w.T @ sysm.b) - st.fr) <= 1e-10 * (1 + np.linalg.norm(st.fr))
    assert np.linalg.norm(v.T @ sysm.c - st.cr) <= 1e-10 * (1 + np.linalg.norm(st.cr))


def test_reuse_report_layout(mpg, orc, gen):
    sysm = gen.config1(N=12)
    op, st, rep, _ = _run_both(mpg, orc, sysm, 4, 2, tol=1e-4)
    assert rep.converged and rep.sweeps >= 2
    assert all(r.solves == 1 and r.point in (1, 2) for r in rep.rows)
    assert len(rep.rows) == 2 * 4 * rep.sweeps  # one row per (sweep, side, real unit)
    for r in rep.rows:
        # fresh at sweep 1, vertical updates until the chain would exceed
        # max_chain_len = 16, then fresh again (birka.cpp:233-251)
        want = "fresh" if (r.sweep - 1) % 17 == 0 else "vertical"
        assert r.kind == want, (r.sweep, r.kind)
        if r.kind == "vertical":
            assert r.min_residual <= r.matrix_change


def test_irka_identity_mass_matches_reference_loop(mpg, orc, gen):
    # E = I: the toy bilinear model with N = 0 (test_birka.cpp:51-75), default seed
    k, f, c = gen.bilinear_toy(8, 1, 5)
    op = mpg.ShiftedOperator(_m(mpg, k))
    cfg = mpg.IrkaConfig(r=2, tol=1e-12, max_sweeps=200, seed=5, gmres=mpg.GmresConfig(1e-13, 1000))
    st, rep = mpg.irka_reduce(op, f, c, cfg, mpg.PrecondMode.NONE)
    ores = orc.irka_reduce(orc.Csr.of(k), None, f, c, orc.IrkaConfig(r=2, tol=1e-12, max_sweeps=200, seed=5,
                                                                       gmres=orc.GmresConfig(1e-13, 1000)), mode=0)
    assert rep.converged and ores.converged
    assert rel(np.sort_complex(st.lam), np.sort_complex(ores.lam)) <= 1e-8
    kd = k.to_dense()
    for lam in st.lam:
        s = -lam
        h = c[:, 0] @ np.linalg.solve(s * np.eye(8) - kd, f[:, 0])
        assert abs(h - st.transfer(s)[0, 0]) <= 1e-8 * abs(h)


def test_spai_bench_rows_and_parity(mpg, orc, gen):
    sysm = gen.config1(N=16)
    op = mpg.ShiftedOperator(_m(mpg, sysm.a), _m(mpg, sysm.e_csr()))
    pts = [6.28, 80.0, 300.0]
    g = mpg.GmresConfig(1e-8, 500)
    res = mpg.run_spai_bench(op, sysm.b[:, 0], pts, gmres=g, keep_solutions=True)
    assert res.failed_solves == 0
    assert [r.kind for r in res.report.rows] == ["fresh", "horizontal", "horizontal"]
    rows, failed, xo = orc.spai_bench(orc.Csr.of(sysm.a), orc.Csr.of(sysm.e_csr()), sysm.b[:, 0], pts,
                                      gmres=orc.GmresConfig(1e-8, 500), keep_solutions=True)
    assert failed == 0
    for i in range(3):
        assert rel(res.x[i], xo[i]) <= 1e-6
    bad = mpg.run_spai_bench(op, sysm.b[:, 0], pts, gmres=mpg.GmresConfig(1e-6, 3), mode=mpg.PrecondMode.NONE)
    assert bad.failed_solves == 3 and not bad.report.converged


def test_spai_bench_zipf_rows_match_oracle(mpg, orc, gen):
    """C5-type matrix (Zipf(1.8) row lengths up to 300, diagonal E): the shift
    sweep's SPAI / horizontal updates, solves and failure accounting match the
    oracle (long rows exercise the SpMV and SPAI load imbalance)."""
    s = gen.config5(n=3000, nshifts=6, max_len=300)
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e_csr()))
    pts = [float(x) for x in s.shifts]
    g = mpg.GmresConfig(1e-8, 1000)
    res = mpg.run_spai_bench(op, s.b[:, 0], pts, gmres=g, keep_solutions=True)
    rows, failed, xo = orc.spai_bench(orc.Csr.of(s.a), orc.Csr.of(s.e_csr()), s.b[:, 0], pts,
                                      gmres=orc.GmresConfig(1e-8, 1000), keep_solutions=True)
    assert res.failed_solves == failed
    assert [r.kind for r in res.report.rows] == [
        {1: "fresh", 2: "horizontal", 3: "vertical", 4: "reused_same_matrix"}.get(r.kind, "none") for r in rows]
    for i, r in enumerate(rows):
        assert abs(res.report.rows[i].gmres_iterations - r.iterations) <= max(3, 0.05 * r.iterations)
        if r.kind != 1:
            assert abs(res.report.rows[i].min_residual - r.min_residual) <= 1e-8 * max(1.0, r.min_residual)
            assert abs(res.report.rows[i].matrix_change - r.matrix_change) <= 1e-10 * r.matrix_change
        if res.report.rows[i].gmres_iterations < 1000:
            assert rel(res.x[i], xo[i]) <= 1e-6


def test_irka_consistent_mass_small_matches_oracle(mpg, orc, gen):
    """C3-type system (Q1 FEM, E = consistent mass sharing A's pattern) at 8^3
    nodes, FROZEN reuse with unstable shifts mirrored: shifts within 1e-6 and
    H_r(i w) within 1e-6 of the oracle."""
    s = gen.config3(8)
    r = 4
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e))
    cfg = mpg.IrkaConfig(r=r, tol=1e-8, max_sweeps=60, seed=1, gmres=mpg.GmresConfig(1e-11, 1000),
                         mirror_unstable=True)
    st, rep = mpg.irka_reduce(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=s.shifts[:r])
    ocfg = orc.IrkaConfig(r=r, tol=1e-8, max_sweeps=60, seed=1, gmres=orc.GmresConfig(1e-11, 1000),
                          explicit_nnz_cap=10**12, decoupled=True, mirror_unstable=True)
    ores = orc.irka_reduce(orc.Csr.of(s.a), orc.Csr.of(s.e), s.b, s.c, ocfg, mode=2, init_shifts=s.shifts[:r])
    assert rep.converged and ores.converged
    lg, lo = np.sort_complex(st.lam), np.sort_complex(ores.lam)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-6
    ho = np.array([ores.cr.T @ np.linalg.solve(1j * w * np.eye(r) - ores.kr, ores.fr) for w in GRID])
    assert np.max(np.abs(_hr_grid(st) - ho) / np.abs(ho)) <= 1e-6


def test_projection_entry_matches_dense(mpg, gen):
    """mpg_project (birka.cpp:283-291, E-generalised) against W^T E V, W^T A V."""
    s = gen.config1(N=30)
    ec = s.e_csr()
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, ec))
    rng = np.random.default_rng(3)
    V = rng.standard_normal((s.n, 5))
    W = rng.standard_normal((s.n, 5))
    er, ar = mpg.project(op, V, W)
    assert rel(er, W.T @ (ec.to_scipy() @ V)) <= 1e-13
    assert rel(ar, W.T @ (s.a.to_scipy() @ V)) <= 1e-13
