"""GPU BIRKA with couplings N_j != 0 (birka.cpp:139-310,
kron.cpp:72-131) against the oracle's coupled BIRKA on the same seeded
bilinear toys (generator.cpp:141-179): converged reduced poles within 1e-6
relative, basis-invariant reduced transfer functions (linear and the
second-order Volterra kernel through N_r) within 1e-6, and the reference's
own oracle-free checks (test_birka.cpp:77-187)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _m(mpg, h):
    return mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)


def _kernels(kr, nr, fr, cr, pts):
    """H1(s) = c^T (s-K)^-1 F and H2_j(s1, s2) = c^T (s2-K)^-1 N_j (s1-K)^-1 F: invariant under the basis
    change the two implementations' orthonormalisations may differ by."""
    r = kr.shape[0]
    out = []
    for s in pts:
        r1 = np.linalg.solve(s * np.eye(r) - kr, fr)
        out.append((cr.T @ r1).ravel())
        for nj in nr:
            out.append((cr.T @ np.linalg.solve((s + 0.5j) * np.eye(r) - kr, nj @ r1)).ravel())
    return np.concatenate(out)


def _both(mpg, orc, gen, n, m, seed, r, mode, cap=10**9):
    kh, nh, f, c = gen.bilinear_toy_n(n, m, seed)
    cfg = mpg.IrkaConfig(r=r, tol=1e-9, max_sweeps=200, seed=seed, gmres=mpg.GmresConfig(1e-11, 1000),
                         explicit_nnz_cap=cap)
    st, rep = mpg.birka_reduce(_m(mpg, kh), [_m(mpg, x) for x in nh], f, c, cfg, mode, want_bases=True)
    ocfg = orc.IrkaConfig(r=r, tol=1e-9, max_sweeps=200, seed=seed, gmres=orc.GmresConfig(1e-11, 1000),
                          explicit_nnz_cap=cap)
    ores = orc.birka_reduce(orc.Csr.of(kh), [orc.Csr.of(x) for x in nh], f, c, ocfg, mode=min(mode, 2))
    return kh, nh, f, c, st, rep, ores


@pytest.mark.parametrize("n,m,seed,r,mode", [(6, 1, 1, 2, 2), (8, 2, 2, 2, 2), (12, 2, 5, 3, 1), (40, 1, 7, 3, 0),
                                             (60, 3, 9, 3, 2), (200, 1, 3, 3, 2)])
def test_coupled_birka_matches_oracle(mpg, orc, gen, n, m, seed, r, mode):
    kh, nh, f, c, st, rep, ores = _both(mpg, orc, gen, n, m, seed, r, mode)
    assert rep.converged and ores.converged
    lam, lamo = np.sort_complex(st.lam), np.sort_complex(ores.lam)
    assert np.linalg.norm(lam - lamo) <= 1e-6 * np.linalg.norm(lamo)
    assert abs(st.sweeps - ores.sweeps) <= max(1, ores.sweeps // 10)
    pts = [0.1j, 1.0j, 10.0j, 1.0]
    a = _kernels(st.kr, st.nr, st.fr, st.cr, pts)
    b = _kernels(ores.kr, ores.nr, ores.fr, ores.cr, pts)
    assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b)


def test_coupled_projection_identities(mpg, orc, gen):  # test_birka.cpp:102-132
    kh, nh, f, c, st, rep, _ = _both(mpg, orc, gen, 30, 2, 2, 3, 2)
    v, w = st.v, st.w
    assert np.linalg.norm(v.T @ v - np.eye(3)) <= 1e-12 and np.linalg.norm(w.T @ w - np.eye(3)) <= 1e-12
    obl = lambda x: np.linalg.solve(w.T @ v, w.T @ x)
    assert np.linalg.norm(obl(kh.to_dense() @ v) - st.kr) <= 1e-10 * (1 + np.linalg.norm(st.kr))
    for j in range(2):
        assert np.linalg.norm(obl(nh[j].to_dense() @ v) - st.nr[j]) <= 1e-10 * (1 + np.linalg.norm(st.nr[j]))
    assert np.linalg.norm(obl(f) - st.fr) <= 1e-10 * (1 + np.linalg.norm(st.fr))
    assert np.linalg.norm(v.T @ c - st.cr) <= 1e-10 * (1 + np.linalg.norm(st.cr))


def test_coupled_report_fresh_then_vertical(mpg, orc, gen):  # test_birka.cpp:134-168
    *_, st, rep, ores = _both(mpg, orc, gen, 6, 1, 3, 2, 2)
    assert rep.converged and len(rep.rows) == 2 * rep.sweeps
    kinds = [r.kind for r in rep.rows]
    assert kinds.count("fresh") == 2 and kinds.count("vertical") == 2 * (rep.sweeps - 1)
    if rep.sweeps == ores.sweeps:
        assert kinds == [{0: "none", 1: "fresh", 3: "vertical"}[r.kind] for r in ores.rows]


def test_coupled_oversized_explicit_degrades(mpg, orc, gen):  # test_birka.cpp:170-187
    *_, st, rep, ores = _both(mpg, orc, gen, 6, 1, 4, 2, 2, cap=3)
    assert rep.converged and all(r.kind == "none" for r in rep.rows)
    assert len(rep.warnings) == 2 and all("cap" in w for w in rep.warnings)
    assert np.linalg.norm(np.sort_complex(st.lam) - np.sort_complex(ores.lam)) <= 1e-6 * np.linalg.norm(ores.lam)


def test_coupled_input_validation(mpg, gen):
    kh, nh, f, c = gen.bilinear_toy_n(6, 2, 1)
    k = _m(mpg, kh)
    cfg = mpg.IrkaConfig(r=2)
    with pytest.raises(ValueError):
        mpg.birka_reduce(k, [_m(mpg, nh[0])], f, c, cfg)
    with pytest.raises(mpg.ConfigError):
        mpg.birka_reduce(k, [_m(mpg, x) for x in nh], f, c, mpg.IrkaConfig(r=7))


def test_coupled_frozen_preconditioner(mpg, orc, gen):
    """REUSE_FROZEN (extension): one SPAI per side at the first sweep, applied unchanged afterwards; the fixed
    point is the oracle's."""
    kh, nh, f, c, st, rep, ores = _both(mpg, orc, gen, 60, 3, 9, 3, 3)
    assert rep.converged and ores.converged
    kinds = [r.kind for r in rep.rows]
    assert kinds[:2] == ["fresh", "fresh"] and all(k == "reused_same_matrix" for k in kinds[2:])
    lam, lamo = np.sort_complex(st.lam), np.sort_complex(ores.lam)
    assert np.linalg.norm(lam - lamo) <= 1e-6 * np.linalg.norm(lamo)
