"""AIRGA (proj/src/airga.cpp:136-384, proj/src/h2.cpp) on the
GPU path, restating proj/tests/test_airga.cpp (cited per test) with the dense
oracles those tests use; the host helpers (H2 norm, expansion-point update)
run without a device and are checked on the CPU against scipy / the
reference's hand values."""
import numpy as np
import pytest

NONE, FRESH, REUSE = 0, 1, 2
KIND = {"fresh": 1, "horizontal": 2, "vertical": 3, "reused_same_matrix": 4, "none": 0}


def spd(gen, n, seed):  # test_airga.cpp:32-36
    r = gen.random_dense(n, n, seed)
    return r @ r.T + n * np.eye(n)


def dense_shift(M, D, K, s):
    return s * s * M + s * D + K


def reduced_transfer(red, s):
    return red.c.T @ np.linalg.solve(s * s * red.m + s * red.d + red.k, red.f)


def same_span(a, b, tol):
    def rank(x):
        sv = np.linalg.svd(x, compute_uv=False)
        return 0 if sv.size == 0 or sv[0] == 0 else int(np.sum(sv > tol * sv[0]))
    return rank(a) == rank(b) == rank(np.hstack([a, b]))


# ---------------------------------------------------------------- host helpers (CPU)
@pytest.mark.parametrize("ns", [2, 7, 20, 40])
def test_h2_norm_matches_lyapunov(mpg, ns):  # h2.cpp:28-60 vs a Lyapunov solve
    import scipy.linalg as sl
    rng = np.random.default_rng(ns)
    A = rng.standard_normal((ns, ns))
    A -= (np.max(np.linalg.eigvals(A).real) + 0.5) * np.eye(ns)
    B, Cc = rng.standard_normal((ns, 2)), rng.standard_normal((3, ns))
    P = sl.solve_continuous_lyapunov(A, -B @ B.T)
    want = np.sqrt(np.trace(Cc @ P @ Cc.T))
    assert abs(mpg.h2_norm(A, B, Cc) - want) <= 1e-10 * want


def test_h2_norm_unstable_is_inf_and_self_distance_zero(mpg):
    assert mpg.h2_norm(np.array([[0.1]]), np.ones((1, 1)), np.ones((1, 1))) == float("inf")
    A = np.diag([-1.0, -2.0, -3.0])
    AA = np.block([[A, np.zeros((3, 3))], [np.zeros((3, 3)), A]])
    assert mpg.h2_norm(AA, np.ones((6, 1)), np.hstack([np.ones((1, 3)), -np.ones((1, 3))])) <= 1e-12


def test_expansion_point_update(mpg):  # test_airga.cpp:267-289
    nxt = mpg.update_expansion_points(np.eye(4), np.zeros((4, 4)), np.diag([1.0, 4, 9, 16]), [5.0, 6.0])
    assert len(nxt) == 2 and abs(nxt[0] - 3.0) <= 3e-9 and abs(nxt[1] - 4.0) <= 4e-9
    kept = mpg.update_expansion_points(np.eye(3), np.zeros((3, 3)), np.zeros((3, 3)), [7.0, 9.0])
    assert kept == [7.0, 9.0]


# ---------------------------------------------------------------- GPU path
def _sys(mpg, M, D, K, F, Cc, alpha=0.0, beta=0.0):
    sm = mpg.SparseMatrix.from_dense
    return mpg.SecondOrderSystem.create(sm(M), sm(D), sm(K), F, Cc, alpha, beta)


def _small(mpg, gen, n, n_in, seed, alpha, beta):  # test_airga.cpp:51-58
    M, K = spd(gen, n, seed), spd(gen, n, seed + 1)
    F, Cc = gen.random_dense(n, n_in, seed + 2), gen.random_dense(n, n_in, seed + 3)
    return _sys(mpg, M, alpha * M + beta * K, K, F, Cc, alpha, beta), (M, alpha * M + beta * K, K, F, Cc)


def _brake(mpg, gen, n, omega, alpha, beta, seed):
    m, k = gen.disc_brake(n, omega, seed)
    M, K = m.to_scipy(), k.to_scipy()
    D = (alpha * M + beta * K).tocsr()
    D.eliminate_zeros()
    e1 = np.zeros((n, 1))
    e1[0] = 1.0
    ms = mpg.SparseMatrix.from_scipy
    return mpg.SecondOrderSystem.create(ms(M), ms(D), ms(K), e1, e1, alpha, beta), (M, D, K, e1, e1)


@pytest.mark.gpu
def test_decoupled_mode_exact_at_order_one(mpg):  # test_airga.cpp:84-107
    e1 = np.eye(4)[:, :1]
    sys_ = _sys(mpg, np.eye(4), np.zeros((4, 4)), np.diag([1.0, 2, 3, 4]), e1, e1)
    red, rep = mpg.airga_reduce(sys_, mpg.AirgaConfig(expansion_points=[1.0], r_max=2, inner_tol=0.0, max_outer=1,
                                                      gmres=mpg.GmresConfig(1e-13, 1000)), NONE)
    assert red.order() == 1
    for s in (0.5, 1.0, 3.0):
        assert abs(reduced_transfer(red, s)[0, 0] - 1.0 / (s * s + 1.0)) <= 1e-10


@pytest.mark.gpu
def test_single_point_spans_shifted_block_krylov(mpg, gen):  # :109-132
    sys_, (M, D, K, F, Cc) = _small(mpg, gen, 10, 1, 21, 0.1, 0.05)
    s0 = 1.7
    red, _ = mpg.airga_reduce(sys_, mpg.AirgaConfig(expansion_points=[s0], r_max=4, inner_tol=0.0, max_outer=1,
                                                    gmres=mpg.GmresConfig(1e-13, 200)), NONE)
    assert red.order() == 4
    A = dense_shift(M, D, K, s0)
    kry = [np.linalg.solve(A, F[:, 0])]
    for _ in range(3):
        kry.append(np.linalg.solve(A, M @ kry[-1]))
    kry = np.column_stack([v / np.linalg.norm(v) for v in kry])
    assert same_span(red.basis, kry, 1e-8)


@pytest.mark.gpu
def test_first_moments_match_in_damped_shift(mpg, gen):  # :134-168
    alpha, beta = 0.02, 0.01
    sys_, (M, D, K, F, Cc) = _small(mpg, gen, 12, 2, 33, alpha, beta)
    s0 = 1.3
    red, _ = mpg.airga_reduce(sys_, mpg.AirgaConfig(expansion_points=[s0], r_max=6, inner_tol=0.0, max_outer=1,
                                                    gmres=mpg.GmresConfig(1e-13, 200)), NONE)
    assert red.order() == 6
    w0 = (s0 * s0 + alpha * s0) / (beta * s0 + 1.0)
    x = np.linalg.solve(w0 * M + K, F)
    xr = np.linalg.solve(w0 * red.m + red.k, red.f)
    for _ in range(3):
        mom, momr = Cc.T @ x, red.c.T @ xr
        assert np.linalg.norm(mom - momr) <= 1e-8 * max(1.0, np.linalg.norm(mom))
        x = np.linalg.solve(w0 * M + K, M @ x)
        xr = np.linalg.solve(w0 * red.m + red.k, red.m @ xr)


@pytest.mark.gpu
def test_projection_identities(mpg, gen):  # :170-187
    sys_, (M, D, K, F, Cc) = _brake(mpg, gen, 80, 6.28, 5e-2, 5e-6, 7)
    red, _ = mpg.airga_reduce(sys_, mpg.AirgaConfig(expansion_points=[6.28, 200.0], r_max=8, max_outer=2,
                                                    outer_tol=1e30), REUSE)
    V, r = red.basis, red.order()
    assert np.linalg.norm(V.T @ V - np.eye(r)) <= 1e-10
    for full, got in ((M, red.m), (D, red.d), (K, red.k)):
        assert np.linalg.norm(V.T @ (full @ V) - got) <= 1e-10 * (1.0 + np.linalg.norm(got))
    assert np.linalg.norm(V.T @ F - red.f) <= 1e-10 * (1.0 + np.linalg.norm(red.f))
    assert np.linalg.norm(V.T @ Cc - red.c) <= 1e-10 * (1.0 + np.linalg.norm(red.c))


@pytest.mark.gpu
def test_fresh_and_reused_give_same_model(mpg, gen):  # :189-265
    sys_, _ = _brake(mpg, gen, 120, 6.283, 5e-2, 5e-6, 3)
    cfg = mpg.AirgaConfig(expansion_points=[6.283, 700.0, 1500.0, 3100.0], r_max=12, max_outer=2, outer_tol=1e30,
                          gmres=mpg.GmresConfig(1e-10, 1000))
    red_f, rep_f = mpg.airga_reduce(sys_, cfg, FRESH)
    red_r, rep_r = mpg.airga_reduce(sys_, cfg, REUSE)
    assert red_f.order() == red_r.order()
    for s in (10.0, 300.0, 2000.0):
        hf, hr = reduced_transfer(red_f, s), reduced_transfer(red_r, s)
        assert np.linalg.norm(hf - hr) <= 1e-6 * max(1e-300, np.linalg.norm(hf))
    assert rep_f.totals()["solves"] == rep_r.totals()["solves"]
    kinds = [KIND[x.kind] for x in rep_r.rows]
    assert kinds.count(1) == 1 and kinds.count(2) == 2 * 3 and kinds.count(3) == 1 and kinds.count(4) >= 1
    for x in rep_r.rows:
        if x.kind == "fresh":
            assert x.sweep == 1 and x.point == 1
        if x.kind == "vertical":
            assert x.sweep == 2 and x.point == 1
        if x.kind in ("horizontal", "vertical"):
            assert np.isfinite(x.min_residual) and x.min_residual <= x.matrix_change
        if x.kind == "reused_same_matrix":
            assert x.precond_build_seconds == 0.0 and x.solves >= 1
        else:
            assert np.isfinite(x.standard_residual) and x.standard_residual > 0.0


@pytest.mark.gpu
def test_non_proportional_damping_warns(mpg, gen):  # :291-311
    M, K = spd(gen, 6, 51), spd(gen, 6, 52)
    D = 0.1 * M + 0.02 * K
    D[0, 1] += 0.5
    sys_ = _sys(mpg, M, D, K, gen.random_dense(6, 1, 53), gen.random_dense(6, 1, 54), 0.1, 0.02)
    _, rep = mpg.airga_reduce(sys_, mpg.AirgaConfig(expansion_points=[1.0], r_max=2, max_outer=1), NONE)
    assert any("damping deviates" in w for w in rep.warnings)


@pytest.mark.gpu
def test_configuration_is_validated(mpg, gen):  # :379-395
    sys_, _ = _small(mpg, gen, 6, 1, 99, 0.1, 0.01)
    for pts, r_max, max_outer in (([], 20, 20), ([1.0, -2.0], 20, 20), ([1.0, 1.0], 20, 20), ([1.0, 2.0, 3.0], 2, 20),
                                  ([1.0, 2.0, 3.0], 8, 0)):
        with pytest.raises(mpg.ConfigError):
            mpg.airga_reduce(sys_, mpg.AirgaConfig(expansion_points=pts, r_max=r_max, max_outer=max_outer), NONE)


@pytest.mark.gpu
def test_config_scale_run_interpolates(mpg, gen):
    """A C2-size second-order model (M = E, K = -A of config 2 at 24^3, D = 0.05 M +
    1e-4 K, SISO): the reduced model is a Galerkin projection containing the
    zeroth moments, so it reproduces H(s) at the final expansion points."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    c2 = gen.config2(M=24)
    Ms, Ks = c2.e_csr().to_scipy(), -c2.a.to_scipy()
    Ds = (0.05 * Ms + 1e-4 * Ks).tocsr()
    f, c = c2.b[:, :1], c2.c[:, :1]
    ms = lambda a: mpg.SparseMatrix.from_scipy(sp.csr_matrix(a))
    sys_ = mpg.SecondOrderSystem.create(ms(Ms), ms(Ds), ms(Ks), f, c, 0.05, 1e-4)
    red, rep = mpg.airga_reduce(sys_, mpg.AirgaConfig(expansion_points=[1.0, 10.0, 100.0], r_max=12, max_outer=3,
                                                      gmres=mpg.GmresConfig(1e-10, 1000)), REUSE)
    V, r = red.basis, red.order()
    assert r >= 3 and np.linalg.norm(V.T @ V - np.eye(r)) <= 1e-8
    # the zeroth moments of the last sweep's points are in the basis: exact interpolation there
    for s in rep.final_points:
        full = float(c[:, 0] @ sla.spsolve((s * s * Ms + s * Ds + Ks).tocsc(), f[:, 0]))
        assert abs(reduced_transfer(red, s)[0, 0] - full) <= 1e-6 * abs(full)
