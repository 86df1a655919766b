"""transfer_function_error (SURVEY.md §8 f2's grid walk, proj/src/airga.cpp:
386-447): the oracle restatement pinned to proj/tests/test_airga.cpp:313-377
(CPU), and the GPU path (-m gpu) on the same cases and against the oracle."""
import numpy as np
import pytest

NONE, FRESH, REUSE = 0, 1, 2


def spd(gen, n, seed):  # test_airga.cpp:32-36
    r = gen.random_dense(n, n, seed)
    return r @ r.T + n * np.eye(n)


def small_system(gen, n, n_in, seed, alpha, beta):  # test_airga.cpp:51-58
    m, k = spd(gen, n, seed), spd(gen, n, seed + 1)
    return m, alpha * m + beta * k, k, gen.random_dense(n, n_in, seed + 2), gen.random_dense(n, n_in, seed + 3)


def dense_transfer(M, D, K, F, Cc, s):
    return Cc.T @ np.linalg.solve(s * s * M + s * D + K, F)


def projected(M, D, K, F, Cc, U):
    return U.T @ M @ U, U.T @ D @ U, U.T @ K @ U, U.T @ F, U.T @ Cc


def moment_basis(M, D, K, F, points):
    cols = [np.linalg.solve(s * s * M + s * D + K, F) for s in points]
    q, _ = np.linalg.qr(np.hstack(cols))
    return q


def reduced_transfer(red, s):
    m, d, k, f, c = red
    return c.T @ np.linalg.solve(s * s * m + s * d + k, f)


def _orc_tf(orc, M, D, K, F, Cc, red, grid, mode, tol):
    c = orc.Csr.from_dense
    return orc.transfer_function_error(c(M), c(D), c(K), F, Cc, red, grid, orc.GmresConfig(tol, 1000), mode=mode)


@pytest.mark.parametrize("mode", [NONE, FRESH, REUSE])
def test_oracle_matches_dense(orc, gen, mode):  # test_airga.cpp:313-334
    M, D, K, F, Cc = small_system(gen, 20, 1, 77, 0.3, 0.02)
    red = projected(M, D, K, F, Cc, moment_basis(M, D, K, F, [1.0, 4.0]))
    grid = [0.5, 1.0, 2.5, 4.0, 8.0]
    got = _orc_tf(orc, M, D, K, F, Cc, red, grid, mode, 1e-12)
    for g, s in zip(got, grid):
        h = dense_transfer(M, D, K, F, Cc, s)
        want = np.linalg.norm(h - reduced_transfer(red, s)) / np.linalg.norm(h)
        assert np.isfinite(g) and abs(g - want) <= 1e-8 * max(1.0, want)


def test_oracle_identity_reduction_is_zero(orc, gen):  # :336-353
    M, D, K, F, Cc = small_system(gen, 6, 1, 91, 0.4, 0.05)
    errs = _orc_tf(orc, M, D, K, F, Cc, (M, D, K, F, Cc), [1.0, 2.0, 5.0], NONE, 1e-10)
    assert np.all(np.isfinite(errs)) and np.all(errs <= 1e-6)


def test_oracle_unsolvable_points_are_nan(orc):  # :355-377
    e1 = np.eye(3)[:, :1]
    M, D, K = np.eye(3), np.zeros((3, 3)), -np.eye(3)
    errs = _orc_tf(orc, M, D, K, e1, e1, (M, D, K, e1, e1), [0.5, 1.0, 2.0, -3.0], NONE, 1e-10)
    assert errs[0] <= 1e-6 and np.isnan(errs[1]) and errs[2] <= 1e-6 and np.isnan(errs[3])


# ---------------------------------------------------------------- GPU path
def _gpu_sys(mpg, M, D, K, F, Cc):
    sm = lambda a: mpg.SparseMatrix.from_dense(a) if isinstance(a, np.ndarray) else a
    return mpg.SecondOrderSystem.create(sm(M), sm(D), sm(K), F, Cc)


def _gpu_tf(mpg, sys_, red, grid, mode, tol):
    return mpg.transfer_function_error(sys_, mpg.ReducedSecondOrder(*red), grid,
                                       mpg.TransferErrorConfig(mpg.GmresConfig(tol, 1000), mode=mode))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [NONE, FRESH, REUSE])
def test_gpu_matches_dense_and_oracle(mpg, orc, gen, mode):
    M, D, K, F, Cc = small_system(gen, 20, 1, 77, 0.3, 0.02)
    red = projected(M, D, K, F, Cc, moment_basis(M, D, K, F, [1.0, 4.0]))
    grid = [0.5, 1.0, 2.5, 4.0, 8.0]
    got = _gpu_tf(mpg, _gpu_sys(mpg, M, D, K, F, Cc), red, grid, mode, 1e-12)
    want_o = _orc_tf(orc, M, D, K, F, Cc, red, grid, mode, 1e-12)
    for g, wo, s in zip(got, want_o, grid):
        h = dense_transfer(M, D, K, F, Cc, s)
        want = np.linalg.norm(h - reduced_transfer(red, s)) / np.linalg.norm(h)
        assert np.isfinite(g) and abs(g - want) <= 1e-8 * max(1.0, want)
        assert abs(g - wo) <= 1e-6 * max(abs(wo), 1e-8)  # errors at the interpolation points are rounding-level


@pytest.mark.gpu
def test_gpu_identity_and_unsolvable(mpg, gen):  # :336-377 on the GPU path
    M, D, K, F, Cc = small_system(gen, 6, 1, 91, 0.4, 0.05)
    errs = _gpu_tf(mpg, _gpu_sys(mpg, M, D, K, F, Cc), (M, D, K, F, Cc), [1.0, 2.0, 5.0], NONE, 1e-10)
    assert np.all(np.isfinite(errs)) and np.all(errs <= 1e-6)
    e1 = np.eye(3)[:, :1]
    M, D, K = np.eye(3), np.zeros((3, 3)), -np.eye(3)
    sys_ = mpg.SecondOrderSystem.create(mpg.SparseMatrix.identity(3), mpg.SparseMatrix.zero(3, 3),
                                        mpg.SparseMatrix.from_dense(K), e1, e1)
    errs = _gpu_tf(mpg, sys_, (M, D, K, e1, e1), [0.5, 1.0, 2.0, -3.0], NONE, 1e-10)
    assert errs[0] <= 1e-6 and np.isnan(errs[1]) and errs[2] <= 1e-6 and np.isnan(errs[3])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [FRESH, REUSE])
def test_gpu_config_scale_grid_walk(mpg, orc, gen, mode):
    """A damped second-order model from C2's matrices (M = E, K = -A, D = 0.1 M +
    1e-4 K, MIMO 2 x 2 from the config's B, C) at n = 16^3 against the oracle,
    on an 8-point log grid walked by one horizontal chain (REUSE) or fresh SPAI."""
    import scipy.sparse as sp
    c2 = gen.config2(M=16)
    n = c2.n
    Ms = c2.e_csr().to_scipy()
    Ks = -c2.a.to_scipy()
    Ds = (0.1 * Ms + 1e-4 * Ks).tocsr()
    rng = np.random.default_rng(5)
    F = rng.standard_normal((n, 2))
    Cc = rng.standard_normal((n, 2))
    U, _ = np.linalg.qr(rng.standard_normal((n, 6)))
    red = (U.T @ (Ms @ U), U.T @ (Ds @ U), U.T @ (Ks @ U), U.T @ F, U.T @ Cc)
    grid = list(np.logspace(0, 2, 8))
    msp = lambda a: mpg.SparseMatrix.from_scipy(sp.csr_matrix(a))
    got = mpg.transfer_function_error(mpg.SecondOrderSystem.create(msp(Ms), msp(Ds), msp(Ks), F, Cc),
                                      mpg.ReducedSecondOrder(*red), grid,
                                      mpg.TransferErrorConfig(mpg.GmresConfig(1e-10, 1000), mode=mode))
    oc = lambda a: orc.Csr.from_csr(a.shape[0], a.shape[1], a.indptr, a.indices, a.data)
    want = orc.transfer_function_error(oc(sp.csr_matrix(Ms)), oc(Ds), oc(sp.csr_matrix(Ks)), F, Cc, red, grid,
                                       orc.GmresConfig(1e-10, 1000), mode=mode)
    assert np.all(np.isfinite(got)) and np.all(np.isfinite(want))
    assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-6
