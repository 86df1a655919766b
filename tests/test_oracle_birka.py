"""Pins the oracle's BIRKA with couplings (N_j != 0, SURVEY.md §8 f4;
proj/src/birka.cpp:139-310, kron.cpp:34-131) to proj/tests/test_birka.cpp
(cited per test) on the bilinear toy with its couplings
(proj/src/generator.cpp:141-179, restated in csrc/gen/generators.cpp)."""
import numpy as np
import pytest


def _toy(orc, gen, n, m, seed):
    k, ns, f, c = gen.bilinear_toy_n(n, m, seed)
    return orc.Csr.of(k), [orc.Csr.of(x) for x in ns], f, c, k, ns


def test_kron_apply_and_assembly_with_couplers(orc, gen):  # test_kron.cpp:81-97 with couplers
    k, ns, f, c, kh, nh = _toy(orc, gen, 7, 2, 11)
    r = 3
    rng = np.random.default_rng(1)
    lam = np.diag([-1.0, -2.0, -3.5])
    S = [rng.standard_normal((r, r)) for _ in range(2)]
    x = rng.standard_normal(7 * r)
    X = x.reshape((7, r), order="F")
    K, N = kh.to_dense(), [h.to_dense() for h in nh]
    want = -(X @ lam.T) - K @ X - sum(N[j] @ X @ S[j] for j in range(2))
    dense = -np.kron(lam, np.eye(7)) - np.kron(np.eye(r), K) - sum(np.kron(S[j].T, N[j]) for j in range(2))
    assert np.linalg.norm(dense @ x - want.reshape(-1, order="F")) <= 1e-12 * np.linalg.norm(want)
    got = orc.kron_apply_coupled(lam, k, [(S[j], ns[j]) for j in range(2)], x)
    assert np.linalg.norm(got - want.reshape(-1, order="F")) <= 1e-13 * np.linalg.norm(want)
    m = orc.kron_assemble_coupled(lam, k, [(S[j], ns[j]) for j in range(2)])
    assert np.linalg.norm(m.to_dense() - dense) <= 1e-13 * np.linalg.norm(dense)


def test_fixed_point_deterministic_and_mode_independent(orc, gen):  # :77-100
    k, ns, f, c, _, _ = _toy(orc, gen, 6, 1, 1)
    cfg = orc.IrkaConfig(r=2, tol=1e-10, max_sweeps=200, seed=1, gmres=orc.GmresConfig(1e-12, 1000))
    r1 = orc.birka_reduce(k, ns, f, c, cfg, mode=2)
    r2 = orc.birka_reduce(k, ns, f, c, cfg, mode=2)
    r3 = orc.birka_reduce(k, ns, f, c, cfg, mode=1)
    assert r1.converged and r2.converged and r3.converged
    l1 = np.sort_complex(r1.lam)
    assert np.linalg.norm(l1 - np.sort_complex(r2.lam)) <= 1e-10 * np.linalg.norm(l1)
    assert np.linalg.norm(l1 - np.sort_complex(r3.lam)) <= 1e-6 * np.linalg.norm(l1)
    assert np.all(l1.real < 0) and r1.sweeps == r2.sweeps


def test_two_sided_projection_identities(orc, gen):  # :102-132
    k, ns, f, c, kh, nh = _toy(orc, gen, 8, 2, 2)
    res = orc.birka_reduce(k, ns, f, c, orc.IrkaConfig(r=2, tol=1e-8, max_sweeps=200, seed=2,
                                                       gmres=orc.GmresConfig(1e-12, 1000)), mode=2)
    assert res.converged
    v, w = res.v, res.w
    assert np.linalg.norm(v.T @ v - np.eye(2)) <= 1e-12 and np.linalg.norm(w.T @ w - np.eye(2)) <= 1e-12
    obl = lambda x: np.linalg.solve(w.T @ v, w.T @ x)
    assert np.linalg.norm(obl(kh.to_dense() @ v) - res.kr) <= 1e-10 * (1 + np.linalg.norm(res.kr))
    for j in range(2):
        assert np.linalg.norm(obl(nh[j].to_dense() @ v) - res.nr[j]) <= 1e-10 * (1 + np.linalg.norm(res.nr[j]))
    assert np.linalg.norm(obl(f) - res.fr) <= 1e-10 * (1 + np.linalg.norm(res.fr))
    assert np.linalg.norm(v.T @ c - res.cr) <= 1e-10 * (1 + np.linalg.norm(res.cr))


def test_reuse_report_fresh_then_vertical(orc, gen):  # :134-168
    k, ns, f, c, _, _ = _toy(orc, gen, 6, 1, 3)
    res = orc.birka_reduce(k, ns, f, c, orc.IrkaConfig(r=2, tol=1e-8, max_sweeps=200, seed=3,
                                                       gmres=orc.GmresConfig(1e-12, 1000)), mode=2)
    assert res.converged and len(res.rows) == 2 * res.sweeps
    kinds = [r.kind for r in res.rows]
    assert kinds.count(1) == 2 and kinds.count(3) == 2 * (res.sweeps - 1)
    for r in res.rows:
        if r.kind == 3:
            assert r.sweep >= 2 and r.min_residual <= r.matrix_change


def test_oversized_explicit_degrades(orc, gen):  # :170-187
    k, ns, f, c, _, _ = _toy(orc, gen, 6, 1, 4)
    res = orc.birka_reduce(k, ns, f, c, orc.IrkaConfig(r=2, tol=1e-8, max_sweeps=200, seed=4,
                                                       gmres=orc.GmresConfig(1e-12, 1000), explicit_nnz_cap=3), mode=2)
    assert res.converged and all(r.kind == 0 for r in res.rows)
