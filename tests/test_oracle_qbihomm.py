"""Pins the CPU oracle's QB-IHOMM restatement (oracle/qbihomm.cpp) to the
reference's own tests, proj/tests/test_qbihomm.cpp (cited per test), on the
same seeded fixtures (generate_qb_toy and support.hpp's random_dense,
restated in csrc/gen/generators.cpp with the same libstdc++ streams)."""
import numpy as np
import pytest

NONE, FRESH, REUSE = 0, 1, 2
KIND_FRESH, KIND_HORIZONTAL, KIND_REUSED = 1, 2, 4


def _svd_rank(m, tol):
    if m.size == 0:
        return 0
    s = np.linalg.svd(m, compute_uv=False)
    return 0 if s[0] == 0 else int(np.sum(s > tol * s[0]))


def same_span(a, b, tol=1e-10):  # support.hpp:70-79
    ra, rb = _svd_rank(a, tol), _svd_rank(b, tol)
    return ra == rb and _svd_rank(np.hstack([a, b]), tol) == ra


def tight(orc, sigmas, p, q):  # test_qbihomm.cpp:42-49
    return orc.QbConfig(sigmas=list(sigmas), p_moments=p, q_moments=q, gmres=orc.GmresConfig(1e-13, 500))


def qb(orc, s):
    c = orc.Csr.of
    return c(s.d), c(s.k), c(s.n_op), c(s.h), s.f, s.c


def test_single_point_zeroth_order_by_hand(orc):  # test_qbihomm.cpp:52-71
    n = 4
    e1 = np.zeros(n)
    e1[0] = 1.0
    red = orc.qbihomm_reduce(orc.Csr.identity(n), orc.Csr.from_dense(-np.eye(n)), orc.Csr.zero(n, n),
                             orc.Csr.zero(n, n * n), e1, e1, tight(orc, [1.0], 0, 0), NONE)
    assert red.order() == 1
    assert red.d[0, 0] == pytest.approx(1.0, rel=1e-10)
    assert red.k[0, 0] == pytest.approx(-1.0, rel=1e-10)
    assert abs(red.n_op[0, 0]) <= 1e-12
    assert np.linalg.norm(red.h) <= 1e-12
    assert red.f[0, 0] * red.c[0, 0] == pytest.approx(1.0, rel=1e-10)


def test_basis_spans_two_sided_moments(orc, gen):  # test_qbihomm.cpp:73-108
    s = gen.qb_toy(5, 3)
    sig, p, q = [1.0, 2.5], 1, 1
    red = orc.qbihomm_reduce(*qb(orc, s), tight(orc, sig, p, q), NONE)
    D, K = s.d.to_dense(), s.k.to_dense()
    cols = []
    for sg in sig:
        x = np.linalg.solve(sg * D - K, s.f)
        cols.append(x)
        for _ in range(p + q):
            x = np.linalg.solve(sg * D - K, D @ x)
            cols.append(x)
        y = np.linalg.solve((2 * sg * D - K).T, s.c)
        cols.append(y)
        for _ in range(q):
            y = np.linalg.solve((2 * sg * D - K).T, D.T @ y)
            cols.append(y)
    want = np.column_stack([v / np.linalg.norm(v) for v in cols])
    assert same_span(red.basis, want, 1e-8)
    r = red.order()
    assert np.linalg.norm(red.basis.T @ red.basis - np.eye(r)) <= 1e-10


def test_quadratic_compression_matches_dense_kron(orc, gen):  # test_qbihomm.cpp:110-129
    hd = gen.random_dense(3, 9, 17)
    h = orc.Csr.from_dense(hd)
    u, _ = np.linalg.qr(gen.random_dense(3, 2, 18))
    got = orc.kron_compress_quadratic(h, u)
    want = u.T @ hd @ np.kron(u, u)
    assert got.shape == (2, 4)
    assert np.linalg.norm(got - want) <= 1e-12 * (1 + np.linalg.norm(want))
    assert np.linalg.norm(orc.kron_compress_quadratic(orc.Csr.zero(3, 9), u)) == 0.0
    assert np.linalg.norm(orc.kron_compress_quadratic(h, np.eye(3)) - hd) == 0.0
    with pytest.raises(ValueError):
        orc.kron_compress_quadratic(orc.Csr.from_dense(gen.random_dense(3, 8, 19)), u)


def test_reduced_matrices_are_projections(orc, gen):  # test_qbihomm.cpp:131-148
    s = gen.qb_toy(6, 4)
    red = orc.qbihomm_reduce(*qb(orc, s), tight(orc, [0.8, 1.7, 3.0], 1, 1), NONE)
    u, r = red.basis, red.order()
    assert np.linalg.norm(u.T @ u - np.eye(r)) <= 1e-10
    for full, got in ((s.d, red.d), (s.k, red.k), (s.n_op, red.n_op)):
        assert np.linalg.norm(u.T @ full.to_dense() @ u - got) <= 1e-10 * (1 + np.linalg.norm(got))
    assert np.linalg.norm(u.T @ s.f - red.f[:, 0]) <= 1e-10 * (1 + np.linalg.norm(red.f))
    assert np.linalg.norm(u.T @ s.c - red.c[:, 0]) <= 1e-10 * (1 + np.linalg.norm(red.c))
    want_h = u.T @ s.h.to_dense() @ np.kron(u, u)
    assert np.linalg.norm(red.h - want_h) <= 1e-10 * (1 + np.linalg.norm(want_h))


def test_report_rows_follow_side_chain_layout(orc, gen):  # test_qbihomm.cpp:150-213
    s = gen.qb_toy(8, 5)
    cfg = tight(orc, [0.9, 1.8, 2.7], 1, 1)
    reuse = orc.qbihomm_reduce(*qb(orc, s), cfg, REUSE)
    fresh = horizontal = reused = 0
    for row in reuse.rows:
        assert row.sweep in (1, 2)
        if row.kind == KIND_FRESH:
            fresh += 1
            assert row.point == 1 and row.solves == 1
        elif row.kind == KIND_HORIZONTAL:
            horizontal += 1
            assert row.point >= 2 and row.solves == 1
            assert np.isfinite(row.min_residual) and row.min_residual <= row.matrix_change
        elif row.kind == KIND_REUSED:
            reused += 1
            assert row.build_seconds == 0.0
        else:
            pytest.fail("unexpected row kind")
        if row.kind != KIND_REUSED:
            assert np.isfinite(row.standard_residual) and row.standard_residual > 0.0
    assert (fresh, horizontal, reused) == (2, 4, 6)
    trial = sum(r.solves for r in reuse.rows if r.sweep == 1)
    test = sum(r.solves for r in reuse.rows if r.sweep == 2)
    assert (trial, test) == (9, 6)
    fr = orc.qbihomm_reduce(*qb(orc, s), cfg, FRESH)
    assert sum(1 for r in fr.rows if r.kind == KIND_FRESH) == 6
    assert fr.order() == reuse.order()
    for sv in (0.9, 2.0, 4.0):
        hf, hr = fr.linear_transfer(sv), reuse.linear_transfer(sv)
        assert abs(hf - hr) <= 1e-6 * max(1e-300, abs(hf))


def test_inputs_are_validated(orc, gen):  # test_qbihomm.cpp:249-268
    s = gen.qb_toy(5, 7)
    d, k, nop, h, f, c = qb(orc, s)
    with pytest.raises(orc.ConfigError):
        orc.qbihomm_reduce(d, k, nop, orc.Csr.zero(5, 24), f, c, tight(orc, [1.0], 1, 1), NONE)
    with pytest.raises(orc.ConfigError):
        orc.qbihomm_reduce(d, k, nop, h, gen.random_dense(5, 2, 1), c, tight(orc, [1.0], 1, 1), NONE)
    for sig, p in (([], 1), ([1.0, 1.0], 1), ([0.0], 1), ([1.0], -1)):
        with pytest.raises(orc.ConfigError):
            orc.qbihomm_reduce(d, k, nop, h, f, c, tight(orc, sig, p, 1), NONE)
