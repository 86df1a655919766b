"""GPU parity: shifted SpMV (K1/K1T/K1c), transpose, chain apply (K2), SPAI and
update builds (K4) against the CPU oracle on the same seeded inputs."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _pair(gen, host):
    import oracle as O
    from paper_2003_12759_b200 import SparseMatrix
    return SparseMatrix.from_csr(host.nrows, host.ncols, host.rowptr, host.colind, host.val), O.Csr.of(host)


def test_csr_multiply_and_transpose(mpg, orc, gen):
    for n in (1, 7, 23, 50, 333):
        h = gen.random_sparse(n, n, 0.3, 100 + n)
        g, o = _pair(gen, h)
        x = gen.random_dense(n, 1, 200 + n)[:, 0]
        assert rel(g.multiply(x), o.multiply(x)) <= 1e-13
        assert rel(g.multiply_transpose(x), o.multiply_transpose(x)) <= 1e-13
        rp, ci, v = g.transpose().download()
        rp2, ci2, v2 = o.transpose().export()
        assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2)


def test_csr_validation(mpg):
    with pytest.raises(ValueError):
        mpg.SparseMatrix.from_csr(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        mpg.SparseMatrix.from_csr(2, 2, [0, 1, 2], [0, 5], [1.0, 1.0])
    with pytest.raises(ValueError):
        mpg.SparseMatrix.from_csr(1, 3, [0, 2], [1, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        mpg.SparseMatrix.identity(3).multiply(np.ones(2))


@pytest.mark.parametrize("emode", ["ident", "diag", "samepat", "general"])
@pytest.mark.parametrize("sigma", [0.7, 3.0 - 1.5j])
@pytest.mark.parametrize("transpose", [False, True])
def test_shifted_operator_matches_kronecker_unit(mpg, orc, gen, emode, sigma, transpose):
    n = 57
    a = gen.random_sparse(n, n, 0.2, 11, -4.0)
    if emode == "ident":
        e = None
    elif emode == "diag":
        e = gen.from_triplets(n, n, np.arange(n), np.arange(n), 1.0 + np.arange(n) / n)
    elif emode == "samepat":
        e = gen.HostCsr(a.nrows, a.ncols, a.rowptr, a.colind, np.abs(a.val) + 0.5)
    else:
        e = gen.random_sparse(n, n, 0.1, 12, 2.0)
    A, Ao = _pair(gen, a)
    E, Eo = _pair(gen, e) if e is not None else (None, None)
    op = mpg.ShiftedOperator(A, E)
    w = 2 if complex(sigma).imag != 0 else 1
    x = gen.random_dense(n * w, 1, 5)[:, 0]
    got = op.apply(sigma, x, transpose)
    if transpose:
        Ao, Eo = Ao.transpose(), (Eo.transpose() if Eo is not None else None)
    want = orc.kron_apply(orc.shifted(sigma), Ao, Eo, x)
    assert rel(got, want) <= 1e-13
    # explicit unit matrix == the reference's assemble_explicit block
    ex = op.explicit(sigma, transpose).to_dense()
    exo = orc.kron_assemble(orc.shifted(sigma), Ao, Eo, cap=10**9).to_dense()
    assert np.linalg.norm(ex - exo) <= 1e-13 * np.linalg.norm(exo)


def test_chain_apply_equals_factor_product(mpg, orc, gen):
    base = gen.random_sparse(8, 8, 0.5, 33)
    g, o = _pair(gen, base)
    prod = base.to_dense()
    gc, oc = mpg.PrecondChain(g), orc.Chain(o)
    keep = []
    for k in range(3):
        q = gen.random_sparse(8, 8, 0.5, 40 + k)
        gq, oq = _pair(gen, q)
        keep.append(gq)
        prod = q.to_dense() @ prod
        gc, oc = gc.extended(gq), oc.extended(oq)
    for t in range(4):
        v = gen.random_dense(8, 1, 50 + t)[:, 0]
        assert rel(gc.apply(v), prod @ v) <= 1e-12
        assert rel(gc.apply(v), oc.apply(v)) <= 1e-13


def test_chain_prefix_sharing(mpg, gen):
    b = mpg.SparseMatrix.from_csr(*[getattr(gen.random_sparse(6, 6, 0.5, 63), k) for k in
                                    ("nrows", "ncols", "rowptr", "colind", "val")])
    c1 = mpg.PrecondChain(b).extended(mpg.SparseMatrix.identity(6))
    c2 = c1.extended(mpg.SparseMatrix.identity(6))
    c3 = c1.extended(mpg.SparseMatrix.identity(6))
    assert (c1.length(), c2.length(), c3.length()) == (1, 2, 2)
    assert c2.factor_id(1) == c1.factor_id(1) == c3.factor_id(1)


@pytest.mark.parametrize("seed,n,dens,shift", [(25, 30, 0.25, 4.0), (35, 18, 0.3, 3.0), (45, 16, 0.3, 2.5),
                                               (7, 120, 0.05, 3.0)])
def test_spai_build_matches_oracle(mpg, orc, gen, seed, n, dens, shift):
    h = gen.random_sparse(n, n, dens, seed, shift)
    g, o = _pair(gen, h)
    for cfg_kw in ({}, dict(fill_tol=1e-2, max_pattern_sweeps=6), dict(pattern="diagonal"),
                   dict(pattern="a_pow", power=2), dict(pattern="a_pow", power=3, max_fill_per_col=24)):
        gr = mpg.spai_build(g, mpg.SpaiConfig(**cfg_kw))
        op_, ores, ofb, _ = orc.spai_build(o, orc.SpaiConfig(**cfg_kw))
        assert gr.fallback_count == ofb
        assert np.array_equal(gr.p.download()[0], op_.export()[0])
        assert np.array_equal(gr.p.download()[1], op_.export()[1])
        assert rel(gr.p.download()[2], op_.export()[2]) <= 1e-10
        assert np.allclose(gr.column_residuals, ores, rtol=1e-10, atol=1e-13)  # exact fits sit at rounding level


def test_spai_known_answers(mpg, gen):
    a = mpg.SparseMatrix.identity(4)
    r = mpg.spai_build(a)
    assert np.linalg.norm(np.eye(4) - r.p.to_dense()) == 0.0 and r.fallback_count == 0
    d = mpg.SparseMatrix.diagonal([2.0, 4.0])
    p = mpg.spai_build(d, mpg.SpaiConfig(pattern="diagonal")).p.to_dense()
    assert p[0, 0] == pytest.approx(0.5) and p[1, 1] == pytest.approx(0.25) and p[0, 1] == 0.0
    # structurally singular column falls back to the unit column (test_spai.cpp:200-209)
    s = mpg.SparseMatrix.from_csr(3, 3, [0, 1, 1, 2], [0, 2], [1.0, 1.0])
    r = mpg.spai_build(s)
    assert r.fallback_count == 1 and r.p.to_dense()[1, 1] == 1.0
    assert r.column_residuals[1] == pytest.approx(1.0)


@pytest.mark.parametrize("trial", range(4))
def test_update_build_matches_oracle(mpg, orc, gen, trial):
    prev = gen.random_sparse(12, 12, 0.3, 100 + trial, 3.0)
    new = gen.random_sparse(12, 12, 0.3, 200 + trial, 3.0)
    gp, op_ = _pair(gen, prev)
    gn, on = _pair(gen, new)
    f = mpg.update_build(gp, gn)
    q, mr, mc, fb, _ = orc.update_build(op_, on)
    assert np.array_equal(f.q.download()[1], q.export()[1])
    assert rel(f.q.download()[2], q.export()[2]) <= 1e-10
    assert f.min_residual == pytest.approx(mr, rel=1e-10)
    assert f.matrix_change == pytest.approx(mc, rel=1e-12)
    assert f.min_residual <= f.matrix_change * (1 + 1e-12)


def test_update_identity_and_rescale(mpg, gen):
    a = gen.random_sparse(6, 6, 0.5, 3, 4.0)
    g = mpg.SparseMatrix.from_csr(a.nrows, a.ncols, a.rowptr, a.colind, a.val)
    f = mpg.update_build(g, g)
    assert f.matrix_change == 0.0 and f.min_residual <= 1e-12
    assert np.linalg.norm(f.q.to_dense() - np.eye(6)) <= 1e-12
    f = mpg.update_build(mpg.SparseMatrix.identity(3), mpg.SparseMatrix.diagonal([2.0, 2.0, 2.0]))
    assert np.linalg.norm(f.q.to_dense() - 0.5 * np.eye(3)) <= 1e-14


def test_spai_column_solve(mpg, orc, gen):
    h = gen.random_sparse(7, 7, 0.6, 15, 3.0)
    g, o = _pair(gen, h)
    full = list(range(7))
    for j in range(7):
        rows, vals, res, rd = mpg.spai_column_solve(g, j, full)
        r2, v2, res2, rd2 = orc.spai_column_solve(o, j, full)
        assert rel(vals, v2) <= 1e-10 and res == pytest.approx(res2, abs=1e-12) and rd == rd2


@pytest.mark.parametrize("case", ["random", "c1_chain", "c3_pair"])
def test_standard_residual_matches_oracle(mpg, orc, gen, case):
    """standard_residual (chain.cpp:140-157): ||I - A P||_F / sqrt(n) by n probes,
    P the whole chain -- the GPU value against the oracle's on the same matrices:
    a random sparse matrix with its SPAI, a C1 operator with a fresh SPAI plus
    two update factors, and a C3 complex-pair (2n) unit with its SPAI."""
    if case == "random":
        h = gen.random_sparse(40, 40, 0.15, 7, 4.0)
        g, o = _pair(gen, h)
        gch = mpg.PrecondChain(mpg.spai_build(g).p)
        och = orc.Chain(orc.spai_build(o)[0])
    elif case == "c1_chain":
        s = gen.config1(N=14)
        ec = s.e_csr()
        A, E = orc.Csr.of(s.a), orc.Csr.of(ec)
        op = mpg.ShiftedOperator(_pair(gen, s.a)[0], _pair(gen, ec)[0])
        mats_g = [op.explicit(x) for x in (0.1, 0.3, 0.9)]
        mats_o = [orc.kron_assemble(orc.shifted(x), A, E, cap=10 ** 9) for x in (0.1, 0.3, 0.9)]
        gch = mpg.PrecondChain(mpg.spai_build(mats_g[0]).p)
        och = orc.Chain(orc.spai_build(mats_o[0])[0])
        for i in (1, 2):
            gch = gch.extended(mpg.update_build(mats_g[i - 1], mats_g[i]))
            och = och.extended(orc.update_build(mats_o[i - 1], mats_o[i])[0])
        g, o = mats_g[2], mats_o[2]
    else:
        s = gen.config3(6)
        op = mpg.ShiftedOperator(_pair(gen, s.a)[0], _pair(gen, s.e)[0])
        g = op.explicit(complex(0.7, 0.4))
        o = orc.kron_assemble(orc.shifted(complex(0.7, 0.4)), orc.Csr.of(s.a), orc.Csr.of(s.e), cap=10 ** 9)
        gch = mpg.PrecondChain(mpg.spai_build(g).p)
        och = orc.Chain(orc.spai_build(o)[0])
    gv = mpg.standard_residual(g, gch)
    ov = orc.standard_residual(o, och)
    assert ov > 0 and abs(gv - ov) <= 1e-10 * ov, (gv, ov)


@pytest.mark.parametrize("power,fill", [(2, 50), (3, 50), (2, 12)])
def test_spai_a_pow_pattern_on_fem_matches_oracle(mpg, orc, gen, power, fill):
    """PatternOfAPow (spai.cpp:55-85) on a C3-type operator (27-point rows, so
    the A^2 support of a column passes max_fill_per_col and is truncated to the
    lowest indices with the diagonal kept): pattern bitwise, values 1e-10."""
    s = gen.config3(7)
    op = mpg.ShiftedOperator(_pair(gen, s.a)[0], _pair(gen, s.e)[0])
    g = op.explicit(0.3)
    o = orc.kron_assemble(orc.shifted(0.3), orc.Csr.of(s.a), orc.Csr.of(s.e), cap=10 ** 9)
    kw = dict(pattern="a_pow", power=power, max_fill_per_col=fill)
    gr = mpg.spai_build(g, mpg.SpaiConfig(**kw))
    op_, ores, ofb, _ = orc.spai_build(o, orc.SpaiConfig(**kw))
    assert gr.fallback_count == ofb
    assert np.array_equal(gr.p.download()[0], op_.export()[0])
    assert np.array_equal(gr.p.download()[1], op_.export()[1])
    assert rel(gr.p.download()[2], op_.export()[2]) <= 1e-10
    assert np.allclose(gr.column_residuals, ores, rtol=1e-10, atol=1e-13)
