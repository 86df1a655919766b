"""GPU GMRES: the reference's gmres tests (proj/tests/test_gmres.cpp) on the
device engine, plus parity with the oracle on shifted preconditioned solves."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _m(mpg, h):
    return mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)


def test_identity_converges_in_one_iteration(mpg):
    res = mpg.gmres_right_preconditioned(mpg.SparseMatrix.identity(2), None, np.array([3.0, 4.0]))
    assert res.report.converged and res.report.iterations == 1
    assert np.linalg.norm(res.x - [3, 4]) <= 1e-12


def test_diagonal_solve(mpg):
    res = mpg.gmres_right_preconditioned(mpg.SparseMatrix.diagonal([2.0, 3.0]), None, np.array([2.0, 3.0]))
    assert res.report.converged and np.linalg.norm(res.x - 1.0) <= 1e-10


def test_exact_inverse_preconditioner(mpg, gen):
    h = gen.random_sparse(10, 10, 0.5, 7, 8.0)
    a = _m(mpg, h)
    inv = mpg.SparseMatrix.from_dense(np.linalg.inv(h.to_dense()))
    b = gen.random_dense(10, 1, 8)[:, 0]
    res = mpg.gmres_right_preconditioned(a, mpg.PrecondChain(inv), b)
    assert res.report.converged and res.report.iterations == 1
    assert np.linalg.norm(h.to_dense() @ res.x - b) <= 1e-6 * np.linalg.norm(b)


def test_zero_operator_reports_breakdown(mpg):
    res = mpg.gmres_right_preconditioned(mpg.SparseMatrix.zero(3, 3), None, np.array([1.0, 0, 0]))
    assert res.report.breakdown and not res.report.converged


def test_zero_rhs_rejected(mpg):
    with pytest.raises(ValueError):
        mpg.gmres_right_preconditioned(mpg.SparseMatrix.identity(2), None, np.zeros(2))


def test_history_nonincreasing(mpg, gen):
    h = gen.random_sparse(30, 30, 0.2, 17, 4.0)
    res = mpg.gmres_right_preconditioned(_m(mpg, h), None, gen.random_dense(30, 1, 18)[:, 0],
                                         mpg.GmresConfig(record_history=True))
    assert res.report.converged
    hist = res.report.residual_history
    assert len(hist) >= 2
    assert all(hist[i] <= hist[i - 1] * (1 + 1e-14) for i in range(1, len(hist)))


def test_solution_in_unpreconditioned_variable(mpg, gen):
    h = gen.random_sparse(12, 12, 0.4, 27, 5.0)
    p = mpg.SparseMatrix.diagonal(1.0 + 0.3 * np.arange(12))
    b = gen.random_dense(12, 1, 28)[:, 0]
    cfg = mpg.GmresConfig(rel_tol=1e-8)
    res = mpg.gmres_right_preconditioned(_m(mpg, h), mpg.PrecondChain(p), b, cfg)
    assert res.report.converged
    assert np.linalg.norm(h.to_dense() @ res.x - b) <= 1e-8 * np.linalg.norm(b)
    assert res.report.final_residual <= 1e-8 * np.linalg.norm(b)


def test_preconditioned_and_plain_agree(mpg, gen):
    h = gen.random_sparse(15, 15, 0.4, 37, 6.0)
    b = gen.random_dense(15, 1, 38)[:, 0]
    cfg = mpg.GmresConfig(rel_tol=1e-12)
    plain = mpg.gmres_right_preconditioned(_m(mpg, h), None, b, cfg)
    pre = mpg.gmres_right_preconditioned(_m(mpg, h), mpg.PrecondChain(mpg.SparseMatrix.diagonal(np.full(15, 0.5))),
                                         b, cfg)
    assert plain.report.converged and pre.report.converged
    assert np.linalg.norm(plain.x - pre.x) <= 1e-8 * (1 + np.linalg.norm(plain.x))


def test_iteration_cap_reported(mpg, gen):
    h = gen.random_sparse(40, 40, 0.3, 47, 3.0)
    res = mpg.gmres_right_preconditioned(_m(mpg, h), None, gen.random_dense(40, 1, 48)[:, 0],
                                         mpg.GmresConfig(rel_tol=1e-14, max_iter=2))
    assert not res.report.converged and res.report.iterations == 2 and res.x.size == 40


def test_final_residual_matches_recomputation(mpg, gen):
    h = gen.random_sparse(20, 20, 0.4, 57, 5.0)
    b = gen.random_dense(20, 1, 58)[:, 0]
    res = mpg.gmres_right_preconditioned(_m(mpg, h), None, b)
    direct = np.linalg.norm(b - h.to_dense() @ res.x)
    assert res.report.final_residual == pytest.approx(direct, rel=1e-10)


@pytest.mark.parametrize("sigma", [0.5, 20.0, 3.0 + 2.0j])
@pytest.mark.parametrize("transpose", [False, True])
def test_shifted_spai_solve_matches_oracle(mpg, orc, gen, sigma, transpose):
    sysm = gen.config1(N=24)
    A = _m(mpg, sysm.a)
    ecsr = sysm.e_csr()
    E = _m(mpg, ecsr)
    op = mpg.ShiftedOperator(A, E)
    Ao, Eo = orc.Csr.of(sysm.a), orc.Csr.of(ecsr)
    if transpose:
        Ao, Eo = Ao.transpose(), Eo.transpose()
    w = 2 if complex(sigma).imag else 1
    b = np.tile(sysm.b[:, 0], w)
    M = op.explicit(sigma, transpose)
    P = mpg.spai_build(M).p
    cfg = mpg.GmresConfig(rel_tol=1e-8)
    res = mpg.gmres_shifted(op, sigma, b, mpg.PrecondChain(P), transpose, cfg)
    Mo = orc.kron_assemble(orc.shifted(sigma), Ao, Eo, cap=10**9)
    Po = orc.spai_build(Mo)[0]
    xo, ro = orc.gmres_kron(orc.shifted(sigma), Ao, Eo, orc.Chain(Po), b, orc.GmresConfig(1e-8))
    assert res.report.converged and ro.converged
    assert res.report.final_residual <= 1e-8 * np.linalg.norm(b)
    assert rel(res.x, xo) <= 1e-6
    assert abs(res.report.iterations - ro.iterations) <= max(2, 0.1 * ro.iterations)


def test_batch_equals_single_solves(mpg, gen):
    sysm = gen.config1(N=20)
    op = mpg.ShiftedOperator(_m(mpg, sysm.a), _m(mpg, sysm.e_csr()))
    sig = [0.01, 0.3, 5.0, 2.0 + 1.0j]
    bs = [np.tile(sysm.b[:, 0], 2 if complex(s).imag else 1) for s in sig]
    cfg = mpg.GmresConfig(rel_tol=1e-9)
    batch = mpg.gmres_batch(op, sig, bs, transposes=[0, 1, 0, 1], cfg=cfg)
    for s, b, t, r in zip(sig, bs, [0, 1, 0, 1], batch):
        single = mpg.gmres_shifted(op, s, b, None, bool(t), cfg)
        assert r.report.converged
        assert r.report.iterations == single.report.iterations
        assert rel(r.x, single.x) <= 1e-12


@pytest.mark.parametrize("n,maxit", [(300, 1000), (700, 1000), (1500, 1000), (2600, 2000)])
def test_long_krylov_runs_match_oracle(mpg, orc, gen, n, maxit):
    """251 / 490 / 882 / ~1300 iterations: exercises every Gram-Schmidt tile
    shape (k+1 up to 2048) and the measured second pass."""
    d = 1.0 + np.arange(n) ** 1.5  # spectrum [1, n^1.5]
    h = gen.from_triplets(n, n, np.arange(n), np.arange(n), d)
    b = gen.random_dense(n, 1, 5)[:, 0]
    cfg = mpg.GmresConfig(rel_tol=1e-10, max_iter=maxit)
    g = mpg.gmres_right_preconditioned(_m(mpg, h), None, b, cfg)
    xo, ro = orc.gmres_csr(orc.Csr.of(h), None, b, orc.GmresConfig(1e-10, maxit))
    assert ro.converged and g.report.converged, (g.report.iterations, ro.iterations)
    assert abs(g.report.iterations - ro.iterations) <= max(3, 0.03 * ro.iterations)
    assert np.linalg.norm(d * g.x - b) <= 1e-10 * np.linalg.norm(b)
    assert rel(g.x, xo) <= 1e-6


def test_large_batch_with_shared_preconditioners_matches_single(mpg, gen):
    """24 solves in one batch (more than the 8-wide shared-matrix groups and than
    SMs per solve): primal/dual sides sharing one frozen SPAI each (interleaved
    multi-RHS SpMVs), complex pairs, and solves finishing at different
    iterations; every solve equals its single-solve run."""
    sysm = gen.config1(N=24)
    op = mpg.ShiftedOperator(_m(mpg, sysm.a), _m(mpg, sysm.e_csr()))
    pv = mpg.PrecondChain(mpg.spai_build(op.explicit(0.05, False)).p)
    pw = mpg.PrecondChain(mpg.spai_build(op.explicit(0.05, True)).p)
    sig, trs, chains, bs = [], [], [], []
    for i in range(24):
        s = float(np.logspace(-2, 2, 24)[i]) + (1j * 3.0 if i % 7 == 3 else 0.0)
        t = i % 2
        sig.append(s)
        trs.append(t)
        chains.append(None if (i % 7 == 3) else (pw if t else pv))
        bs.append(np.tile(sysm.b[:, 0] * (1 + 0.1 * i), 2 if complex(s).imag else 1))
    cfg = mpg.GmresConfig(rel_tol=1e-9)
    batch = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)
    for s, b, t, ch, r in zip(sig, bs, trs, chains, batch):
        single = mpg.gmres_shifted(op, s, b, ch, bool(t), cfg)
        assert r.report.converged and single.report.converged
        assert abs(r.report.iterations - single.report.iterations) <= 1
        assert rel(r.x, single.x) <= 1e-8


def test_unfused_gram_schmidt_path_beyond_2047_max_iter(mpg, orc, gen):
    """max_iter > 2047 selects the unfused dot / update kernels; the answer and
    iteration count still match the oracle."""
    n = 600
    d = 1.0 + np.arange(n) ** 1.5
    h = gen.from_triplets(n, n, np.arange(n), np.arange(n), d)
    b = gen.random_dense(n, 1, 9)[:, 0]
    g = mpg.gmres_right_preconditioned(_m(mpg, h), None, b, mpg.GmresConfig(rel_tol=1e-10, max_iter=2100))
    xo, ro = orc.gmres_csr(orc.Csr.of(h), None, b, orc.GmresConfig(1e-10, 2100))
    assert g.report.converged and ro.converged
    assert abs(g.report.iterations - ro.iterations) <= max(3, 0.03 * ro.iterations)
    assert rel(g.x, xo) <= 1e-6


@pytest.mark.parametrize("env", [{"MPG_GS_UPD": "reg"}, {"MPG_GS_UPD": "tma"}, {"MPG_GS_UPD": "tmx"},
                                 {"MPG_GS_SPLIT": "28"}, {"MPG_GS_LOW": "0"}, {"MPG_GS_DOT": "reg"},
                                 {"MPG_GS_DOT_SPLIT": "64"}])
def test_gram_schmidt_kernel_variants_agree(mpg, gen, monkeypatch, env):
    """Every update / projection kernel choice (register-tiled, 1-D bulk TMA, swizzled tensor TMA with each
    register-tile size, and the split points between them) gives the default run's answer on a 490-iteration
    solve that walks k + 1 through all of their ranges."""
    n = 700
    d = 1.0 + np.arange(n) ** 1.5
    h = gen.from_triplets(n, n, np.arange(n), np.arange(n), d)
    b = gen.random_dense(n, 1, 5)[:, 0]
    cfg = mpg.GmresConfig(rel_tol=1e-10, max_iter=1000)
    base = mpg.gmres_right_preconditioned(_m(mpg, h), None, b, cfg)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = mpg.gmres_right_preconditioned(_m(mpg, h), None, b, cfg)
    assert g.report.converged and abs(g.report.iterations - base.report.iterations) <= 1
    assert rel(g.x, base.x) <= 1e-8
    assert np.linalg.norm(d * g.x - b) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("cfgname", ["c3", "c2", "c5"])
def test_halo_sell_spmv_matches_csr_kernels(mpg, gen, monkeypatch, cfgname):
    """The run-mode multi-RHS SpMVs in the SELL-8 layout (the default) and the
    halo-staged sliced-ELL layout (MPG_SPMV_HALO; 27-point FEM with E sharing A's
    pattern, 7-point with diagonal E) give the CSR kernels' solves (MPG_SPMV_CSR)
    on 8-solve groups of both sides; on a
    Zipf(1.8) pattern with rows up to 600 entries (blocks past HALO_MAXNZ) the
    layout is declined and the CSR kernels run."""
    if cfgname == "c3":
        s = gen.config3(20)
    elif cfgname == "c2":
        s = gen.config2(M=24)
    else:
        s = gen.config5(n=6000, max_len=600)
    ec = s.e_csr()
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, ec))
    sig0 = 0.5 if cfgname != "c5" else 1.0
    pv = mpg.PrecondChain(mpg.spai_build(op.explicit(sig0, False)).p)
    pw = mpg.PrecondChain(mpg.spai_build(op.explicit(sig0, True)).p)
    sig = [float(x) for x in np.logspace(-2, 1, 8)] * 2
    trs = [0] * 8 + [1] * 8
    chains = [pv] * 8 + [pw] * 8
    bs = [s.b[:, 0] * (1 + 0.1 * i) for i in range(8)] + [s.c[:, 0] * (1 + 0.1 * i) for i in range(8)]
    cfg = mpg.GmresConfig(rel_tol=1e-10)
    sell = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)  # default: SELL-8
    monkeypatch.setenv("MPG_SPMV_CSR", "1")
    csr = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)
    monkeypatch.delenv("MPG_SPMV_CSR")
    monkeypatch.setenv("MPG_SPMV_HALO", "1")
    halo = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)
    for h, c, sl in zip(halo, csr, sell):
        assert h.report.converged and c.report.converged and sl.report.converged
        assert abs(h.report.iterations - c.report.iterations) <= 1
        assert abs(sl.report.iterations - c.report.iterations) <= 1
        assert rel(h.x, c.x) <= 1e-8 and rel(sl.x, c.x) <= 1e-8
    if cfgname == "c5":
        # irregular rows: the runs above took the row-binned interleaved kernel (k_spmv_il2b: 4 ... 32 lanes per
        # row by length class); with MPG_IL_BINS=0 the fixed four lanes per row give the same solves
        monkeypatch.delenv("MPG_SPMV_HALO")
        monkeypatch.setenv("MPG_IL_BINS", "0")
        fixed = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)
        for f4, sl in zip(fixed, sell):
            assert f4.report.converged
            assert abs(f4.report.iterations - sl.report.iterations) <= 1
            assert rel(f4.x, sl.x) <= 1e-8


@pytest.mark.parametrize("cfgname", ["c3", "c2"])
def test_narrow_interleave_for_the_last_running_columns(mpg, gen, monkeypatch, cfgname):
    """Solves of one 8-column group that finish at very different iterations: once four or fewer are still
    running the group switches to the 4-column interleave (one right-hand side per lane, 32-byte x-gathers).
    Per column the arithmetic is that of the 8-column kernels, so the solves agree with MPG_NO_IL_NARROW to
    rounding and take the same iterations; a complex pair keeps the group wide while it runs."""
    s = gen.config3(20) if cfgname == "c3" else gen.config2(M=24)
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e_csr()))
    pv = mpg.PrecondChain(mpg.spai_build(op.explicit(0.5, False)).p)
    pw = mpg.PrecondChain(mpg.spai_build(op.explicit(0.5, True)).p)
    side = [0.5, 0.6, 1.5, 5.0, 20.0, 80.0, 30.0 + 9.0j]
    sig, trs, chains, bs = side * 2, [0] * 7 + [1] * 7, [pv] * 7 + [pw] * 7, []
    for i, z in enumerate(sig):
        v = (s.b if i < 7 else s.c)[:, 0] * (1 + 0.1 * i)
        bs.append(np.concatenate([v, 0.3 * v[::-1]]) if complex(z).imag else v)
    cfg = mpg.GmresConfig(rel_tol=1e-10)
    narrow = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)
    monkeypatch.setenv("MPG_NO_IL_NARROW", "1")
    wide = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)
    its = [r.report.iterations for r in wide]
    assert len(set(its[:6])) >= 3  # the columns drop out one after the other
    for a, b in zip(narrow, wide):
        assert a.report.converged and b.report.converged
        assert a.report.iterations == b.report.iterations
        assert rel(a.x, b.x) <= 1e-12


@pytest.mark.parametrize("cfgname", ["c3", "c2"])
def test_complex_pairs_ride_in_interleaved_groups(mpg, gen, monkeypatch, cfgname):
    """Per side 4 real shifts and 2 complex pairs sharing one frozen n x n SPAI (the C3 IRKA's unit mix from
    sweep 3 on): the pairs occupy two columns each of the side's interleaved 8-column group (block-diagonal
    preconditioner, 2 x 2 coupling in the operator epilogue, kron.cpp:34-64 pair form) and give the solves of
    the separate pair kernels (MPG_NO_IL_PAIRS); the profiled chain bytes show the factor is no longer read
    per pair."""
    s = gen.config3(20) if cfgname == "c3" else gen.config2(M=24)
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e_csr()))
    pv = mpg.PrecondChain(mpg.spai_build(op.explicit(0.5, False)).p)
    pw = mpg.PrecondChain(mpg.spai_build(op.explicit(0.5, True)).p)
    side = [0.05, 0.4, 2.0, 9.0, 3.0 + 2.0j, 40.0 - 15.0j]
    sig, trs, chains, bs = side * 2, [0] * 6 + [1] * 6, [pv] * 6 + [pw] * 6, []
    for i, z in enumerate(sig):
        v = (s.b if i < 6 else s.c)[:, 0] * (1 + 0.1 * i)
        bs.append(np.concatenate([v, 0.3 * v[::-1]]) if complex(z).imag else v)
    cfg = mpg.GmresConfig(rel_tol=1e-10)

    def run():
        mpg.profile_enable(True)
        out = mpg.gmres_batch(op, sig, bs, chains=chains, transposes=trs, cfg=cfg)
        prof = mpg.profile_read()
        mpg.profile_enable(False)
        return out, prof["chain_spmv"]["bytes"]

    riding, bytes_riding = run()
    monkeypatch.setenv("MPG_NO_IL_PAIRS", "1")
    apart, bytes_apart = run()
    for a, b in zip(riding, apart):
        assert a.report.converged and b.report.converged
        assert abs(a.report.iterations - b.report.iterations) <= 1
        assert rel(a.x, b.x) <= 1e-8
    assert bytes_riding < 0.8 * bytes_apart


@pytest.mark.parametrize("env", [{"MPG_DCGS2": "0"}, {"MPG_GS_DOT_SPLIT": "64"}, {"MPG_GS_DOT_SPLIT": "300"}])
def test_delayed_second_pass_matches_immediate(mpg, orc, gen, monkeypatch, env):
    """The delayed (DCGS2-style) second Gram-Schmidt pass gives the immediate
    pass's solves: the same second-pass decisions (reorth_passes), iterations
    within 1, solutions within 1e-9 -- on a C3-type batch (16 solves sharing two
    frozen SPAIs, 150-300 iterations, the projection in k_gs_tmx<true> from
    k + 1 = 129 on). Every variant also stays within the oracle's iteration count."""
    monkeypatch.setenv("MPG_GS_F32", "0")  # the fp64 projection: the second-pass decisions are comparable
    s = gen.config3(18)
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e))
    sh = [float(x) for x in s.shifts[:8]]
    pv = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], False)).p)
    pw = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], True)).p)
    sig, trs, ch = sh + sh, [0] * 8 + [1] * 8, [pv] * 8 + [pw] * 8
    bs = [s.b[:, 0]] * 8 + [s.c[:, 0]] * 8
    cfg = mpg.GmresConfig(rel_tol=1e-10, max_iter=1000)
    base = mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    var = mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
    assert sum(r.report.reorth_passes for r in base) > 0
    for b, r in zip(base, var):
        assert b.report.converged and r.report.converged
        assert abs(b.report.iterations - r.report.iterations) <= 1
        assert abs(b.report.reorth_passes - r.report.reorth_passes) <= 1
        assert rel(r.x, b.x) <= 1e-9
    # against the oracle (the reference's MGS + measured second pass), solve 0
    A, E = orc.Csr.of(s.a), orc.Csr.of(s.e)
    m = orc.kron_assemble(orc.shifted(sh[0]), A, E, cap=10 ** 12)
    xo, ro = orc.gmres_kron(orc.shifted(sh[0]), A, E, orc.Chain(orc.spai_build(m)[0]), s.b[:, 0],
                            orc.GmresConfig(1e-10, 1000))
    assert abs(var[0].report.iterations - ro.iterations) <= max(3, 0.03 * ro.iterations)
    assert rel(var[0].x, xo) <= 1e-6


@pytest.mark.parametrize("tol", [1e-8, 1e-12])
def test_float_shadow_projection_matches_fp64_projection(mpg, orc, gen, monkeypatch, tol):
    """k_gs_tmxf projects on a single-precision shadow of the basis (half the bytes of the pass); the
    update pass, the probe and the delayed correction keep the Arnoldi relation in fp64. Same solves as
    with the fp64 projection: identical iteration counts, solutions within 1e-11, true residuals at the
    tolerance (also at 1e-12, far below single precision), and within the oracle's iteration count."""
    monkeypatch.setenv("MPG_GS_DOT_SPLIT", "32")  # both variants: k_gs_tmx<true> / k_gs_tmxf from k + 1 = 33 on
    s = gen.config3(40)
    op = mpg.ShiftedOperator(_m(mpg, s.a), _m(mpg, s.e))
    sh = [float(x) for x in s.shifts[:8]]
    pv = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], False)).p)
    pw = mpg.PrecondChain(mpg.spai_build(op.explicit(sh[0], True)).p)
    sig, trs, ch = sh + sh, [0] * 8 + [1] * 8, [pv] * 8 + [pw] * 8
    bs = [s.b[:, 0]] * 8 + [s.c[:, 0]] * 8
    cfg = mpg.GmresConfig(rel_tol=tol, max_iter=1000)
    f32 = mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)  # default
    monkeypatch.setenv("MPG_GS_F32", "0")
    f64 = mpg.gmres_batch(op, sig, bs, chains=ch, transposes=trs, cfg=cfg)
    assert min(r.report.iterations for r in f32) > 80
    for i, (a, b) in enumerate(zip(f32, f64)):
        assert a.report.converged and b.report.converged
        assert a.report.iterations == b.report.iterations
        assert rel(a.x, b.x) <= 1e-11
        res = bs[i] - op.apply(sig[i], a.x, transpose=bool(trs[i]))
        assert np.linalg.norm(res) <= 1.0001 * tol * np.linalg.norm(bs[i])
        assert a.report.reorth_passes >= b.report.reorth_passes  # every shadow projection is followed by a correction
    A, E = orc.Csr.of(s.a), orc.Csr.of(s.e)
    m = orc.kron_assemble(orc.shifted(sh[0]), A, E, cap=10 ** 12)
    xo, ro = orc.gmres_kron(orc.shifted(sh[0]), A, E, orc.Chain(orc.spai_build(m)[0]), s.b[:, 0],
                            orc.GmresConfig(tol, 1000))
    assert abs(f32[0].report.iterations - ro.iterations) <= max(3, 0.03 * ro.iterations)
    assert rel(f32[0].x, xo) <= 1e-6
