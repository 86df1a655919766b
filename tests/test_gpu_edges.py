"""GPU edge cases: ragged rows (empty rows next to a dense row), 1 x 1 systems,
an empty solve batch, and a ragged SPAI / preconditioned solve, each against the
oracle (sparse.cpp:236-269, spai.cpp:16-238, gmres.cpp:40-186)."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _pair(gen, host):
    import oracle as O
    from paper_2003_12759_b200 import SparseMatrix
    return SparseMatrix.from_csr(host.nrows, host.ncols, host.rowptr, host.colind, host.val), O.Csr.of(host)


def _ragged(gen, n, seed, empty_rows=True, diag=0.0):
    """Row 0 dense, every 7th row empty (unless `diag`), the rest 1-3 entries;
    column 0 dense with small values when `diag` is set (an arrow matrix)."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for j in range(n):
        rows.append(0); cols.append(j); vals.append(rng.uniform(-1, 1))
    for i in range(1, n):
        if empty_rows and i % 7 == 0:
            continue
        for j in rng.choice(n, size=int(rng.integers(1, 4)), replace=False):
            rows.append(i); cols.append(int(j)); vals.append(rng.uniform(-1, 1))
        if diag:
            rows.append(i); cols.append(i); vals.append(diag)
            rows.append(i); cols.append(0); vals.append(0.01 * rng.uniform(-1, 1))
    if diag:
        rows.append(0); cols.append(0); vals.append(diag * n)
    return gen.from_triplets(n, n, np.array(rows), np.array(cols), np.array(vals))


@pytest.mark.parametrize("n", [1, 9, 700, 5000])
def test_ragged_spmv_and_transpose(mpg, orc, gen, n):
    h = _ragged(gen, n, 40 + n)
    g, o = _pair(gen, h)
    x = gen.random_dense(n, 1, 60 + n)[:, 0]
    assert rel(g.multiply(x), o.multiply(x)) <= 1e-13
    assert rel(g.multiply_transpose(x), o.multiply_transpose(x)) <= 1e-13
    rp, ci, v = g.transpose().download()
    rp2, ci2, v2 = o.transpose().export()
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2)


@pytest.mark.parametrize("sigma", [0.5, 2.0 - 1.0j])
@pytest.mark.parametrize("transpose", [False, True])
def test_ragged_shifted_operator(mpg, orc, gen, sigma, transpose):
    n = 400
    a, e = _ragged(gen, n, 3), _ragged(gen, n, 4)
    (A, Ao), (E, Eo) = _pair(gen, a), _pair(gen, e)
    op = mpg.ShiftedOperator(A, E)
    w = 2 if complex(sigma).imag else 1
    x = gen.random_dense(n * w, 1, 5)[:, 0]
    if transpose:
        Ao, Eo = Ao.transpose(), Eo.transpose()
    assert rel(op.apply(sigma, x, transpose), orc.kron_apply(orc.shifted(sigma), Ao, Eo, x)) <= 1e-13


def test_ragged_spai_and_solve_match_oracle(mpg, orc, gen):
    n = 90
    h = _ragged(gen, n, 8, empty_rows=False, diag=4.0)
    g, o = _pair(gen, h)
    gr = mpg.spai_build(g)
    op_, ores, ofb, _ = orc.spai_build(o)
    assert gr.fallback_count == ofb
    assert np.array_equal(gr.p.download()[0], op_.export()[0])
    assert np.array_equal(gr.p.download()[1], op_.export()[1])
    assert rel(gr.p.download()[2], op_.export()[2]) <= 1e-10
    assert rel(gr.column_residuals, ores) <= 1e-10
    b = gen.random_dense(n, 1, 9)[:, 0]
    cfg = mpg.GmresConfig(rel_tol=1e-10)
    res = mpg.gmres_right_preconditioned(g, mpg.PrecondChain(gr.p), b, cfg)
    assert res.report.converged
    assert np.linalg.norm(h.to_dense() @ res.x - b) <= 1e-9 * np.linalg.norm(b)
    assert rel(res.x, np.linalg.solve(h.to_dense(), b)) <= 1e-8


def test_one_by_one_system(mpg, orc, gen):
    g = mpg.SparseMatrix.from_csr(1, 1, [0, 1], [0], [4.0])
    assert mpg.spai_build(g).p.to_dense()[0, 0] == pytest.approx(0.25)
    res = mpg.gmres_right_preconditioned(g, None, np.array([2.0]))
    assert res.report.converged and res.report.iterations == 1 and res.x[0] == pytest.approx(0.5)
    op = mpg.ShiftedOperator(g, None)
    r = mpg.gmres_shifted(op, 6.0, np.array([1.0]), None, False, mpg.GmresConfig())
    assert r.report.converged and r.x[0] == pytest.approx(0.5)  # (6 - 4) x = 1


def test_empty_batch(mpg, gen):
    sysm = gen.config1(N=8)
    op = mpg.ShiftedOperator(mpg.SparseMatrix.from_csr(sysm.a.nrows, sysm.a.ncols, sysm.a.rowptr, sysm.a.colind,
                                                       sysm.a.val), None)
    assert mpg.gmres_batch(op, [], []) == []


@pytest.mark.parametrize("n", [3000, 60000])
def test_zipf_rows_spmv_and_shifted_operator(mpg, orc, gen, n):
    """C5-type rows (Zipf(1.8) lengths 3 ... 2 000): the row-binned kernels
    (runtime.cuh row bins: sub-warps of 2 ... 32 lanes by row length) against
    the oracle (sparse.cpp:236-269, kron.cpp:34-64), both sides, real and pair."""
    s = gen.config5(n=n, max_len=2000)
    (A, Ao), (E, Eo) = _pair(gen, s.a), _pair(gen, s.e_csr())
    x = gen.random_dense(n, 1, 70)[:, 0]
    assert rel(A.multiply(x), Ao.multiply(x)) <= 1e-13
    assert rel(A.multiply_transpose(x), Ao.multiply_transpose(x)) <= 1e-13
    op = mpg.ShiftedOperator(A, E)
    for sigma in (0.3, 1.5 + 0.7j):
        xx = gen.random_dense(n * (2 if complex(sigma).imag else 1), 1, 71)[:, 0]
        for transpose in (False, True):
            ao, eo = (Ao.transpose(), Eo.transpose()) if transpose else (Ao, Eo)
            assert rel(op.apply(sigma, xx, transpose), orc.kron_apply(orc.shifted(sigma), ao, eo, xx)) <= 1e-13
