"""Matrix Market IO and the report CSV: the library's
parallel reader/writer (csrc/host/mmio.cpp, through the C ABI) and the
oracle's sequential istream restatement are both pinned to the reference's
own tests (proj/tests/test_io.cpp, cited per test), then compared with each
other on generated and fuzzed inputs: identical CSR (bitwise) and identical
error messages, line numbers included, for any thread count."""
import io
import random

import numpy as np
import pytest

GEN = "%%MatrixMarket matrix coordinate real general\n"
SYM = "%%MatrixMarket matrix coordinate real symmetric\n"


class Impl:
    def __init__(self, name, mpg, orc, threads=0):
        self.name, self.mpg, self.orc, self.threads = name, mpg, orc, threads

    @property
    def IoError(self):
        return self.orc.IoError if self.name == "oracle" else self.mpg.IoError

    def parse(self, text, origin="test"):
        if self.name == "oracle":
            return self.orc.read_matrix_market(text, origin).to_dense()
        return self.mpg.read_matrix_market(text, origin, self.threads, device=None).to_dense()

    def parse_csr(self, text, origin="test"):
        if self.name == "oracle":
            rp, ci, v = self.orc.read_matrix_market(text, origin).export()
            return np.asarray(rp), np.asarray(ci), np.asarray(v)
        h = self.mpg.read_matrix_market(text, origin, self.threads, device=None)
        return h.rowptr, h.colind, h.val


@pytest.fixture(params=["native", "native1", "native7", "oracle"])
def impl(request, mpg, orc):
    t = {"native": 0, "native1": 1, "native7": 7, "oracle": 0}[request.param]
    return Impl("oracle" if request.param == "oracle" else "native", mpg, orc, t)


def test_write_then_read_is_exact(impl, mpg, orc, gen):  # test_io.cpp:30-39
    a = gen.random_sparse(17, 9, 0.3, 42)
    text = orc.write_matrix_market(orc.Csr.of(a)) if impl.name == "oracle" else mpg.write_matrix_market(a)
    b = impl.parse(text, "roundtrip")
    assert b.shape == (17, 9)
    assert np.array_equal(b, a.to_dense())


def test_dense_write_keeps_shape_and_zeros(impl, mpg):  # test_io.cpp:41-51
    m = np.array([[1.5, 0.0, -2.25], [0.0, 0.0, 1e-300]])
    b = impl.parse(mpg.write_matrix_market(m), "dense")
    assert b.shape == (2, 3) and np.array_equal(b, m)


def test_single_entry(impl):  # :53-61
    a = impl.parse(GEN + "1 1 1\n1 1 5.0\n")
    assert a.shape == (1, 1) and a[0, 0] == 5.0


def test_comments_and_spacing(impl):  # :63-74
    rp, ci, v = impl.parse_csr(GEN + "% produced by hand\n%\n2 2 2\n  1   2   3.5\n2 1 -1.0\n")
    assert rp[-1] == 2
    a = impl.parse(GEN + "% produced by hand\n%\n2 2 2\n  1   2   3.5\n2 1 -1.0\n")
    assert a[0, 1] == 3.5 and a[1, 0] == -1.0


def test_symmetric_expands_lower_triangle(impl):  # :76-89
    a = impl.parse(SYM + "3 3 3\n1 1 2.0\n2 1 7.0\n3 3 1.0\n")
    want = np.zeros((3, 3))
    want[0, 0], want[1, 0], want[0, 1], want[2, 2] = 2.0, 7.0, 7.0, 1.0
    assert np.array_equal(a, want)


def test_symmetric_diagonal_not_doubled(impl):  # :91-97
    assert impl.parse(SYM + "2 2 1\n1 1 3.0\n")[0, 0] == 3.0


def test_duplicates_summed(impl):  # :99-106
    assert impl.parse(GEN + "1 1 2\n1 1 2.0\n1 1 3.0\n")[0, 0] == 5.0


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix array real general\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coodinate real general\n1 x 1\n",
    GEN + "2 2 1\n3 1 1.0\n",
    GEN + "1 1 1\n1 1 abc\n",
    GEN + "2 2 2\n1 1 1.0\n",
])
def test_malformed_input_raises(impl, text):  # :108-134
    with pytest.raises(impl.IoError):
        impl.parse(text)


def test_error_names_origin_and_line(impl):  # :126-134
    with pytest.raises(impl.IoError) as e:
        impl.parse(GEN + "2 2 1\n3 1 1.0\n")
    assert "test:" in str(e.value) and "3" in str(e.value)


def test_missing_file_reports_path(mpg, orc):  # :136-145
    p = "/nonexistent/morprec-io-test.mtx"
    for fn, err in ((lambda: mpg.read_matrix_market_file(p, device=None), mpg.IoError),
                    (lambda: orc.read_matrix_market_file(p), orc.IoError)):
        with pytest.raises(err) as e:
            fn()
        assert p in str(e.value)


# ---------------------------------------------------------------- native vs oracle
def _fuzz_text(rng, n, m, k, symmetric):
    lines = [SYM if symmetric else GEN, "% generated\n"]
    if rng.random() < 0.5:
        lines.append("\n")
    lines.append(f"{n} {m} {k}\n")
    for _ in range(k):
        i = rng.randint(1, n)
        j = rng.randint(1, min(i, m) if symmetric else m)
        v = rng.choice([rng.uniform(-1, 1), float(rng.randint(-5, 5)), rng.uniform(-1, 1) * 10 ** rng.randint(-300, 300)])
        sep = rng.choice([" ", "  ", "\t", " \t "])
        fmt = rng.choice(["{!r}", "{:.17g}", "{:e}", "{:.3f}"])
        lines.append(f"{rng.choice(['', ' ', '  '])}{i}{sep}{j}{sep}{fmt.format(v)}{rng.choice(['', ' ', chr(13)])}\n")
        if rng.random() < 0.05:
            lines.append(rng.choice(["\n", "   \n", "\t\r\n"]))
    return "".join(lines)


@pytest.mark.parametrize("seed", range(24))
def test_native_matches_oracle_on_generated_files(mpg, orc, seed):
    rng = random.Random(seed)
    sym = seed % 3 == 0
    n, m = rng.randint(1, 300), rng.randint(1, 300)
    if sym:
        m = n
    text = _fuzz_text(rng, n, m, rng.randint(0, 3000), sym)
    want = orc.read_matrix_market(text, "f").export()
    wv = np.asarray(want[2])
    ref = None
    for t in (1, 3, 16):
        h = mpg.read_matrix_market(text, "f", t, device=None)
        assert np.array_equal(h.rowptr, want[0]) and np.array_equal(h.colind, want[1])  # pattern: bitwise
        # values: duplicate sums follow the reference's std::sort order, which the standard leaves
        # unspecified -> agreement to rounding of the sum of |contributions| (bitwise without duplicates,
        # test_native_is_bitwise_without_duplicates)
        scale = _abs_sums(text, h)
        assert np.all(np.abs(h.val - wv) <= 1e-14 * scale)
        if ref is None:
            ref = h.val.copy()
        assert np.array_equal(h.val.view(np.int64), ref.view(np.int64))  # independent of the thread count


@pytest.mark.parametrize("seed", range(6))
def test_native_is_bitwise_without_duplicates(mpg, orc, seed):
    rng = np.random.default_rng(seed)
    n, m, k = 400, 300, 5000
    cells = rng.choice(n * m, size=k, replace=False)
    vals = rng.standard_normal(k) * 10.0 ** rng.integers(-200, 200, k)
    text = GEN + f"{n} {m} {k}\n" + "".join(f"{c // m + 1} {c % m + 1} {float(v)!r}\n" for c, v in zip(cells, vals))
    want = orc.read_matrix_market(text, "f").export()
    h = mpg.read_matrix_market(text, "f", 8, device=None)
    assert np.array_equal(h.rowptr, want[0]) and np.array_equal(h.colind, want[1])
    assert np.array_equal(h.val.view(np.int64), np.asarray(want[2]).view(np.int64))


def _abs_sums(text, h):
    """Per stored entry of h: the sum of |contributions| from the file (symmetric mirrored)."""
    lines = [l for l in text.split("\n") if l.strip(" \t\r")]
    sym = "symmetric" in lines[0]
    body = [l for l in lines[1:] if not l.startswith("%")][1:]
    acc = {}
    for l in body:
        i, j, v = l.split()[:3]
        i, j, v = int(i) - 1, int(j) - 1, abs(float(v))
        acc[(i, j)] = acc.get((i, j), 0.0) + v
        if sym and i != j:
            acc[(j, i)] = acc.get((j, i), 0.0) + v
    out = np.zeros(h.val.size)
    for r in range(h.nrows):
        for q in range(h.rowptr[r], h.rowptr[r + 1]):
            out[q] = acc[(r, int(h.colind[q]))]
    return out


def _corrupt(rng, text):
    lines = text.split("\n")
    body = [i for i, l in enumerate(lines) if i >= 3]
    if not body:
        return text
    i = rng.choice(body)
    kind = rng.randrange(5)
    if kind == 0:
        lines[i] = "1 2 abc"
    elif kind == 1:
        lines[i] = "999999 1 1.0"
    elif kind == 2:
        lines[i] = "% a comment inside the entries"
    elif kind == 3:
        lines[i] = "1"
    else:
        lines = lines[: i]  # truncated
    return "\n".join(lines)


@pytest.mark.parametrize("seed", range(40))
def test_native_errors_match_oracle(mpg, orc, seed):
    rng = random.Random(1000 + seed)
    text = _corrupt(rng, _fuzz_text(rng, 50, 40, rng.randint(1, 400), False))
    try:
        want = ("ok", orc.read_matrix_market(text, "f").export())
    except orc.IoError as e:
        want = ("err", str(e))
    for t in (1, 4, 32):
        try:
            h = mpg.read_matrix_market(text, "f", t, device=None)
            got = ("ok", (h.rowptr, h.colind, h.val))
        except mpg.IoError as e:
            got = ("err", str(e))
        assert got[0] == want[0]
        if want[0] == "err":
            assert got[1] == want[1]
        else:
            assert all(np.array_equal(x, np.asarray(y)) for x, y in zip(got[1], want[1]))


def test_lines_after_the_last_entry_are_ignored(impl):
    a = impl.parse(GEN + "2 2 1\n1 1 4.0\nthis line is never read\n")
    assert a[0, 0] == 4.0


def test_config_matrix_round_trip(mpg, gen, tmp_path):
    a = gen.config2(M=12).a
    p = tmp_path / "c2.mtx"
    mpg.write_matrix_market_file(p, a, threads=4)
    b = mpg.read_matrix_market_file(p, threads=5, device=None)
    assert np.array_equal(b.rowptr, a.rowptr) and np.array_equal(b.colind, a.colind)
    assert np.array_equal(b.val, a.val)


# ---------------------------------------------------------------- report CSV
def test_report_csv_layout(mpg):  # report.cpp:46-63
    nan = float("nan")
    rows = [mpg.ReportRow(1, 1, "fresh", 1, 33, 1.5, 0.25, nan, nan, 0.5),
            mpg.ReportRow(1, 2, "horizontal", 1, 40, 0.123456789, 1e-7, 0.0625, 3.0, nan),
            mpg.ReportRow(2, 1, "reused_same_matrix", 2, 7, 0.0, 12345678.9, nan, nan, nan)]
    f = io.StringIO()
    mpg.ReductionReport(rows, True).write_csv(f)
    assert f.getvalue() == (
        "sweep,point,precond,solves,precond_build_seconds,gmres_iterations,gmres_seconds,min_residual,"
        "matrix_change,standard_residual,first_approach_min_residual\n"
        "1,1,fresh,1,1.5,33,0.25,,,0.5,\n"
        "1,2,horizontal,1,0.123457,40,1e-07,0.0625,3,,\n"
        "2,1,reused_same_matrix,2,0,7,1.23457e+07,,,,\n"
        "TOTAL,,,4,1.62346,80,1.23457e+07,,,,\n")
