"""CPU ORACLE — test infrastructure only.

ctypes wrapper of oracle/liboracle.so, the C++ restatement of the reference
`morprec` solve path (see oracle/oracle.hpp for the file:line map). Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this package, and only as the checker / the timed CPU baseline. The product
(paper_2003_12759_b200) never imports it.

Parity status: pinned to the reference's own test assertions
(proj/tests/*.cpp, restated in tests/test_oracle_*.py); the reference itself
cannot be built here (Eigen3 and vendored doctest/CLI11 are absent), so there
are no reference-generated golden outputs.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE, "-j8"], check=True)


if not os.path.exists(LIB_PATH):
    build()

lib = C.CDLL(LIB_PATH)

vp, dp, ip, lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_longlong)


class SpaiCfg(C.Structure):
    _fields_ = [("pattern_kind", C.c_int), ("power", C.c_int), ("fill_tol", C.c_double),
                ("max_fill_per_col", C.c_int), ("max_pattern_sweeps", C.c_int), ("threads", C.c_int)]


class GmresCfg(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iter", C.c_int), ("record_history", C.c_int)]


class GmresRep(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int), ("history_len", C.c_int),
                ("rhs_norm", C.c_double), ("final_residual", C.c_double), ("solve_seconds", C.c_double),
                ("reorth_passes", C.c_int)]


class AirgaCfgO(C.Structure):
    _fields_ = [("r_max", C.c_int), ("outer_tol", C.c_double), ("inner_tol", C.c_double), ("max_outer", C.c_int),
                ("gmres", GmresCfg), ("spai", SpaiCfg), ("max_chain_len", C.c_int),
                ("standard_residual_max_dim", C.c_longlong)]


class IrkaCfg(C.Structure):
    _fields_ = [("r", C.c_int), ("tol", C.c_double), ("max_sweeps", C.c_int), ("decoupled", C.c_int),
                ("seed", C.c_ulonglong), ("gmres", GmresCfg), ("spai", SpaiCfg), ("max_chain_len", C.c_int),
                ("explicit_nnz_cap", C.c_longlong), ("standard_residual_max_dim", C.c_longlong),
                ("mirror_unstable", C.c_int), ("unit_threads", C.c_int)]


class ReportRow(C.Structure):
    _fields_ = [("sweep", C.c_int), ("point", C.c_int), ("kind", C.c_int), ("solves", C.c_int),
                ("iterations", C.c_longlong), ("build_seconds", C.c_double), ("gmres_seconds", C.c_double),
                ("min_residual", C.c_double), ("matrix_change", C.c_double), ("standard_residual", C.c_double)]


_SIGS = {
    "orc_airga_reduce": (C.c_int, [vp, vp, vp, vp, C.c_int, vp, C.c_int, C.c_double, C.c_double, vp, C.c_int, vp,
                                   C.c_int, C.POINTER(C.c_int)] + [vp] * 7 + [C.POINTER(C.c_int), C.POINTER(C.c_int),
                                                                             vp, C.c_int, C.POINTER(C.c_int)]),
    "orc_update_expansion_points": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, vp]),
    "orc_h2_norm": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, dp]),
    "orc_last_error": (C.c_char_p, []),
    "orc_csr_from_csr": (C.c_int, [C.c_longlong, C.c_longlong, vp, vp, vp, C.POINTER(vp)]),
    "orc_csr_from_triplets": (C.c_int, [C.c_longlong, C.c_longlong, C.c_longlong, vp, vp, vp, C.POINTER(vp)]),
    "orc_csr_free": (None, [vp]),
    "orc_csr_info": (None, [vp, lp, lp, lp]),
    "orc_csr_export": (None, [vp, vp, vp, vp]),
    "orc_csr_multiply": (C.c_int, [vp, C.c_longlong, vp, vp]),
    "orc_csr_multiply_transpose": (C.c_int, [vp, C.c_longlong, vp, vp]),
    "orc_csr_transpose": (C.c_int, [vp, C.POINTER(vp)]),
    "orc_csr_linear_combination": (C.c_int, [C.c_int, vp, vp, C.POINTER(vp)]),
    "orc_csr_frobenius_norm": (C.c_double, [vp]),
    "orc_csr_extract": (C.c_int, [vp, C.c_longlong, vp, lp, vp, vp, C.c_longlong]),
    "orc_spai_build": (C.c_int, [vp, C.POINTER(SpaiCfg), C.POINTER(vp), vp, lp, dp]),
    "orc_spai_column_solve": (C.c_int, [vp, C.c_longlong, C.c_longlong, vp, vp, dp, ip]),
    "orc_update_build": (C.c_int, [vp, vp, C.POINTER(SpaiCfg), C.POINTER(vp), dp, dp, lp, dp]),
    "orc_chain_create": (C.c_int, [vp, C.POINTER(vp)]),
    "orc_chain_extend": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "orc_chain_length": (C.c_int, [vp]),
    "orc_chain_free": (None, [vp]),
    "orc_chain_apply": (C.c_int, [vp, C.c_longlong, vp, vp]),
    "orc_standard_residual": (C.c_int, [vp, vp, dp]),
    "orc_gmres_csr": (C.c_int, [vp, vp, C.c_longlong, vp, vp, C.POINTER(GmresCfg), C.POINTER(GmresRep), vp]),
    "orc_gmres_kron": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, C.POINTER(GmresCfg), C.POINTER(GmresRep), vp]),
    "orc_kron_apply": (C.c_int, [vp, C.c_int, vp, vp, vp, vp]),
    "orc_kron_assemble": (C.c_int, [vp, C.c_int, vp, vp, C.c_longlong, C.POINTER(vp)]),
    "orc_real_spectrum": (C.c_int, [vp, C.c_int, vp, vp, vp]),
    "orc_sorted_eigenvalues": (C.c_int, [vp, C.c_int, vp, vp]),
    "orc_colpiv_solve": (C.c_int, [vp, C.c_longlong, C.c_longlong, vp, vp, lp]),
    "orc_thin_q": (C.c_int, [vp, C.c_longlong, C.c_longlong, vp]),
    "orc_irka_default_seed": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, C.c_int, C.c_ulonglong, vp, vp, vp]),
    "orc_irka_reduce": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, C.POINTER(IrkaCfg), C.c_int, vp, vp, vp, vp, vp,
                                  vp, vp, vp, vp, vp, vp, vp, ip, ip, vp, C.c_int, ip]),
    "orc_spai_bench": (C.c_int, [vp, vp, vp, C.c_int, vp, C.POINTER(SpaiCfg), C.POINTER(GmresCfg), C.c_int, C.c_int,
                                 vp, vp, C.c_int, ip, ip]),
    "orc_qbihomm_reduce": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, vp, C.c_int, C.c_int, C.POINTER(GmresCfg),
                                     C.POINTER(SpaiCfg), C.c_int, C.c_longlong, C.c_int, C.c_int, ip, vp, vp, vp, vp,
                                     vp, vp, vp, vp, C.c_int, ip]),
    "orc_birka_reduce": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, C.POINTER(IrkaCfg), C.c_int] + [vp] * 8
                         + [ip, ip, vp, C.c_int, ip]),
    "orc_kron_coupled": (C.c_int, [vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, C.POINTER(vp)]),
    "orc_kron_compress_quadratic": (C.c_int, [vp, vp, C.c_longlong, C.c_longlong, vp]),
    "orc_mm_read_buffer": (C.c_int, [C.c_char_p, C.c_longlong, C.c_char_p, C.POINTER(vp)]),
    "orc_mm_read_file": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "orc_mm_write_buffer": (C.c_int, [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_longlong)]),
    "orc_buffer_free": (None, [vp]),
    "orc_transfer_function_error": (C.c_int, [vp, vp, vp, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, C.c_int, vp,
                                              C.c_int, C.POINTER(GmresCfg), C.POINTER(SpaiCfg), C.c_int, C.c_int, vp]),
}
for _n, (_r, _a) in _SIGS.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a


class ConfigError(RuntimeError):
    pass


class SolverError(RuntimeError):
    pass


class IoError(RuntimeError):
    pass


def _check(st: int) -> None:
    if st == 0:
        return
    msg = lib.orc_last_error().decode()
    if st == 1:
        raise ValueError(msg)
    if st == 2:
        raise ConfigError(msg)
    if st == 3:
        raise SolverError(msg)
    if st == 7:
        raise IoError(msg)
    raise RuntimeError(msg)


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _i64(x):
    return np.ascontiguousarray(x, dtype=np.int64)


def _p(a):
    return None if a is None else a.ctypes.data


class Csr:
    """Oracle SparseMatrix (proj/src/sparse.cpp)."""

    def __init__(self, h):
        self._h = C.c_void_p(h)
        nr, nc, nz = C.c_longlong(), C.c_longlong(), C.c_longlong()
        lib.orc_csr_info(self._h, C.byref(nr), C.byref(nc), C.byref(nz))
        self.shape = (nr.value, nc.value)
        self._nnz = nz.value

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.orc_csr_free(self._h)
            self._h = None

    @staticmethod
    def from_csr(nrows, ncols, rp, ci, v) -> "Csr":
        rp, ci, v = _i64(rp), _i64(ci), _f64(v)
        h = C.c_void_p()
        _check(lib.orc_csr_from_csr(nrows, ncols, _p(rp), _p(ci), _p(v), C.byref(h)))
        return Csr(h.value)

    @staticmethod
    def of(host) -> "Csr":
        """From a paper_2003_12759_b200.gen.HostCsr (or anything with nrows/ncols/rowptr/colind/val)."""
        return Csr.from_csr(host.nrows, host.ncols, host.rowptr, host.colind, host.val)

    @staticmethod
    def from_triplets(nr, nc, rows, cols, vals) -> "Csr":
        r, c, v = _i64(rows), _i64(cols), _f64(vals)
        h = C.c_void_p()
        _check(lib.orc_csr_from_triplets(nr, nc, r.size, _p(r), _p(c), _p(v), C.byref(h)))
        return Csr(h.value)

    @staticmethod
    def from_dense(d, drop_tol=0.0) -> "Csr":
        d = np.asarray(d, dtype=np.float64)
        r, c = np.nonzero(np.abs(d) > drop_tol)
        return Csr.from_triplets(d.shape[0], d.shape[1], r, c, d[r, c])

    @staticmethod
    def identity(n) -> "Csr":
        return Csr.from_csr(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    @staticmethod
    def diagonal(d) -> "Csr":
        d = _f64(d)
        return Csr.from_csr(d.size, d.size, np.arange(d.size + 1), np.arange(d.size), d)

    @staticmethod
    def zero(nr, nc) -> "Csr":
        return Csr.from_csr(nr, nc, np.zeros(nr + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))

    @staticmethod
    def linear_combination(terms) -> "Csr":
        coeffs = _f64([c for c, _ in terms])
        mats = (C.c_void_p * len(terms))(*[m._h.value for _, m in terms])
        h = C.c_void_p()
        _check(lib.orc_csr_linear_combination(len(terms), _p(coeffs), mats, C.byref(h)))
        return Csr(h.value)

    def nnz(self) -> int:
        return self._nnz

    def rows(self) -> int:
        return self.shape[0]

    def cols(self) -> int:
        return self.shape[1]

    def export(self):
        rp = np.empty(self.shape[0] + 1, np.int64)
        ci = np.empty(self._nnz, np.int64)
        v = np.empty(self._nnz)
        lib.orc_csr_export(self._h, _p(rp), _p(ci), _p(v))
        return rp, ci, v

    def to_dense(self) -> np.ndarray:
        rp, ci, v = self.export()
        d = np.zeros(self.shape)
        for i in range(self.shape[0]):
            d[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
        return d

    def to_scipy(self):
        import scipy.sparse as sp
        rp, ci, v = self.export()
        return sp.csr_matrix((v, ci, rp), shape=self.shape)

    def multiply(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(self.shape[0])
        _check(lib.orc_csr_multiply(self._h, x.size, _p(x), _p(y)))
        return y

    def multiply_transpose(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(self.shape[1])
        _check(lib.orc_csr_multiply_transpose(self._h, x.size, _p(x), _p(y)))
        return y

    def transpose(self) -> "Csr":
        h = C.c_void_p()
        _check(lib.orc_csr_transpose(self._h, C.byref(h)))
        return Csr(h.value)

    def frobenius_norm(self) -> float:
        return float(lib.orc_csr_frobenius_norm(self._h))

    def extract_column_submatrix(self, pattern):
        pat = _i64(pattern)
        nr = C.c_longlong()
        _check(lib.orc_csr_extract(self._h, pat.size, _p(pat), C.byref(nr), None, None, 0))
        rm = np.empty(nr.value, np.int64)
        blk = np.empty(nr.value * pat.size)
        _check(lib.orc_csr_extract(self._h, pat.size, _p(pat), C.byref(nr), _p(rm), _p(blk), nr.value))
        return blk.reshape((nr.value, pat.size), order="F"), rm


@dataclasses.dataclass
class SpaiConfig:
    pattern: str = "a"
    fill_tol: float = 1e-4
    max_fill_per_col: int = 50
    max_pattern_sweeps: int = 3
    threads: int = 1
    power: int = 2

    def c(self):
        return SpaiCfg({"diagonal": 0, "a": 1, "a_pow": 2}[self.pattern], self.power, self.fill_tol,
                       self.max_fill_per_col, self.max_pattern_sweeps, self.threads)


@dataclasses.dataclass
class GmresConfig:
    rel_tol: float = 1e-6
    max_iter: int = 1000
    record_history: bool = False

    def c(self):
        return GmresCfg(self.rel_tol, self.max_iter, int(self.record_history))


@dataclasses.dataclass
class GmresReport:
    iterations: int
    converged: bool
    breakdown: bool
    rhs_norm: float
    final_residual: float
    solve_seconds: float
    residual_history: list
    reorth_passes: int = 0


class Chain:
    def __init__(self, base: Optional[Csr] = None, _h=None, _keep=()):
        self._keep = list(_keep)
        if _h is not None:
            self._h = C.c_void_p(_h)
        else:
            h = C.c_void_p()
            _check(lib.orc_chain_create(base._h, C.byref(h)))
            self._h = h
            self._keep = [base]
        self.n = self._keep[0].shape[0]

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.orc_chain_free(self._h)
            self._h = None

    def extended(self, q: Csr) -> "Chain":
        h = C.c_void_p()
        _check(lib.orc_chain_extend(self._h, q._h, C.byref(h)))
        return Chain(_h=h.value, _keep=self._keep + [q])

    def length(self) -> int:
        return lib.orc_chain_length(self._h)

    def apply(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(self.n)
        _check(lib.orc_chain_apply(self._h, x.size, _p(x), _p(y)))
        return y


def _rep(r: GmresRep, hist):
    return GmresReport(r.iterations, bool(r.converged), bool(r.breakdown), r.rhs_norm, r.final_residual,
                       r.solve_seconds, list(hist[: r.history_len]) if hist is not None else [], r.reorth_passes)


def gmres_csr(a: Csr, chain: Optional[Chain], b, cfg: GmresConfig = GmresConfig()):
    b = _f64(b)
    x = np.empty(b.size)
    rep = GmresRep()
    hist = np.empty(cfg.max_iter + 2) if cfg.record_history else None
    c = cfg.c()
    _check(lib.orc_gmres_csr(a._h, chain._h if chain else None, b.size, _p(b), _p(x), C.byref(c), C.byref(rep),
                             _p(hist)))
    return x, _rep(rep, hist)


def gmres_kron(lam, a: Csr, e: Optional[Csr], chain: Optional[Chain], b, cfg: GmresConfig = GmresConfig()):
    """GMRES on -(Lambda (x) E) - (I (x) A); a real shift sigma is lam = [[-sigma]]."""
    lam = np.asfortranarray(np.atleast_2d(np.asarray(lam, dtype=np.float64)))
    b = _f64(b)
    x = np.empty(b.size)
    rep = GmresRep()
    hist = np.empty(cfg.max_iter + 2) if cfg.record_history else None
    c = cfg.c()
    _check(lib.orc_gmres_kron(_p(lam), lam.shape[0], a._h, e._h if e else None, chain._h if chain else None, _p(b),
                              _p(x), C.byref(c), C.byref(rep), _p(hist)))
    return x, _rep(rep, hist)


def kron_apply(lam, a: Csr, e: Optional[Csr], x) -> np.ndarray:
    lam = np.asfortranarray(np.atleast_2d(np.asarray(lam, dtype=np.float64)))
    x = _f64(x)
    y = np.empty(x.size)
    _check(lib.orc_kron_apply(_p(lam), lam.shape[0], a._h, e._h if e else None, _p(x), _p(y)))
    return y


def kron_assemble(lam, a: Csr, e: Optional[Csr], cap: int = 200000) -> Csr:
    lam = np.asfortranarray(np.atleast_2d(np.asarray(lam, dtype=np.float64)))
    h = C.c_void_p()
    _check(lib.orc_kron_assemble(_p(lam), lam.shape[0], a._h, e._h if e else None, cap, C.byref(h)))
    return Csr(h.value)


def shifted(sigma: complex) -> np.ndarray:
    """The Lambda block whose Kronecker unit is sigma E - A (pair form for complex sigma)."""
    s = complex(sigma)
    if s.imag == 0:
        return np.array([[-s.real]])
    a, b = -s.real, -s.imag
    return np.array([[a, b], [-b, a]])


def spai_build(a: Csr, cfg: SpaiConfig = SpaiConfig()):
    res = np.empty(a.shape[0])
    p = C.c_void_p()
    fb = C.c_longlong()
    secs = C.c_double()
    c = cfg.c()
    _check(lib.orc_spai_build(a._h, C.byref(c), C.byref(p), _p(res), C.byref(fb), C.byref(secs)))
    return Csr(p.value), res, fb.value, secs.value


def spai_column_solve(a: Csr, col: int, pattern):
    pat = np.sort(_i64(pattern))
    vals = np.empty(pat.size)
    r = C.c_double()
    rd = C.c_int()
    _check(lib.orc_spai_column_solve(a._h, col, pat.size, _p(pat), _p(vals), C.byref(r), C.byref(rd)))
    return pat, vals, r.value, bool(rd.value)


def update_build(prev: Csr, new: Csr, cfg: SpaiConfig = SpaiConfig()):
    q = C.c_void_p()
    mr, mc, secs = C.c_double(), C.c_double(), C.c_double()
    fb = C.c_longlong()
    c = cfg.c()
    _check(lib.orc_update_build(prev._h, new._h, C.byref(c), C.byref(q), C.byref(mr), C.byref(mc), C.byref(fb),
                                C.byref(secs)))
    return Csr(q.value), mr.value, mc.value, fb.value, secs.value


def standard_residual(a: Csr, chain: Chain) -> float:
    out = C.c_double()
    _check(lib.orc_standard_residual(a._h, chain._h, C.byref(out)))
    return out.value


def real_spectrum(m):
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    r = m.shape[0]
    bl, ba, bi = (np.zeros((r, r), order="F") for _ in range(3))
    st = lib.orc_real_spectrum(_p(m), r, _p(bl), _p(ba), _p(bi))
    if st != 0:
        return None
    return bl, ba, bi


def sorted_eigenvalues(m) -> np.ndarray:
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    r = m.shape[0]
    re, im = np.zeros(r), np.zeros(r)
    _check(lib.orc_sorted_eigenvalues(_p(m), r, _p(re), _p(im)))
    return re + 1j * im


def colpiv_solve(a, b):
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    b = _f64(b)
    x = np.empty(a.shape[1])
    rank = C.c_longlong()
    _check(lib.orc_colpiv_solve(_p(a), a.shape[0], a.shape[1], _p(b), _p(x), C.byref(rank)))
    return x, rank.value


def thin_q(a) -> np.ndarray:
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    q = np.zeros(a.shape, order="F")
    _check(lib.orc_thin_q(_p(a), a.shape[0], a.shape[1], _p(q)))
    return q


@dataclasses.dataclass
class IrkaConfig:
    r: int = 2
    tol: float = 1e-4
    max_sweeps: int = 50
    seed: int = 1
    gmres: GmresConfig = dataclasses.field(default_factory=lambda: GmresConfig(1e-10, 1000, False))
    spai: SpaiConfig = dataclasses.field(default_factory=SpaiConfig)
    max_chain_len: int = 16
    explicit_nnz_cap: int = 200000
    standard_residual_max_dim: int = 5000
    decoupled: bool = False
    mirror_unstable: bool = False
    unit_threads: int = 1

    def c(self):
        return IrkaCfg(self.r, self.tol, self.max_sweeps, int(self.decoupled), self.seed, self.gmres.c(),
                       self.spai.c(), self.max_chain_len, self.explicit_nnz_cap, self.standard_residual_max_dim,
                       int(self.mirror_unstable), int(self.unit_threads))


@dataclasses.dataclass
class IrkaResult:
    kr: np.ndarray
    fr: np.ndarray
    cr: np.ndarray
    er: np.ndarray
    ar: np.ndarray
    lam: np.ndarray
    v: Optional[np.ndarray]
    w: Optional[np.ndarray]
    sweeps: int
    converged: bool
    rows: list

    def transfer(self, s: complex) -> np.ndarray:
        r = self.kr.shape[0]
        return self.cr.T @ np.linalg.solve(s * np.eye(r) - self.kr, self.fr)


def irka_reduce(a: Csr, e: Optional[Csr], b, c, cfg: IrkaConfig, mode: int = 2, init_shifts=None,
                want_bases: bool = False, init_kr=None) -> IrkaResult:
    n = a.shape[0]
    bm = np.asfortranarray(np.asarray(b, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    m, q, r = bm.shape[1], cm.shape[1], cfg.r
    kr, er, ar = (np.zeros((r, r), order="F") for _ in range(3))
    fr, cr = np.zeros((r, m), order="F"), np.zeros((r, q), order="F")
    lre, lim = np.zeros(r), np.zeros(r)
    v = np.zeros((n, r), order="F") if want_bases else None
    w = np.zeros((n, r), order="F") if want_bases else None
    sweeps, conv, nrows = C.c_int(), C.c_int(), C.c_int()
    maxrows = 2 * r * max(cfg.max_sweeps, 1) + 8
    rows = (ReportRow * maxrows)()
    ini = None
    if init_shifts is not None:
        ini = np.asfortranarray(np.diag(-_f64(init_shifts)))
    if init_kr is not None:  # birka_reduce's initial BirkaState (birka.hpp:78-80): K_r given, fr/cr default-seeded
        ini = np.asfortranarray(np.asarray(init_kr, dtype=np.float64))
        assert ini.shape == (cfg.r, cfg.r)
    cc = cfg.c()
    _check(lib.orc_irka_reduce(a._h, e._h if e else None, _p(bm), m, _p(cm), q, C.byref(cc), mode, _p(ini), None, None,
                               _p(kr), _p(fr), _p(cr), _p(er), _p(ar), _p(lre), _p(lim), _p(v), _p(w),
                               C.byref(sweeps), C.byref(conv), rows, maxrows, C.byref(nrows)))
    return IrkaResult(kr, fr, cr, er, ar, lre + 1j * lim, v, w, sweeps.value, bool(conv.value),
                      [rows[i] for i in range(min(nrows.value, maxrows))])


def irka_default_seed(a: Csr, e: Optional[Csr], b, c, r: int, seed: int):
    n = a.shape[0]
    bm = np.asfortranarray(np.asarray(b, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    kr = np.zeros((r, r), order="F")
    fr = np.zeros((r, bm.shape[1]), order="F")
    cr = np.zeros((r, cm.shape[1]), order="F")
    _check(lib.orc_irka_default_seed(a._h, e._h if e else None, _p(bm), bm.shape[1], _p(cm), cm.shape[1], r, seed,
                                     _p(kr), _p(fr), _p(cr)))
    return kr, fr, cr


def spai_bench(a: Csr, e: Optional[Csr], b, points: Sequence[float], spai: SpaiConfig = SpaiConfig(),
               gmres: GmresConfig = GmresConfig(), mode: int = 2, max_chain_len: int = 16, keep_solutions=False):
    b = _f64(b)
    pts = _f64(points)
    x = np.zeros((len(pts), b.size)) if keep_solutions else None
    rows = (ReportRow * len(pts))()
    nrows, failed = C.c_int(), C.c_int()
    s, g = spai.c(), gmres.c()
    _check(lib.orc_spai_bench(a._h, e._h if e else None, _p(b), len(pts), _p(pts), C.byref(s), C.byref(g), mode,
                              max_chain_len, _p(x), rows, len(pts), C.byref(nrows), C.byref(failed)))
    return [rows[i] for i in range(nrows.value)], failed.value, x


@dataclasses.dataclass
class QbConfig:
    """QbConfig (proj/include/morprec/qbihomm.hpp:35-43)."""
    sigmas: Sequence[float] = ()
    p_moments: int = 1
    q_moments: int = 1
    gmres: GmresConfig = dataclasses.field(default_factory=GmresConfig)
    spai: SpaiConfig = dataclasses.field(default_factory=SpaiConfig)
    max_chain_len: int = 16
    standard_residual_max_dim: int = 5000


@dataclasses.dataclass
class ReducedQb:
    d: np.ndarray
    k: np.ndarray
    n_op: np.ndarray
    h: np.ndarray
    f: np.ndarray
    c: np.ndarray
    basis: np.ndarray
    rows: list

    def order(self) -> int:
        return self.d.shape[0]

    def linear_transfer(self, s: float) -> float:
        """c^T (s D_r - K_r)^{-1} f (the basis-invariant check of test_qbihomm.cpp:200-207)."""
        return float(self.c[:, 0] @ np.linalg.solve(s * self.d - self.k, self.f[:, 0]))


def qbihomm_reduce(d: Csr, k: Csr, n_op: Csr, h: Csr, f, c, cfg: QbConfig, mode: int = 2) -> ReducedQb:
    """qbihomm_reduce (proj/src/qbihomm.cpp:144-208); mode 0 None, 1 FreshSpai, 2 ReuseChain."""
    n = d.shape[0]
    for name, v in (("F", f), ("C", c)):  # QbSystem::create (qbihomm.cpp:30-33)
        a = np.asarray(v)
        if a.ndim == 2 and a.shape[1] != 1 or a.size != n:
            raise ConfigError(f"quadratic-bilinear system: {name} must be a single n-column (SISO)")
    f, c = _f64(f).reshape(-1), _f64(c).reshape(-1)
    sig = _f64(cfg.sigmas)
    cap = max(1, len(sig) * (cfg.p_moments + 2 * cfg.q_moments + 2))
    basis = np.zeros((n, cap), order="F")
    rd, rk, rn = (np.zeros((cap, cap), order="F") for _ in range(3))
    rh = np.zeros((cap, cap * cap), order="F")
    rf, rc = np.zeros(cap), np.zeros(cap)
    order, nrows = C.c_int(), C.c_int()
    maxrows = 4 * max(1, len(sig))
    rows = (ReportRow * maxrows)()
    g, s = cfg.gmres.c(), cfg.spai.c()
    _check(lib.orc_qbihomm_reduce(d._h, k._h, n_op._h, h._h, _p(f), _p(c), len(sig), _p(sig), cfg.p_moments,
                                  cfg.q_moments, C.byref(g), C.byref(s), cfg.max_chain_len,
                                  cfg.standard_residual_max_dim, mode, cap, C.byref(order), _p(basis), _p(rd), _p(rk),
                                  _p(rn), _p(rh), _p(rf), _p(rc), rows, maxrows, C.byref(nrows)))
    r = order.value
    take = lambda a, rr, cc: np.asfortranarray(a.reshape(-1, order="F")[: rr * cc].reshape((rr, cc), order="F"))
    return ReducedQb(take(rd, r, r), take(rk, r, r), take(rn, r, r), take(rh, r, r * r), rf[:r].reshape(r, 1).copy(),
                     rc[:r].reshape(r, 1).copy(), take(basis, n, r), [rows[i] for i in range(min(nrows.value, maxrows))])


def kron_compress_quadratic(h: Csr, u) -> np.ndarray:
    """kron_compress_quadratic (proj/src/qbihomm.cpp:210-236)."""
    u = np.asfortranarray(np.asarray(u, dtype=np.float64))
    n, r = u.shape
    out = np.zeros((r, r * r), order="F")
    _check(lib.orc_kron_compress_quadratic(h._h, _p(u), n, r, _p(out)))
    return out


def read_matrix_market(text, origin: str = "<stream>") -> Csr:
    """read_matrix_market (proj/src/matrix_market.cpp:38-98), sequential istream restatement."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = vp()
    _check(lib.orc_mm_read_buffer(data, len(data), origin.encode(), C.byref(h)))
    return Csr(h.value)


def read_matrix_market_file(path: str) -> Csr:
    h = vp()
    _check(lib.orc_mm_read_file(str(path).encode(), C.byref(h)))
    return Csr(h.value)


def write_matrix_market(a: Csr) -> str:
    """write_matrix_market (proj/src/matrix_market.cpp:100-114)."""
    buf, n = C.c_void_p(), C.c_longlong()
    _check(lib.orc_mm_write_buffer(a._h, C.byref(buf), C.byref(n)))
    try:
        return C.string_at(buf.value, n.value).decode()
    finally:
        lib.orc_buffer_free(buf)


def transfer_function_error(m: Csr, d: Csr, k: Csr, f, c, red, grid, gmres: GmresConfig = None,
                            spai: SpaiConfig = None, mode: int = 2, max_chain_len: int = 16) -> np.ndarray:
    """transfer_function_error (proj/src/airga.cpp:386-447); red = (m_r, d_r, k_r, f_r, c_r)."""
    n = m.shape[0]
    fm = np.asfortranarray(np.asarray(f, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    rm, rd, rk = (np.asfortranarray(np.asarray(x, dtype=np.float64)) for x in red[:3])
    r = rm.shape[0]
    rf = np.asfortranarray(np.asarray(red[3], dtype=np.float64).reshape(r, -1))
    rc = np.asfortranarray(np.asarray(red[4], dtype=np.float64).reshape(r, -1))
    g = _f64(grid)
    out = np.zeros(g.size)
    gc = (gmres or GmresConfig(1e-10, 1000)).c()
    sc = (spai or SpaiConfig()).c()
    _check(lib.orc_transfer_function_error(m._h, d._h, k._h, _p(fm), fm.shape[1], _p(cm), cm.shape[1], _p(rm), _p(rd),
                                           _p(rk), _p(rf), _p(rc), r, _p(g), g.size, C.byref(gc), C.byref(sc), mode,
                                           max_chain_len, _p(out)))
    return out


@dataclasses.dataclass
class BirkaResult:
    kr: np.ndarray
    nr: list
    fr: np.ndarray
    cr: np.ndarray
    lam: np.ndarray
    v: np.ndarray
    w: np.ndarray
    sweeps: int
    converged: bool
    rows: list


def birka_reduce(k: Csr, n_ops, b, c, cfg: IrkaConfig, mode: int = 2) -> BirkaResult:
    """birka_reduce with couplings (proj/src/birka.cpp:139-310), joint n r solves."""
    n = k.shape[0]
    bm = np.asfortranarray(np.asarray(b, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    m, q, r = bm.shape[1], cm.shape[1], cfg.r
    nptr = (vp * m)(*[x._h.value for x in n_ops])
    kr, nr = np.zeros((r, r), order="F"), np.zeros(r * r * m)
    fr, cr = np.zeros((r, m), order="F"), np.zeros((r, q), order="F")
    lre, lim = np.zeros(r), np.zeros(r)
    v, w = np.zeros((n, r), order="F"), np.zeros((n, r), order="F")
    sweeps, conv, nrows = C.c_int(), C.c_int(), C.c_int()
    maxrows = 2 * max(cfg.max_sweeps, 1) + 8
    rows = (ReportRow * maxrows)()
    cc = cfg.c()
    _check(lib.orc_birka_reduce(k._h, nptr, _p(bm), m, _p(cm), q, C.byref(cc), mode, _p(kr), _p(nr), _p(fr), _p(cr),
                                _p(lre), _p(lim), _p(v), _p(w), C.byref(sweeps), C.byref(conv), rows, maxrows,
                                C.byref(nrows)))
    nrs = [nr[j * r * r:(j + 1) * r * r].reshape((r, r), order="F").copy() for j in range(m)]
    return BirkaResult(kr, nrs, fr, cr, lre + 1j * lim, v, w, sweeps.value, bool(conv.value),
                       [rows[i] for i in range(min(nrows.value, maxrows))])


def _kron_coupled(lam, k: Csr, couplers, x=None, assemble=False):
    lam = np.asfortranarray(np.asarray(lam, dtype=np.float64))
    r = lam.shape[0]
    smalls = np.concatenate([np.asfortranarray(np.asarray(s, dtype=np.float64)).reshape(-1, order="F")
                             for s, _ in couplers]) if couplers else np.zeros(1)
    sp = (vp * max(1, len(couplers)))(*[m._h.value for _, m in couplers])
    y = np.zeros(k.shape[0] * r) if x is not None else None
    xx = _f64(x) if x is not None else None
    h = vp()
    _check(lib.orc_kron_coupled(_p(lam), r, k._h, len(couplers), _p(smalls), sp, _p(xx), _p(y),
                                C.byref(h) if assemble else None))
    return Csr(h.value) if assemble else y


def kron_apply_coupled(lam, k: Csr, couplers, x):
    """vec(-X Lambda^T - K X - sum_j N_j X S_j) (kron.cpp:34-64); couplers = [(S_j, N_j)]."""
    return _kron_coupled(lam, k, couplers, x=x)


def kron_assemble_coupled(lam, k: Csr, couplers) -> Csr:
    """assemble_explicit with couplers (kron.cpp:72-131), no cap."""
    return _kron_coupled(lam, k, couplers, assemble=True)



@dataclasses.dataclass
class AirgaResultO:
    m: np.ndarray
    d: np.ndarray
    k: np.ndarray
    f: np.ndarray
    c: np.ndarray
    final_points: list
    point_history: list
    sweeps: int
    converged: bool
    rows: list

    def transfer(self, s: complex) -> np.ndarray:
        return self.c.T @ np.linalg.solve(s * s * self.m + s * self.d + self.k, self.f)


def airga_reduce(m: Csr, d: Csr, k: Csr, f, c, points, r_max: int = 20, outer_tol: float = 1e-4,
                 inner_tol: float = 1e-6, max_outer: int = 20, gmres: GmresConfig = None, spai: SpaiConfig = None,
                 mode: int = 2, max_chain_len: int = 16, alpha: float = 0.0, beta: float = 0.0) -> AirgaResultO:
    """airga_reduce (proj/src/airga.cpp:136-317) on the oracle, with every sweep's expansion points."""
    n = m.shape[0]
    fm = np.asfortranarray(np.asarray(f, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    pts = _f64(points)
    cfg = AirgaCfgO(r_max, outer_tol, inner_tol, max_outer, (gmres or GmresConfig()).c(), (spai or SpaiConfig()).c(),
                    max_chain_len, 5000)
    cap = max(1, r_max)
    rm, rd, rk = (np.zeros(cap * cap) for _ in range(3))
    rf, rc = np.zeros(cap * fm.shape[1]), np.zeros(cap * cm.shape[1])
    fp = np.zeros(max(1, pts.size))
    hist = np.zeros(max(1, pts.size) * max(1, max_outer))
    order, sweeps, conv, nrows = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    maxrows = 2 * max(1, pts.size) * max(1, max_outer) + 4
    rows = (ReportRow * maxrows)()
    _check(lib.orc_airga_reduce(m._h, d._h, k._h, _p(fm), fm.shape[1], _p(cm), cm.shape[1], alpha, beta, _p(pts),
                                pts.size, C.byref(cfg), mode, C.byref(order), _p(rm), _p(rd), _p(rk), _p(rf), _p(rc),
                                _p(fp), _p(hist), C.byref(sweeps), C.byref(conv), rows, maxrows, C.byref(nrows)))
    r = order.value
    sq = lambda x: x[: r * r].reshape((r, r), order="F")
    return AirgaResultO(sq(rm), sq(rd), sq(rk), rf[: r * fm.shape[1]].reshape((r, -1), order="F"),
                        rc[: r * cm.shape[1]].reshape((r, -1), order="F"), fp[: pts.size].tolist(),
                        [hist[z * pts.size:(z + 1) * pts.size].tolist() for z in range(sweeps.value)],
                        sweeps.value, bool(conv.value), [rows[i] for i in range(min(nrows.value, maxrows))])


def update_expansion_points(m, d, k, current) -> list:
    """update_expansion_points (proj/src/airga.cpp:319-384)."""
    mm, dd, kk = (np.asfortranarray(np.asarray(x, dtype=np.float64)) for x in (m, d, k))
    cur = _f64(current)
    out = np.zeros(max(1, cur.size))
    _check(lib.orc_update_expansion_points(_p(mm), _p(dd), _p(kk), mm.shape[0], _p(cur), cur.size, _p(out)))
    return out[: cur.size].tolist()


def h2_norm(a, b, c) -> float:
    """h2_norm (proj/src/h2.cpp:28-60); the Gramian by the matrix sign function."""
    a, b, c = (np.asfortranarray(np.asarray(x, dtype=np.float64)) for x in (a, b, c))
    out = C.c_double()
    _check(lib.orc_h2_norm(_p(a), _p(b), _p(c), a.shape[0], b.shape[1], c.shape[0], C.byref(out)))
    return out.value
