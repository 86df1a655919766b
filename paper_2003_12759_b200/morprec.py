"""Python mirror of the reference `morprec` solve-path API over libmpg.so.

Names, argument meaning and error behaviour follow proj/include/morprec:
SparseMatrix (sparse.hpp:33-101), gmres_right_preconditioned (gmres.hpp:49-50),
spai_build / spai_column_solve (spai.hpp:56-63), update_build and PrecondChain
(chain.hpp:45-77), standard_residual (chain.hpp:79-81), birka_reduce with N = 0
(birka.hpp:78-80, generalised to E) and run_spai_bench (bench.hpp:50-57).
std::invalid_argument maps to ValueError; ConfigError / SolverError keep their
names. Every call runs on the GPU; there is no CPU fallback.

Vectors may be numpy arrays (host) or torch CUDA tensors (device); results
come back in the same kind of container as the right-hand side.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import ConfigError, IoError, SolverError, check, lib

__all__ = [
    "SparseMatrix", "ShiftedOperator", "PrecondChain", "GmresConfig", "GmresReport", "GmresResult", "SpaiConfig",
    "SpaiResult", "UpdateFactor", "IrkaConfig", "IrkaState", "ReportRow", "ReductionReport", "SweepResult",
    "gmres_right_preconditioned", "gmres_shifted", "gmres_batch", "spai_build", "spai_column_solve", "update_build",
    "standard_residual", "irka_reduce", "run_spai_bench", "ConfigError", "SolverError", "PrecondMode",
    "QbSystem", "QbConfig", "ReducedQb", "qbihomm_reduce", "IoError", "read_matrix_market",
    "read_matrix_market_file", "write_matrix_market", "write_matrix_market_file", "SecondOrderSystem",
    "ReducedSecondOrder", "TransferErrorConfig", "transfer_function_error", "project", "AirgaConfig",
    "airga_reduce", "update_expansion_points", "h2_norm", "BirkaState", "birka_reduce",
]


class PrecondMode:
    """PrecondMode (proj/include/morprec/chain.hpp:21) plus FROZEN (build once, reuse unchanged)."""
    NONE = L.PRECOND_NONE
    FRESH_SPAI = L.PRECOND_FRESH
    REUSE_CHAIN = L.PRECOND_REUSE_CHAIN
    REUSE_FROZEN = L.PRECOND_REUSE_FROZEN


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Vec:
    """Pointer + keep-alive for a host (numpy) or device (torch) vector."""

    def __init__(self, x, n: Optional[int] = None):
        if _is_torch(x):
            import torch
            t = x.detach()
            if t.dtype != torch.float64:
                t = t.to(torch.float64)
            self.obj = t.contiguous()
            self.p = self.obj.data_ptr()
            self.size = self.obj.numel()
            self.device = self.obj.device
        else:
            self.obj = L.f64(x).ravel()
            self.p = self.obj.ctypes.data
            self.size = self.obj.size
            self.device = None
        if n is not None and self.size != n:
            raise ValueError(f"dimension mismatch: expected {n} entries, got {self.size}")

    def empty_like(self, n: int):
        if self.device is not None:
            import torch
            return torch.empty(n, dtype=torch.float64, device=self.device)
        return np.empty(n, dtype=np.float64)


def _ptr(x) -> int:
    return x.data_ptr() if _is_torch(x) else x.ctypes.data


class SparseMatrix:
    """Immutable device CSR matrix (SparseMatrix, proj/include/morprec/sparse.hpp:33-101)."""

    def __init__(self, handle, keep=None):
        self._h = C.c_void_p(handle)
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.mpg_csr_info(self._h, C.byref(nr), C.byref(nc), C.byref(nz)))
        self._shape = (nr.value, nc.value)
        self._nnz = nz.value
        self._keep = keep

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.mpg_csr_destroy(h)
            self._h = None

    # -- construction -------------------------------------------------------
    @staticmethod
    def from_csr(nrows: int, ncols: int, row_offsets, col_indices, values, device: int = 0) -> "SparseMatrix":
        rp, ci, v = L.i64(row_offsets), L.i64(col_indices), L.f64(values)
        if rp.size != nrows + 1:
            raise ValueError("sparse: row_offsets length must be nrows + 1")
        if ci.size != v.size:
            raise ValueError("sparse: col_indices and values lengths differ")
        if rp[-1] != ci.size:
            raise ValueError("sparse: row_offsets must end at nnz")
        h = C.c_void_p()
        check(lib.mpg_csr_create(device, nrows, ncols, L.ptr(rp), L.ptr(ci), L.ptr(v), C.byref(h)))
        return SparseMatrix(h.value)

    @staticmethod
    def from_triplets(nrows: int, ncols: int, rows, cols, values, device: int = 0) -> "SparseMatrix":
        ri, ci, v = L.i64(rows), L.i64(cols), L.f64(values)
        if not (ri.size == ci.size == v.size):
            raise ValueError("sparse: triplet arrays differ in length")
        p = C.POINTER(L.HostCsr)()
        check(lib.mpg_host_csr_from_triplets(nrows, ncols, ri.size, L.ptr(ri), L.ptr(ci), L.ptr(v), C.byref(p)))
        hc = _take_host_csr(p)
        return SparseMatrix.from_csr(nrows, ncols, hc.rowptr, hc.colind, hc.val, device)

    @staticmethod
    def from_scipy(m, device: int = 0) -> "SparseMatrix":
        m = m.tocsr()
        m.sort_indices()
        m.sum_duplicates()
        return SparseMatrix.from_csr(m.shape[0], m.shape[1], m.indptr, m.indices, m.data, device)

    @staticmethod
    def from_dense(d, device: int = 0, drop_tol: float = 0.0) -> "SparseMatrix":
        d = np.asarray(d, dtype=np.float64)
        rows, cols = np.nonzero(np.abs(d) > drop_tol)
        return SparseMatrix.from_triplets(d.shape[0], d.shape[1], rows, cols, d[rows, cols], device)

    @staticmethod
    def identity(n: int, device: int = 0) -> "SparseMatrix":
        return SparseMatrix.from_csr(n, n, np.arange(n + 1), np.arange(n), np.ones(n), device)

    @staticmethod
    def diagonal(entries, device: int = 0) -> "SparseMatrix":
        e = L.f64(entries)
        n = e.size
        return SparseMatrix.from_csr(n, n, np.arange(n + 1), np.arange(n), e, device)

    @staticmethod
    def zero(nrows: int, ncols: int, device: int = 0) -> "SparseMatrix":
        return SparseMatrix.from_csr(nrows, ncols, np.zeros(nrows + 1, np.int64), np.zeros(0, np.int64),
                                     np.zeros(0), device)

    # -- queries ----------------------------------------------------------------
    def rows(self) -> int:
        return self._shape[0]

    def cols(self) -> int:
        return self._shape[1]

    @property
    def shape(self):
        return self._shape

    def nnz(self) -> int:
        return self._nnz

    def download(self):
        rp = np.empty(self._shape[0] + 1, np.int64)
        ci = np.empty(self._nnz, np.int64)
        v = np.empty(self._nnz, np.float64)
        check(lib.mpg_csr_download(self._h, L.ptr(rp), L.ptr(ci), L.ptr(v)))
        return rp, ci, v

    def to_dense(self, max_entries: int = 1 << 24) -> np.ndarray:
        if self._shape[0] * self._shape[1] > max_entries:
            raise ValueError("sparse to_dense: matrix too large to materialize")
        rp, ci, v = self.download()
        d = np.zeros(self._shape)
        for i in range(self._shape[0]):
            d[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
        return d

    def to_scipy(self):
        import scipy.sparse as sp
        rp, ci, v = self.download()
        return sp.csr_matrix((v, ci, rp), shape=self._shape)

    def multiply(self, x):
        """y = A x (sparse.cpp:236-249); throws ValueError on dimension mismatch."""
        xv = _Vec(x)
        if xv.size != self._shape[1]:
            raise ValueError("sparse multiply: dimension mismatch")
        y = xv.empty_like(self._shape[0])
        check(lib.mpg_csr_multiply(self._h, xv.p, _ptr(y)))
        return y

    def multiply_transpose(self, x):
        xv = _Vec(x)
        if xv.size != self._shape[0]:
            raise ValueError("sparse multiply_transpose: dimension mismatch")
        y = xv.empty_like(self._shape[1])
        check(lib.mpg_csr_multiply_transpose(self._h, xv.p, _ptr(y)))
        return y

    def transpose(self) -> "SparseMatrix":
        h = C.c_void_p()
        check(lib.mpg_csr_transpose(self._h, C.byref(h)))
        return SparseMatrix(h.value)

    def frobenius_norm(self) -> float:
        return float(lib.mpg_csr_frobenius_norm(self._h))


class ShiftedOperator:
    """sigma E - A formed on the fly (replaces linear_combination, qbihomm.cpp:164-171,
    and the N = 0 KroneckerOperator, kron.cpp:34-64). E None = identity."""

    def __init__(self, a: SparseMatrix, e: Optional[SparseMatrix] = None):
        h = C.c_void_p()
        check(lib.mpg_op_create(a._h, e._h if e is not None else None, C.byref(h)))
        self._h = h
        self.a, self.e = a, e
        self.n = int(lib.mpg_op_dim(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.mpg_op_destroy(h)
            self._h = None

    def apply(self, sigma: complex, x, transpose: bool = False):
        s = complex(sigma)
        n = self.n * (2 if s.imag != 0 else 1)
        xv = _Vec(x, n)
        y = xv.empty_like(n)
        check(lib.mpg_op_apply(self._h, s.real, s.imag, int(transpose), xv.p, _ptr(y)))
        return y

    def explicit(self, sigma: complex, transpose: bool = False) -> SparseMatrix:
        s = complex(sigma)
        h = C.c_void_p()
        check(lib.mpg_op_explicit(self._h, s.real, s.imag, int(transpose), C.byref(h)))
        return SparseMatrix(h.value)


@dataclasses.dataclass
class GmresConfig:
    """GmresConfig (proj/include/morprec/gmres.hpp:20-24)."""
    rel_tol: float = 1e-6
    max_iter: int = 1000
    record_history: bool = False

    def c(self) -> L.GmresCfg:
        return L.GmresCfg(self.rel_tol, self.max_iter, int(self.record_history))


@dataclasses.dataclass
class GmresReport:
    """GmresReport (proj/include/morprec/gmres.hpp:26-34)."""
    iterations: int = 0
    converged: bool = False
    breakdown: bool = False
    rhs_norm: float = 0.0
    final_residual: float = 0.0
    solve_seconds: float = 0.0
    residual_history: list = dataclasses.field(default_factory=list)
    reorth_passes: int = 0

    @staticmethod
    def of(r: L.GmresRep, hist=None) -> "GmresReport":
        h = list(hist[: r.history_len]) if hist is not None else []
        return GmresReport(r.iterations, bool(r.converged), bool(r.breakdown), r.rhs_norm, r.final_residual,
                           r.solve_seconds, h, r.reorth_passes)


@dataclasses.dataclass
class GmresResult:
    x: object
    report: GmresReport


@dataclasses.dataclass
class SpaiConfig:
    """SpaiConfig (proj/include/morprec/spai.hpp:15-33); pattern 'diagonal', 'a' (PatternOfA) or 'a_pow'
    (PatternOfAPow: the support of A e_j, ..., A^power e_j)."""
    pattern: str = "a"
    fill_tol: float = 1e-4
    max_fill_per_col: int = 50
    max_pattern_sweeps: int = 3
    threads: int = 1
    power: int = 2

    def c(self) -> L.SpaiCfg:
        kind = {"diagonal": 0, "a": 1, "a_pow": 2}[self.pattern]
        return L.SpaiCfg(kind, self.power, self.fill_tol, self.max_fill_per_col, self.max_pattern_sweeps,
                         self.threads)


class PrecondChain:
    """Immutable chain P, Q_1..Q_L applied as sequential SpMVs (chain.hpp:55-77)."""

    def __init__(self, base: Optional[SparseMatrix] = None, _handle=None, _factors=()):
        self._h = None
        if _handle is not None:
            self._h = C.c_void_p(_handle)
            self._factors = list(_factors)
        elif base is not None:
            h = C.c_void_p()
            check(lib.mpg_chain_create(base._h, C.byref(h)))
            self._h = h
            self._factors = [base]
        else:
            self._factors = []

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.mpg_chain_destroy(h)
            self._h = None

    def empty(self) -> bool:
        return self._h is None

    def length(self) -> int:
        return 0 if self._h is None else int(lib.mpg_chain_length(self._h))

    def dim(self) -> int:
        return self._factors[0].rows() if self._factors else 0

    def factor_id(self, i: int) -> int:
        return lib.mpg_chain_factor_id(self._h, i) or 0

    def extended(self, factor) -> "PrecondChain":
        if self._h is None:
            raise RuntimeError("chain: cannot extend an empty chain")
        q = factor.q if isinstance(factor, UpdateFactor) else factor
        if q is None:
            raise ValueError("chain: null update factor")
        h = C.c_void_p()
        check(lib.mpg_chain_extend(self._h, q._h, C.byref(h)))
        return PrecondChain(_handle=h.value, _factors=self._factors + [q])

    def apply(self, x):
        if self._h is None:
            raise RuntimeError("chain: apply on an empty chain")
        xv = _Vec(x, self.dim())
        y = xv.empty_like(self.dim())
        check(lib.mpg_chain_apply(self._h, xv.p, _ptr(y)))
        return y


@dataclasses.dataclass
class SpaiResult:
    """SpaiResult (proj/include/morprec/spai.hpp:43-48)."""
    p: SparseMatrix
    column_residuals: np.ndarray
    fallback_count: int
    build_seconds: float


@dataclasses.dataclass
class UpdateFactor:
    """UpdateFactor (proj/include/morprec/chain.hpp:33-42)."""
    q: SparseMatrix
    min_residual: float = 0.0
    matrix_change: float = 0.0
    build_seconds: float = 0.0
    fallback_count: int = 0


def spai_build(a: SparseMatrix, cfg: SpaiConfig = SpaiConfig()) -> SpaiResult:
    if a.rows() != a.cols():
        raise ValueError("spai_build: matrix must be square")
    res = np.empty(a.rows())
    p = C.c_void_p()
    fb = C.c_int64()
    secs = C.c_double()
    c = cfg.c()
    check(lib.mpg_spai_build(a._h, C.byref(c), C.byref(p), L.ptr(res), C.byref(fb), C.byref(secs)))
    return SpaiResult(SparseMatrix(p.value), res, fb.value, secs.value)


def spai_column_solve(a: SparseMatrix, col: int, pattern: Sequence[int]):
    """Fixed-pattern least squares for one column (spai.cpp:158-173): (rows, values, residual, rank_deficient)."""
    pat = np.sort(L.i64(pattern))
    vals = np.empty(pat.size)
    r = C.c_double()
    rd = C.c_int()
    check(lib.mpg_spai_column_solve(a._h, int(col), pat.size, L.ptr(pat), L.ptr(vals), C.byref(r), C.byref(rd)))
    return pat, vals, r.value, bool(rd.value)


def update_build(a_prev: SparseMatrix, a_new: SparseMatrix, cfg: SpaiConfig = SpaiConfig()) -> UpdateFactor:
    if a_prev.shape != a_new.shape:
        raise ValueError("update_build: shape mismatch")
    q = C.c_void_p()
    mr, mc, secs = C.c_double(), C.c_double(), C.c_double()
    fb = C.c_int64()
    c = cfg.c()
    check(lib.mpg_update_build(a_prev._h, a_new._h, C.byref(c), C.byref(q), C.byref(mr), C.byref(mc), C.byref(fb),
                               C.byref(secs)))
    return UpdateFactor(SparseMatrix(q.value), mr.value, mc.value, secs.value, fb.value)


def standard_residual(a: SparseMatrix, chain: PrecondChain) -> float:
    out = C.c_double()
    check(lib.mpg_standard_residual(a._h, chain._h, C.byref(out)))
    return out.value


def _gmres_common(call, b, cfg: GmresConfig):
    bv = _Vec(b)
    x = bv.empty_like(bv.size)
    rep = L.GmresRep()
    c = cfg.c()
    hist = np.empty(cfg.max_iter + 2) if cfg.record_history else None
    check(call(bv.p, _ptr(x), C.byref(c), C.byref(rep), L.ptr(hist) if hist is not None else None))
    return GmresResult(x, GmresReport.of(rep, hist))


def gmres_right_preconditioned(a: SparseMatrix, chain: Optional[PrecondChain], b,
                               cfg: GmresConfig = GmresConfig()) -> GmresResult:
    """Full right-preconditioned GMRES on A P xt = b, x = P xt (gmres.cpp:40-186).
    `a` is a SparseMatrix (matvec_operator); chain None is identity_operator()."""
    bv = _Vec(b)
    if bv.size != a.rows():
        raise ValueError("gmres: dimension mismatch")
    ch = chain._h if chain is not None and not chain.empty() else None
    return _gmres_common(lambda bp, xp, c, r, h: lib.mpg_gmres_csr(a._h, ch, bp, xp, c, r, h), b, cfg)


def gmres_shifted(op: ShiftedOperator, sigma: complex, b, chain: Optional[PrecondChain] = None,
                  transpose: bool = False, cfg: GmresConfig = GmresConfig()) -> GmresResult:
    """GMRES on (sigma E - A) (or its transpose side / pair form) with a chain preconditioner."""
    s = complex(sigma)
    ch = chain._h if chain is not None and not chain.empty() else None
    return _gmres_common(lambda bp, xp, c, r, h: lib.mpg_gmres_shifted(op._h, s.real, s.imag, int(transpose), ch, bp,
                                                                       xp, c, r, h), b, cfg)


def gmres_batch(op: ShiftedOperator, sigmas: Sequence[complex], bs: Sequence, chains=None, transposes=None,
                cfg: GmresConfig = GmresConfig()):
    """Independent shifted solves advanced in lockstep on one device."""
    k = len(sigmas)
    sre = np.array([complex(s).real for s in sigmas])
    sim = np.array([complex(s).imag for s in sigmas])
    tr = np.array([int(t) for t in (transposes or [0] * k)], dtype=np.int32)
    bvs = [_Vec(b) for b in bs]
    xs = [bv.empty_like(bv.size) for bv in bvs]
    bp = (C.c_void_p * k)(*[bv.p for bv in bvs])
    xp = (C.c_void_p * k)(*[_ptr(x) for x in xs])
    chs = (C.c_void_p * k)(*[(c._h.value if c is not None and not c.empty() else None) for c in (chains or [None] * k)])
    reps = (L.GmresRep * k)()
    c = cfg.c()
    check(lib.mpg_gmres_batch(op._h, k, L.ptr(sre), L.ptr(sim), tr.ctypes.data, chs, bp, xp, C.byref(c), reps))
    return [GmresResult(xs[i], GmresReport.of(reps[i])) for i in range(k)]


@dataclasses.dataclass
class ReportRow:
    """ReportRow (proj/include/morprec/report.hpp:28-40)."""
    sweep: int
    point: int
    kind: str
    solves: int
    gmres_iterations: int
    precond_build_seconds: float
    gmres_seconds: float
    min_residual: float
    matrix_change: float
    standard_residual: float

    @staticmethod
    def of(r: L.ReportRow) -> "ReportRow":
        return ReportRow(r.sweep, r.point, L.KIND_NAMES.get(r.kind, "none"), r.solves, r.iterations, r.build_seconds,
                         r.gmres_seconds, r.min_residual, r.matrix_change, r.standard_residual)


@dataclasses.dataclass
class ReductionReport:
    rows: list
    converged: bool = False
    reduced_order: int = 0
    sweeps: int = 0
    warnings: list = dataclasses.field(default_factory=list)

    def totals(self):
        return dict(solves=sum(r.solves for r in self.rows),
                    precond_build_seconds=sum(r.precond_build_seconds for r in self.rows),
                    gmres_iterations=sum(r.gmres_iterations for r in self.rows),
                    gmres_seconds=sum(r.gmres_seconds for r in self.rows))

    def write_csv(self, f) -> None:
        """ReductionReport::write_csv (report.cpp:46-63): header, one line per row, TOTAL line; the text is
        produced by the library's C++ writer (default ostream formatting, byte-identical to the reference's)."""
        rows = (L.ReportRow * max(1, len(self.rows)))()
        kinds = {v: k for k, v in L.KIND_NAMES.items()}
        for i, r in enumerate(self.rows):
            rows[i] = L.ReportRow(r.sweep, r.point, kinds.get(r.kind, 0), r.solves, r.gmres_iterations,
                                  r.precond_build_seconds, r.gmres_seconds, r.min_residual, r.matrix_change,
                                  r.standard_residual)
        f.write(_take_text(lambda b, n: lib.mpg_report_csv(rows, len(self.rows), b, n)))


@dataclasses.dataclass
class IrkaConfig:
    """BirkaConfig (proj/include/morprec/birka.hpp:49-61) for N = 0."""
    r: int = 2
    tol: float = 1e-4
    max_sweeps: int = 50
    seed: int = 1
    gmres: GmresConfig = dataclasses.field(default_factory=lambda: GmresConfig(1e-10, 1000, False))
    spai: SpaiConfig = dataclasses.field(default_factory=SpaiConfig)
    max_chain_len: int = 16
    explicit_nnz_cap: int = 200000
    standard_residual_max_dim: int = 5000
    mirror_unstable: bool = False  # extension: reflect unstable reduced poles before solving

    def c(self) -> L.IrkaCfg:
        return L.IrkaCfg(self.r, self.tol, self.max_sweeps, 1, self.seed, self.gmres.c(), self.spai.c(),
                         self.max_chain_len, self.explicit_nnz_cap, self.standard_residual_max_dim,
                         int(self.mirror_unstable))


@dataclasses.dataclass
class IrkaState:
    """Reduced model E_r x' = A_r x + B_r u, y = C_r^T x with K_r = E_r^{-1} A_r (BirkaState, birka.hpp:35-47)."""
    kr: np.ndarray
    fr: np.ndarray
    cr: np.ndarray
    er: Optional[np.ndarray]
    ar: Optional[np.ndarray]
    lam: np.ndarray
    v: Optional[np.ndarray]
    w: Optional[np.ndarray]
    sweeps: int

    def transfer(self, s: complex) -> np.ndarray:
        """H_r(s) = C_r^T (s I - K_r)^{-1} f_r, q x m."""
        r = self.kr.shape[0]
        return self.cr.T @ np.linalg.solve(s * np.eye(r) - self.kr, self.fr)


def project(op: ShiftedOperator, v, w):
    """IRKA's projection step (birka.cpp:283-291, E-generalised): returns (E_r, A_r) = (W^T E V, W^T A V)."""
    vm = np.asfortranarray(np.asarray(v, dtype=np.float64))
    wm = np.asfortranarray(np.asarray(w, dtype=np.float64))
    if vm.shape != wm.shape or vm.ndim != 2 or vm.shape[0] != op.n:
        raise ValueError("project: V and W must both be n x r")
    r = vm.shape[1]
    er, ar = np.zeros((r, r), order="F"), np.zeros((r, r), order="F")
    check(lib.mpg_project(op._h, L.ptr(vm), L.ptr(wm), r, L.ptr(er), L.ptr(ar)))
    return er, ar


def _rows(buf, n):
    return [ReportRow.of(buf[i]) for i in range(n)]


def irka_reduce(op: ShiftedOperator, b, c, cfg: IrkaConfig, mode: int = PrecondMode.REUSE_CHAIN,
                init_shifts=None, want_bases: bool = False, init=None):
    """IRKA (BIRKA with N = 0, birka.cpp:139-310) on the GPU; returns (IrkaState, ReductionReport).
    `init` = (kr, fr, cr), any part None: the reference's initial `BirkaState` (birka.hpp:78-80)."""
    if init is not None:
        if init_shifts is not None or want_bases:
            raise ValueError("irka_reduce: init excludes init_shifts and want_bases")
        return _irka_reduce_from(op, b, c, cfg, mode, init)
    n = op.n
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
    rows = (L.ReportRow * maxrows)()
    ini = L.f64(init_shifts) if init_shifts is not None else None
    cc = cfg.c()
    check(lib.mpg_irka_reduce(op._h, L.ptr(bm), m, L.ptr(cm), q, C.byref(cc), mode,
                              L.ptr(ini) if ini is not None else None, L.ptr(kr), L.ptr(fr), L.ptr(cr), L.ptr(er),
                              L.ptr(ar), L.ptr(lre), L.ptr(lim), L.ptr(v) if v is not None else None,
                              L.ptr(w) if w is not None else None, C.byref(sweeps), C.byref(conv), rows, maxrows,
                              C.byref(nrows)))
    st = IrkaState(kr, fr, cr, er, ar, lre + 1j * lim, v, w, sweeps.value)
    rep = ReductionReport(_rows(rows, min(nrows.value, maxrows)), bool(conv.value), r, sweeps.value)
    if not rep.converged:
        rep.warnings.append(f"fixed point left unconverged after {sweeps.value} sweeps")
    return st, rep


def _irka_reduce_from(op, b, c, cfg, mode, init):
    n = op.n
    bm = np.asfortranarray(np.asarray(b, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    m, q, r = bm.shape[1], cm.shape[1], cfg.r
    shapes = ((r, r), (r, m), (r, q))
    ini = []
    for part, shape, name in zip(init, shapes, ("kr", "fr", "cr")):
        if part is None:
            ini.append(None)
            continue
        a = np.asfortranarray(np.asarray(part, dtype=np.float64))
        if a.shape != shape:
            raise ValueError(f"irka_reduce: initial {name} must be {shape[0]} x {shape[1]}")
        ini.append(a)
    kr, er, ar = (np.zeros((r, r), order="F") for _ in range(3))
    fr, cr = np.zeros((r, m), order="F"), np.zeros((r, q), order="F")
    lre, lim = np.zeros(r), np.zeros(r)
    sweeps, conv, nrows = C.c_int(), C.c_int(), C.c_int()
    maxrows = 2 * r * max(cfg.max_sweeps, 1) + 8
    rows = (L.ReportRow * maxrows)()
    cc = cfg.c()
    check(lib.mpg_irka_reduce_from(op._h, L.ptr(bm), m, L.ptr(cm), q, C.byref(cc), mode,
                                   *[L.ptr(a) if a is not None else None for a in ini], L.ptr(kr), L.ptr(fr),
                                   L.ptr(cr), L.ptr(er), L.ptr(ar), L.ptr(lre), L.ptr(lim), C.byref(sweeps),
                                   C.byref(conv), rows, maxrows, C.byref(nrows)))
    st = IrkaState(kr, fr, cr, er, ar, lre + 1j * lim, None, None, sweeps.value)
    rep = ReductionReport(_rows(rows, min(nrows.value, maxrows)), bool(conv.value), r, sweeps.value)
    if not rep.converged:
        rep.warnings.append(f"fixed point left unconverged after {sweeps.value} sweeps")
    return st, rep


@dataclasses.dataclass
class BirkaState:
    """Reduced bilinear model x' = K_r x + sum_j N_r[j] x u_j + F_r u, y = C_r^T x (BirkaState, birka.hpp:35-47)."""
    kr: np.ndarray
    nr: list
    fr: np.ndarray
    cr: np.ndarray
    lam: np.ndarray
    v: Optional[np.ndarray]
    w: Optional[np.ndarray]
    sweeps: int


def birka_reduce(k: SparseMatrix, n_ops: Sequence[SparseMatrix], b, c, cfg: IrkaConfig,
                 mode: int = PrecondMode.REUSE_CHAIN, want_bases: bool = False):
    """birka_reduce (birka.cpp:139-310) with couplings N_j: one joint n r GMRES per side and sweep on the
    device, on the explicitly assembled Kronecker operator (kron.cpp:72-131); returns (BirkaState,
    ReductionReport) with report.warnings (e.g. a side degraded past cfg.explicit_nnz_cap)."""
    n = k.shape[0]
    bm = np.asfortranarray(np.asarray(b, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    m, q, r = bm.shape[1], cm.shape[1], cfg.r
    if len(n_ops) != m:
        raise ValueError("birka_reduce: one coupling matrix per input column is required")
    kr = np.zeros((r, r), order="F")
    nr = np.zeros(r * r * max(m, 1))
    fr, cr = np.zeros((r, m), order="F"), np.zeros((r, q), order="F")
    lre, lim = np.zeros(r), np.zeros(r)
    v = np.zeros((n, r), order="F") if want_bases else None
    w = np.zeros((n, r), order="F") if want_bases else None
    sweeps, conv, nrows = C.c_int(), C.c_int(), C.c_int()
    maxrows = 2 * max(cfg.max_sweeps, 1) + 4
    rows = (L.ReportRow * maxrows)()
    warn = C.c_void_p()
    hs = (C.c_void_p * max(m, 1))(*[x._h.value for x in n_ops])
    cc = cfg.c()
    check(lib.mpg_birka_reduce(k._h, hs, L.ptr(bm), m, L.ptr(cm), q, C.byref(cc), mode, L.ptr(kr), L.ptr(nr),
                               L.ptr(fr), L.ptr(cr), L.ptr(lre), L.ptr(lim), L.ptr(v) if v is not None else None,
                               L.ptr(w) if w is not None else None, C.byref(sweeps), C.byref(conv), rows, maxrows,
                               C.byref(nrows), C.byref(warn)))
    try:
        text = C.string_at(warn.value).decode() if warn.value else ""
    finally:
        lib.mpg_buffer_free(warn)
    nrs = [nr[j * r * r:(j + 1) * r * r].reshape((r, r), order="F").copy() for j in range(m)]
    st = BirkaState(kr, nrs, fr, cr, lre + 1j * lim, v, w, sweeps.value)
    rep = ReductionReport(_rows(rows, min(nrows.value, maxrows)), bool(conv.value), r, sweeps.value,
                          [x for x in text.split("\n") if x])
    return st, rep


@dataclasses.dataclass
class SweepResult:
    """SpaiBenchResult (proj/include/morprec/bench.hpp:46-49)."""
    report: ReductionReport
    failed_solves: int
    x: Optional[np.ndarray] = None


def run_spai_bench(op: ShiftedOperator, b, points: Sequence[float], spai: SpaiConfig = SpaiConfig(),
                   gmres: GmresConfig = GmresConfig(), mode: int = PrecondMode.REUSE_CHAIN, max_chain_len: int = 16,
                   keep_solutions: bool = False) -> SweepResult:
    """Shift-sweep solve benchmark (bench.cpp:159-249) on sigma_i E - A."""
    n = op.n
    bv = _Vec(b, n)
    pts = L.f64(points)
    x = np.zeros((len(pts), n)) if keep_solutions else None
    rows = (L.ReportRow * max(len(pts), 1))()
    nrows, failed = C.c_int(), C.c_int()
    s, g = spai.c(), gmres.c()
    check(lib.mpg_spai_bench(op._h, bv.p, len(pts), L.ptr(pts), C.byref(s), C.byref(g), mode, max_chain_len,
                             L.ptr(x) if x is not None else None, rows, len(pts), C.byref(nrows), C.byref(failed)))
    rep = ReductionReport(_rows(rows, nrows.value), failed.value == 0, 0, 1)
    return SweepResult(rep, failed.value, x)


# ---- QB-IHOMM (proj/include/morprec/qbihomm.hpp, proj/src/qbihomm.cpp) ---------------
@dataclasses.dataclass
class QbSystem:
    """D x' = K x + H (x (x) x) + N x u + F u, y = C^T x (qbihomm.hpp:15-33).

    d, k, n_op: n x n SparseMatrix on the device; h: the n x n^2 quadratic term
    as triplets (rows, cols = b n + c, values); f, c: n-vectors (SISO).
    create() validates shapes as QbSystem::create does (qbihomm.cpp:17-43)."""
    d: SparseMatrix
    k: SparseMatrix
    n_op: SparseMatrix
    h_rows: np.ndarray
    h_cols: np.ndarray
    h_vals: np.ndarray
    f: np.ndarray
    c: np.ndarray

    @staticmethod
    def create(d: SparseMatrix, k: SparseMatrix, n_op: SparseMatrix, h, f, c) -> "QbSystem":
        n = d.rows()
        if d.cols() != n:
            raise ConfigError("quadratic-bilinear system: D must be square")
        if k.shape != (n, n):
            raise ConfigError("quadratic-bilinear system: K must be n x n")
        if n_op.shape != (n, n):
            raise ConfigError("quadratic-bilinear system: N must be n x n")
        if isinstance(h, tuple):
            hr, hc, hv, hshape = (*h, (n, n * n)) if len(h) == 3 else h
        else:  # scipy-like or host CSR with nrows/ncols/rowptr/colind/val
            hshape = (h.nrows, h.ncols)
            hr = np.repeat(np.arange(h.nrows, dtype=np.int64), np.diff(h.rowptr))
            hc, hv = h.colind, h.val
        if tuple(hshape) != (n, n * n):
            raise ConfigError(f"quadratic-bilinear system: H must be n x n^2 (got {hshape[0]} x {hshape[1]})")
        for name, v in (("F", f), ("C", c)):
            a = np.asarray(v)
            if (a.ndim == 2 and a.shape[1] != 1) or a.size != n:
                raise ConfigError(f"quadratic-bilinear system: {name} must be a single n-column (SISO)")
        return QbSystem(d, k, n_op, L.i64(hr), L.i64(hc), L.f64(hv), L.f64(f).reshape(-1), L.f64(c).reshape(-1))

    def dim(self) -> int:
        return self.d.rows()


@dataclasses.dataclass
class QbConfig:
    """QbConfig (qbihomm.hpp:35-43)."""
    sigmas: Sequence[float] = ()
    p_moments: int = 1
    q_moments: int = 1
    gmres: GmresConfig = dataclasses.field(default_factory=GmresConfig)
    spai: SpaiConfig = dataclasses.field(default_factory=SpaiConfig)
    max_chain_len: int = 16
    standard_residual_max_dim: int = 5000

    def c(self) -> L.QbCfg:
        return L.QbCfg(self.p_moments, self.q_moments, self.gmres.c(), self.spai.c(), self.max_chain_len,
                       self.standard_residual_max_dim)


@dataclasses.dataclass
class ReducedQb:
    """ReducedQb (qbihomm.hpp:45-52): r x r matrices, h r x r^2, f, c r x 1, basis n x r."""
    d: np.ndarray
    k: np.ndarray
    n_op: np.ndarray
    h: np.ndarray
    f: np.ndarray
    c: np.ndarray
    basis: np.ndarray

    def order(self) -> int:
        return self.d.shape[0]

    def linear_transfer(self, s: float) -> float:
        return float(self.c[:, 0] @ np.linalg.solve(s * self.d - self.k, self.f[:, 0]))


def qbihomm_reduce(sys: QbSystem, cfg: QbConfig, mode: int = PrecondMode.REUSE_CHAIN):
    """qbihomm_reduce (qbihomm.cpp:144-208) on the GPU; returns (ReducedQb, ReductionReport)."""
    n = sys.dim()
    op = ShiftedOperator(sys.k, sys.d)
    sig = L.f64(cfg.sigmas)
    cap = max(1, len(sig) * (cfg.p_moments + 2 * cfg.q_moments + 2))
    basis = np.zeros((n, cap), order="F")
    rd, rk, rn = (np.zeros(cap * cap) for _ in range(3))
    rh = np.zeros(cap * cap * cap)
    rf, rc = np.zeros(cap), np.zeros(cap)
    order, nrows = C.c_int(), C.c_int()
    maxrows = 4 * max(1, len(sig))
    rows = (L.ReportRow * maxrows)()
    qc = cfg.c()
    check(lib.mpg_qbihomm_reduce(op._h, sys.n_op._h, sys.h_vals.size, L.ptr(sys.h_rows), L.ptr(sys.h_cols),
                                 L.ptr(sys.h_vals), L.ptr(sys.f), L.ptr(sys.c), len(sig), L.ptr(sig), C.byref(qc), mode,
                                 cap, C.byref(order), L.ptr(basis), L.ptr(rd), L.ptr(rk), L.ptr(rn), L.ptr(rh),
                                 L.ptr(rf), L.ptr(rc), rows, maxrows, C.byref(nrows)))
    r = order.value
    sq = lambda a, cc: a[: r * cc].reshape((r, cc), order="F").copy()
    red = ReducedQb(sq(rd, r), sq(rk, r), sq(rn, r), sq(rh, r * r), rf[:r].reshape(r, 1).copy(),
                    rc[:r].reshape(r, 1).copy(), np.asfortranarray(basis.reshape(-1, order="F")[: n * r].reshape((n, r), order="F")))
    rep = ReductionReport(_rows(rows, min(nrows.value, maxrows)), True, r, 1)
    return red, rep


# ---- Matrix Market IO (proj/include/morprec/matrix_market.hpp, proj/src/matrix_market.cpp) ------
def _take_text(call) -> str:
    buf, n = C.c_void_p(), C.c_int64()
    check(call(C.byref(buf), C.byref(n)))
    try:
        return C.string_at(buf.value, n.value).decode()
    finally:
        lib.mpg_buffer_free(buf)


def _host_csr_struct(a):
    """(HostCsr struct, keep-alive arrays) for a gen.HostCsr / scipy matrix / SparseMatrix."""
    if isinstance(a, SparseMatrix):
        rp, ci, v = a.download()
        nr, nc = a.shape
    elif hasattr(a, "rowptr"):
        rp, ci, v, nr, nc = a.rowptr, a.colind, a.val, a.nrows, a.ncols
    else:
        m = a.tocsr()
        rp, ci, v, (nr, nc) = m.indptr, m.indices, m.data, m.shape
    rp, ci, v = L.i64(rp), L.i64(ci), L.f64(v)
    h = L.HostCsr(nr, nc, int(rp[-1]) if rp.size else 0, rp.ctypes.data_as(C.POINTER(C.c_int64)),
                  ci.ctypes.data_as(C.POINTER(C.c_int64)), v.ctypes.data_as(C.POINTER(C.c_double)))
    return h, (rp, ci, v)


def _take_host_csr(p):
    """Copy a library-owned mpg_host_csr into numpy arrays (HostCsr) and free it."""
    from .gen import HostCsr
    h = p.contents
    nr, nnz = h.nrows, h.nnz
    out = HostCsr(h.nrows, h.ncols, np.ctypeslib.as_array(h.rowptr, (nr + 1,)).copy(),
                  np.ctypeslib.as_array(h.colind, (max(nnz, 1),))[:nnz].copy(),
                  np.ctypeslib.as_array(h.val, (max(nnz, 1),))[:nnz].copy())
    lib.mpg_host_csr_free(p)
    return out


def _from_host(p, device: Optional[int]):
    host = _take_host_csr(p)
    if device is None:
        return host
    return SparseMatrix.from_csr(host.nrows, host.ncols, host.rowptr, host.colind, host.val, device)


def read_matrix_market(text, origin: str = "<stream>", threads: int = 0, device: Optional[int] = 0):
    """read_matrix_market (matrix_market.cpp:38-98): coordinate real general|symmetric text; symmetric storage
    expanded, duplicates summed; malformed input raises IoError("origin:line: ..."). Parsed by `threads` host
    threads (0: all). Returns a SparseMatrix on `device`, or the host CSR (gen.HostCsr) with device=None."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    p = C.POINTER(L.HostCsr)()
    check(lib.mpg_mm_read_buffer(data, len(data), origin.encode(), threads, C.byref(p)))
    return _from_host(p, device)


def read_matrix_market_file(path, threads: int = 0, device: Optional[int] = 0):
    """read_matrix_market_file (matrix_market.cpp:93-97)."""
    p = C.POINTER(L.HostCsr)()
    check(lib.mpg_mm_read_file(str(path).encode(), threads, C.byref(p)))
    return _from_host(p, device)


def write_matrix_market(a, threads: int = 0) -> str:
    """write_matrix_market (matrix_market.cpp:100-142): general, row-major, shortest round-trip values;
    a dense ndarray stores every entry (zeros included)."""
    if isinstance(a, np.ndarray):
        d = np.asfortranarray(a, dtype=np.float64)
        if d.ndim != 2:
            raise ValueError("write_matrix_market: dense blocks must be 2-D")
        return _take_text(lambda b, n: lib.mpg_mm_write_dense_buffer(d.shape[0], d.shape[1], d.ctypes.data, b, n))
    h, keep = _host_csr_struct(a)
    return _take_text(lambda b, n: lib.mpg_mm_write_buffer(C.byref(h), threads, b, n))


def write_matrix_market_file(path, a, threads: int = 0) -> None:
    if isinstance(a, np.ndarray):
        text = write_matrix_market(a)
        try:
            with open(path, "w") as f:
                f.write(text)
        except OSError as e:
            raise IoError(f"cannot open '{path}' for writing") from e
        return
    h, keep = _host_csr_struct(a)
    check(lib.mpg_mm_write_file(str(path).encode(), C.byref(h), threads))


# ---- second-order models (proj/include/morprec/airga.hpp) --------------------------------------
@dataclasses.dataclass
class SecondOrderSystem:
    """M x'' + D x' + K x = F u, y = C^T x (airga.hpp:17-41); m, d, k device SparseMatrix, f (n x n_in) and
    c (n x n_out) dense host arrays."""
    m: SparseMatrix
    d: SparseMatrix
    k: SparseMatrix
    f: np.ndarray
    c: np.ndarray
    alpha: float = 0.0
    beta: float = 0.0

    @staticmethod
    def create(m, d, k, f, c, alpha: float = 0.0, beta: float = 0.0) -> "SecondOrderSystem":
        n = m.rows()
        for name, x in (("M", m), ("D", d), ("K", k)):
            if x.shape != (n, n):
                raise ConfigError(f"second-order system: {name} must be n x n")
        f = np.asfortranarray(np.asarray(f, dtype=np.float64).reshape(n, -1))
        c = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
        return SecondOrderSystem(m, d, k, f, c, alpha, beta)

    @staticmethod
    def with_proportional_damping(m, k, f, c, alpha: float, beta: float) -> "SecondOrderSystem":
        """D = alpha M + beta K, formed exactly (airga.cpp:62-72)."""
        mr, kr = m.download(), k.download()
        import scipy.sparse as sp
        ms = sp.csr_matrix((mr[2], mr[1], mr[0]), shape=m.shape)
        ks = sp.csr_matrix((kr[2], kr[1], kr[0]), shape=k.shape)
        ds = (alpha * ms + beta * ks).tocsr()
        ds.eliminate_zeros()
        d = SparseMatrix.from_csr(ds.shape[0], ds.shape[1], ds.indptr, ds.indices, ds.data)
        return SecondOrderSystem.create(m, d, k, f, c, alpha, beta)

    def dim(self) -> int:
        return self.m.rows()


@dataclasses.dataclass
class ReducedSecondOrder:
    """airga.hpp:64-71: r x r m, d, k; r x n_in f; r x n_out c."""
    m: np.ndarray
    d: np.ndarray
    k: np.ndarray
    f: np.ndarray
    c: np.ndarray
    basis: Optional[np.ndarray] = None

    def order(self) -> int:
        return self.m.shape[0]


@dataclasses.dataclass
class TransferErrorConfig:
    """airga.hpp:91-96."""
    gmres: GmresConfig = dataclasses.field(default_factory=lambda: GmresConfig(1e-10, 1000))
    spai: SpaiConfig = dataclasses.field(default_factory=SpaiConfig)
    mode: int = PrecondMode.REUSE_CHAIN
    max_chain_len: int = 16


def transfer_function_error(sys: SecondOrderSystem, red: ReducedSecondOrder, s_grid,
                            cfg: TransferErrorConfig = TransferErrorConfig()) -> np.ndarray:
    """||H(s) - H_r(s)|| / ||H(s)|| on s_grid (airga.cpp:386-447), full order on the GPU; NaN where undefined."""
    f64 = lambda x: np.asfortranarray(np.asarray(x, dtype=np.float64))
    r = red.order()
    rm, rd, rk = f64(red.m), f64(red.d), f64(red.k)
    rf, rc = f64(np.reshape(red.f, (r, -1))), f64(np.reshape(red.c, (r, -1)))
    g = L.f64(s_grid)
    out = np.zeros(g.size)
    its = C.c_longlong()
    gc, sc = cfg.gmres.c(), cfg.spai.c()
    check(lib.mpg_transfer_function_error(sys.m._h, sys.d._h, sys.k._h, L.ptr(sys.f), sys.f.shape[1], L.ptr(sys.c),
                                          sys.c.shape[1], L.ptr(rm), L.ptr(rd), L.ptr(rk), L.ptr(rf), L.ptr(rc), r,
                                          L.ptr(g), g.size, C.byref(gc), C.byref(sc), cfg.mode, cfg.max_chain_len,
                                          L.ptr(out), C.byref(its)))
    return out


@dataclasses.dataclass
class AirgaConfig:
    """AirgaConfig (airga.hpp:43-62)."""
    expansion_points: Sequence[float] = ()
    r_max: int = 20
    outer_tol: float = 1e-4
    inner_tol: float = 1e-6
    max_outer: int = 20
    gmres: GmresConfig = dataclasses.field(default_factory=GmresConfig)
    spai: SpaiConfig = dataclasses.field(default_factory=SpaiConfig)
    max_chain_len: int = 16
    standard_residual_max_dim: int = 5000

    def c(self) -> L.AirgaCfg:
        return L.AirgaCfg(self.r_max, self.outer_tol, self.inner_tol, self.max_outer, self.gmres.c(), self.spai.c(),
                          self.max_chain_len, self.standard_residual_max_dim)


def airga_reduce(sys: SecondOrderSystem, cfg: AirgaConfig, mode: int = PrecondMode.REUSE_CHAIN):
    """airga_reduce (airga.cpp:136-317): full-order solves on the GPU; returns (ReducedSecondOrder,
    ReductionReport) with report.warnings and report.final_points."""
    n = sys.dim()
    n_in, n_out = sys.f.shape[1], sys.c.shape[1]
    cap = max(1, cfg.r_max)
    pts = L.f64(cfg.expansion_points)
    rm, rd, rk = (np.zeros(cap * cap) for _ in range(3))
    rf, rc = np.zeros(cap * n_in), np.zeros(cap * n_out)
    basis = np.zeros(n * cap)
    fp = np.zeros(max(1, pts.size))
    order, sweeps, conv, nrows = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    maxrows = 2 * max(1, pts.size) * max(1, cfg.max_outer) + 4
    rows = (L.ReportRow * maxrows)()
    warn = C.c_void_p()
    ac = cfg.c()
    check(lib.mpg_airga_reduce(sys.m._h, sys.d._h, sys.k._h, L.ptr(sys.f), n_in, L.ptr(sys.c), n_out, sys.alpha,
                               sys.beta, L.ptr(pts), pts.size, C.byref(ac), mode, C.byref(order), L.ptr(rm), L.ptr(rd),
                               L.ptr(rk), L.ptr(rf), L.ptr(rc), L.ptr(basis), L.ptr(fp), C.byref(sweeps), C.byref(conv),
                               rows, maxrows, C.byref(nrows), C.byref(warn)))
    try:
        text = C.string_at(warn.value).decode() if warn.value else ""
    finally:
        lib.mpg_buffer_free(warn)
    r = order.value
    sq = lambda a, rr, cc: a[: rr * cc].reshape((rr, cc), order="F").copy()
    red = ReducedSecondOrder(sq(rm, r, r), sq(rd, r, r), sq(rk, r, r), sq(rf, r, n_in), sq(rc, r, n_out),
                             sq(basis, n, r))
    rep = ReductionReport(_rows(rows, min(nrows.value, maxrows)), bool(conv.value), r, sweeps.value,
                          [w for w in text.split("\n") if w])
    rep.final_points = fp[: pts.size].tolist()
    return red, rep


def update_expansion_points(m, d, k, current) -> list:
    """update_expansion_points (airga.cpp:319-384) for a reduced pencil."""
    mm, dd, kk = (np.asfortranarray(np.asarray(x, dtype=np.float64)) for x in (m, d, k))
    cur = L.f64(current)
    out = np.zeros(max(1, cur.size))
    check(lib.mpg_update_expansion_points(L.ptr(mm), L.ptr(dd), L.ptr(kk), mm.shape[0], L.ptr(cur), cur.size,
                                          L.ptr(out)))
    return out[: cur.size].tolist()


def h2_norm(a, b, c) -> float:
    """h2_norm (proj/src/h2.cpp:28-60) of x' = A x + B u, y = C x; inf when A is not stable."""
    aa, bb, cc = (np.asfortranarray(np.atleast_2d(np.asarray(x, dtype=np.float64))) for x in (a, b, c))
    out = C.c_double()
    check(lib.mpg_h2_norm(L.ptr(aa), L.ptr(bb), L.ptr(cc), aa.shape[0], bb.shape[1], cc.shape[0], C.byref(out)))
    return out.value

