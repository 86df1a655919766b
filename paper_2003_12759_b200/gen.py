"""Seeded synthetic inputs (include/mpg_gen.h, csrc/gen/generators.cpp) as numpy arrays.

The five BASELINE.json configs and the reference's own test
fixtures (proj/tests/support.hpp:18-49, proj/src/generator.cpp:37-207).
These run on the host and need no GPU. Test/bench fixtures, not the product:
the functions bind to libmpggen.so next to this file, never to libmpg.so.
This file imports nothing from its package, so oracle/gen.py can execute it
bound to oracle/liboracle.so (which compiles the same generator source) and
the CPU reference arm maps no library outside oracle/.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

# Set before the first call to bind another library exporting include/mpg_gen.h.
LIBPATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmpggen.so")


class HostCsrS(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64), ("rowptr", C.POINTER(C.c_int64)),
                ("colind", C.POINTER(C.c_int64)), ("val", C.POINTER(C.c_double))]


class HostSystemS(C.Structure):
    _fields_ = [("n", C.c_int64), ("a", C.POINTER(HostCsrS)), ("e", C.POINTER(HostCsrS)),
                ("e_diag", C.POINTER(C.c_double)), ("m", C.c_int), ("q", C.c_int), ("r", C.c_int),
                ("b", C.POINTER(C.c_double)), ("c", C.POINTER(C.c_double)), ("shifts", C.POINTER(C.c_double))]


_vp, _I, _D, _L, _U = C.c_void_p, C.c_int, C.c_double, C.c_int64, C.c_uint64
_PC, _PS = C.POINTER(C.POINTER(HostCsrS)), C.POINTER(C.POINTER(HostSystemS))
_SIGS = {
    "mpg_gen_last_error": (C.c_char_p, []),
    "mpg_gen_csr_free": (None, [C.POINTER(HostCsrS)]),
    "mpg_gen_system_free": (None, [C.POINTER(HostSystemS)]),
    "mpg_gen_random_dense": (_I, [_L, _L, _U, _vp]),
    "mpg_gen_random_sparse": (_I, [_L, _L, _D, _U, _D, _PC]),
    "mpg_gen_from_triplets": (_I, [_L, _L, _L, _vp, _vp, _vp, _PC]),
    "mpg_gen_bilinear_toy": (_I, [_L, _L, _U, _PC, _vp, _vp]),
    "mpg_gen_disc_brake": (_I, [_L, _D, _U, _PC, _PC]),
    "mpg_gen_bilinear_toy_n": (_I, [_L, _L, _U, _PC, _vp, _vp, _vp]),
    "mpg_gen_qb_toy": (_I, [_L, _U] + [_PC] * 4),
    "mpg_gen_grid2d": (_I, [_L, _U, _PS]),
    "mpg_gen_convdiff3d": (_I, [_L, _U, _PS]),
    "mpg_gen_fem3d": (_I, [_L, _U, _I, _PS]),
    "mpg_gen_zipf": (_I, [_L, _U, _L, _L, _D, _I, _PS]),
}
EXPORTED = tuple(_SIGS)
_lib_handle = None


def _glib():
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIBPATH):
            raise ImportError(f"{LIBPATH} is not built (make -C paper_2003_12759_b200/csrc)")
        h = C.CDLL(LIBPATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib_handle = h
    return _lib_handle


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int64)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


@dataclasses.dataclass
class HostCsr:
    nrows: int
    ncols: int
    rowptr: np.ndarray
    colind: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.val.size)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.colind, self.rowptr), shape=(self.nrows, self.ncols))

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            d[i, self.colind[self.rowptr[i]:self.rowptr[i + 1]]] = self.val[self.rowptr[i]:self.rowptr[i + 1]]
        return d


@dataclasses.dataclass
class System:
    """sigma E - A with inputs B (n x m) and outputs C (n x q), initial shifts."""
    n: int
    a: HostCsr
    e: Optional[HostCsr]  # None with e_diag None: identity
    e_diag: Optional[np.ndarray]
    b: np.ndarray
    c: np.ndarray
    shifts: np.ndarray
    r: int

    def e_csr(self) -> Optional[HostCsr]:
        if self.e is not None:
            return self.e
        if self.e_diag is not None:
            n = self.n
            return HostCsr(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), self.e_diag.copy())
        return None


def _take_csr(p) -> HostCsr:
    h = p.contents
    nr, nnz = h.nrows, h.nnz
    out = HostCsr(h.nrows, h.ncols, np.ctypeslib.as_array(h.rowptr, (nr + 1,)).copy(),
                  np.ctypeslib.as_array(h.colind, (max(nnz, 1),))[:nnz].copy(),
                  np.ctypeslib.as_array(h.val, (max(nnz, 1),))[:nnz].copy())
    _glib().mpg_gen_csr_free(p)
    return out


def _check(st):
    if st != 0:
        raise ValueError(_glib().mpg_gen_last_error().decode())


def random_dense(r: int, c: int, seed: int) -> np.ndarray:
    """support.hpp:18-25: U[-1,1], column-major fill (mt19937_64 + libstdc++ distribution)."""
    out = np.empty(r * c)
    _glib().mpg_gen_random_dense(r, c, seed, _ptr(out))
    return out.reshape((r, c), order="F")


def random_sparse(r: int, c: int, density: float, seed: int, diag_shift: float = 0.0) -> HostCsr:
    """support.hpp:37-49."""
    p = C.POINTER(HostCsrS)()
    _check(_glib().mpg_gen_random_sparse(r, c, density, seed, diag_shift, C.byref(p)))
    return _take_csr(p)


def from_triplets(nr: int, nc: int, rows, cols, vals) -> HostCsr:
    """Duplicates summed, exact-zero sums kept (sparse.cpp:80-115)."""
    ri, ci, v = _i64(rows), _i64(cols), _f64(vals)
    p = C.POINTER(HostCsrS)()
    _check(_glib().mpg_gen_from_triplets(nr, nc, ri.size, _ptr(ri), _ptr(ci), _ptr(v), C.byref(p)))
    return _take_csr(p)


def from_dense(d: np.ndarray, drop_tol: float = 0.0) -> HostCsr:
    """support.hpp:27-33 (sparse_from_dense)."""
    d = np.asarray(d, dtype=np.float64)
    rows, cols = np.nonzero(np.abs(d) > drop_tol)
    return from_triplets(d.shape[0], d.shape[1], rows, cols, d[rows, cols])


def bilinear_toy(n: int, m: int, seed: int):
    """generator.cpp:141-179 with N = 0: returns (K, F (n x m), C (n x 1))."""
    p = C.POINTER(HostCsrS)()
    f = np.empty(n * m)
    c = np.empty(n)
    _check(_glib().mpg_gen_bilinear_toy(n, m, seed, C.byref(p), _ptr(f), _ptr(c)))
    return _take_csr(p), f.reshape((n, m), order="F"), c.reshape((n, 1))


@dataclasses.dataclass
class QbSystem:
    """D x' = K x + H (x (x) x) + N x u + F u, y = C^T x (proj/include/morprec/qbihomm.hpp:15-33)."""
    d: HostCsr
    k: HostCsr
    n_op: HostCsr
    h: HostCsr  # n x n^2, column b n + c
    f: np.ndarray  # n
    c: np.ndarray  # n

    @property
    def n(self) -> int:
        return self.d.nrows


def qb_toy(n: int, seed: int) -> QbSystem:
    """generate_qb_toy (proj/src/generator.cpp:181-207): F = C = e_1."""
    ps = [C.POINTER(HostCsrS)() for _ in range(4)]
    _check(_glib().mpg_gen_qb_toy(n, seed, *[C.byref(p) for p in ps]))
    d, k, nop, h = (_take_csr(p) for p in ps)
    e1 = np.zeros(n)
    e1[0] = 1.0
    return QbSystem(d, k, nop, h, e1, e1.copy())


def disc_brake(n: int, omega: float, seed: int):
    """generate_disc_brake_like (proj/src/generator.cpp:37-139): returns (M, K) host CSR; the reference then
    forms D = alpha M + beta K and F = C = e_1."""
    pm, pk = C.POINTER(HostCsrS)(), C.POINTER(HostCsrS)()
    _check(_glib().mpg_gen_disc_brake(n, omega, seed, C.byref(pm), C.byref(pk)))
    return _take_csr(pm), _take_csr(pk)


def bilinear_toy_n(n: int, m: int, seed: int):
    """generate_bilinear_toy (proj/src/generator.cpp:141-179) with its couplings: (K, [N_1..N_m], F, C)."""
    pk = C.POINTER(HostCsrS)()
    pn = (C.POINTER(HostCsrS) * m)()
    f = np.empty(n * m)
    c = np.empty(n)
    _check(_glib().mpg_gen_bilinear_toy_n(n, m, seed, C.byref(pk), C.cast(pn, C.c_void_p), _ptr(f), _ptr(c)))
    return _take_csr(pk), [_take_csr(pn[j]) for j in range(m)], f.reshape((n, m), order="F"), c.reshape((n, 1))


def _take_system(p) -> System:
    s = p.contents
    n = s.n
    a = HostCsr(s.a.contents.nrows, s.a.contents.ncols,
                np.ctypeslib.as_array(s.a.contents.rowptr, (n + 1,)).copy(),
                np.ctypeslib.as_array(s.a.contents.colind, (s.a.contents.nnz,)).copy(),
                np.ctypeslib.as_array(s.a.contents.val, (s.a.contents.nnz,)).copy())
    e = None
    if s.e:
        ec = s.e.contents
        e = HostCsr(ec.nrows, ec.ncols, np.ctypeslib.as_array(ec.rowptr, (n + 1,)).copy(),
                    np.ctypeslib.as_array(ec.colind, (ec.nnz,)).copy(), np.ctypeslib.as_array(ec.val, (ec.nnz,)).copy())
    ed = np.ctypeslib.as_array(s.e_diag, (n,)).copy() if s.e_diag else None
    b = np.ctypeslib.as_array(s.b, (n * s.m,)).copy().reshape((n, s.m), order="F")
    c = np.ctypeslib.as_array(s.c, (n * s.q,)).copy().reshape((n, s.q), order="F")
    shifts = np.ctypeslib.as_array(s.shifts, (s.r,)).copy()
    out = System(n, a, e, ed, b, c, shifts, s.r)
    _glib().mpg_gen_system_free(p)
    return out


def config1(N: int = 100, seed: int = 0) -> System:
    """C1: 2D cell-centred diffusion, lognormal(0, 0.5) cells, E = diag U[1,2], r = 4."""
    p = C.POINTER(HostSystemS)()
    _check(_glib().mpg_gen_grid2d(N, seed, C.byref(p)))
    return _take_system(p)


def config2(M: int = 64, seed: int = 1) -> System:
    """C2: 3D 7-point convection-diffusion (upwind, v = (0.5, 0.3, 0.2)/h), E = diag U[0.5,1.5], r = 8."""
    p = C.POINTER(HostSystemS)()
    _check(_glib().mpg_gen_convdiff3d(M, seed, C.byref(p)))
    return _take_system(p)


def config3(N: int = 106, seed: int = 2, mimo: bool = False) -> System:
    """C3 / C4 (mimo, seed 3): Q1 hexahedral FEM on N^3 nodes, A = -(K + Robin), E = consistent mass."""
    p = C.POINTER(HostSystemS)()
    _check(_glib().mpg_gen_fem3d(N, seed, int(mimo), C.byref(p)))
    return _take_system(p)


def config4(N: int = 106, seed: int = 3) -> System:
    return config3(N, seed, True)


def config5(n: int = 2_000_000, seed: int = 4, nshifts: int = 64, max_len: int = 2000) -> System:
    """C5: Zipf(1.8) row lengths on [3, max_len], a_ii = -1.1 sum |a_ij|, E = diag U[1,2]."""
    p = C.POINTER(HostSystemS)()
    _check(_glib().mpg_gen_zipf(n, seed, 3, max_len, 1.8, nshifts, C.byref(p)))
    return _take_system(p)
