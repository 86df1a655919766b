"""ctypes binding of libmpg.so (include/mpg.h).

The product path is the CUDA library; there is no CPU fallback. Importing
this module fails loudly when libmpg.so has not been built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_2003_12759_b200/csrc)")

lib = C.CDLL(LIB_PATH)

MPG_OK, MPG_ERR_INVALID, MPG_ERR_CONFIG, MPG_ERR_SOLVER, MPG_ERR_LOGIC, MPG_ERR_CUDA, MPG_ERR_NOMEM, MPG_ERR_IO = range(8)
PRECOND_NONE, PRECOND_FRESH, PRECOND_REUSE_CHAIN, PRECOND_REUSE_FROZEN = range(4)
KIND_NONE, KIND_FRESH, KIND_HORIZONTAL, KIND_VERTICAL, KIND_REUSED_SAME_MATRIX = range(5)
KIND_NAMES = {0: "none", 1: "fresh", 2: "horizontal", 3: "vertical", 4: "reused_same_matrix"}


class ConfigError(RuntimeError):
    """morprec::ConfigError (proj/include/morprec/errors.hpp:12-16)."""


class SolverError(RuntimeError):
    """morprec::SolverError (proj/include/morprec/errors.hpp:18-22)."""


class IoError(RuntimeError):
    """morprec::IoError (proj/include/morprec/errors.hpp:24-28)."""


class CudaError(RuntimeError):
    pass


def check(status: int) -> None:
    if status == MPG_OK:
        return
    msg = lib.mpg_last_error().decode()
    if status == MPG_ERR_INVALID:
        raise ValueError(msg)
    if status == MPG_ERR_CONFIG:
        raise ConfigError(msg)
    if status == MPG_ERR_SOLVER:
        raise SolverError(msg)
    if status == MPG_ERR_NOMEM:
        raise MemoryError(msg)
    if status == MPG_ERR_CUDA:
        raise CudaError(msg)
    if status == MPG_ERR_IO:
        raise IoError(msg)
    raise RuntimeError(msg)


class SpaiCfg(C.Structure):
    _fields_ = [("pattern_kind", C.c_int), ("power", C.c_int), ("fill_tol", C.c_double),
                ("max_fill_per_col", C.c_int), ("max_pattern_sweeps", C.c_int), ("threads", C.c_int)]


class GmresCfg(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iter", C.c_int), ("record_history", C.c_int)]


class GmresRep(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int), ("history_len", C.c_int),
                ("rhs_norm", C.c_double), ("final_residual", C.c_double), ("solve_seconds", C.c_double),
                ("reorth_passes", C.c_int)]


class IrkaCfg(C.Structure):
    _fields_ = [("r", C.c_int), ("tol", C.c_double), ("max_sweeps", C.c_int), ("decoupled", C.c_int),
                ("seed", C.c_ulonglong), ("gmres", GmresCfg), ("spai", SpaiCfg), ("max_chain_len", C.c_int),
                ("explicit_nnz_cap", C.c_longlong), ("standard_residual_max_dim", C.c_longlong),
                ("mirror_unstable", C.c_int)]


class QbCfg(C.Structure):
    _fields_ = [("p_moments", C.c_int), ("q_moments", C.c_int), ("gmres", GmresCfg), ("spai", SpaiCfg),
                ("max_chain_len", C.c_int), ("standard_residual_max_dim", C.c_longlong)]


class AirgaCfg(C.Structure):
    _fields_ = [("r_max", C.c_int), ("outer_tol", C.c_double), ("inner_tol", C.c_double), ("max_outer", C.c_int),
                ("gmres", GmresCfg), ("spai", SpaiCfg), ("max_chain_len", C.c_int),
                ("standard_residual_max_dim", C.c_longlong)]


class ReportRow(C.Structure):
    _fields_ = [("sweep", C.c_int), ("point", C.c_int), ("kind", C.c_int), ("solves", C.c_int),
                ("iterations", C.c_longlong), ("build_seconds", C.c_double), ("gmres_seconds", C.c_double),
                ("min_residual", C.c_double), ("matrix_change", C.c_double), ("standard_residual", C.c_double)]


class HostCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64), ("rowptr", C.POINTER(C.c_int64)),
                ("colind", C.POINTER(C.c_int64)), ("val", C.POINTER(C.c_double))]


class HostSystem(C.Structure):
    _fields_ = [("n", C.c_int64), ("a", C.POINTER(HostCsr)), ("e", C.POINTER(HostCsr)),
                ("e_diag", C.POINTER(C.c_double)), ("m", C.c_int), ("q", C.c_int), ("r", C.c_int),
                ("b", C.POINTER(C.c_double)), ("c", C.POINTER(C.c_double)), ("shifts", C.POINTER(C.c_double))]


vp, dp, ip, i64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int64)
_I = C.c_int
_D = C.c_double
_L = C.c_int64

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)

_SIGS = {
    "mpg_last_error": (C.c_char_p, []),
    "mpg_device_count": (_I, [ip]),
    "mpg_stream": (_I, [_I, C.POINTER(vp)]),
    "mpg_synchronize": (_I, [_I]),
    "mpg_launch_count": (C.c_longlong, []),
    "mpg_copy": (_I, [vp, vp, _L]),
    "mpg_profile_enable": (None, [_I]),
    "mpg_profile_count": (_I, []),
    "mpg_profile_read": (_I, [_I, C.POINTER(C.c_char_p), C.POINTER(C.c_longlong), dp, dp]),
    "mpg_csr_create": (_I, [_I, _L, _L, vp, vp, vp, C.POINTER(vp)]),
    "mpg_csr_destroy": (None, [vp]),
    "mpg_csr_info": (_I, [vp, i64p, i64p, i64p]),
    "mpg_csr_download": (_I, [vp, vp, vp, vp]),
    "mpg_csr_multiply": (_I, [vp, vp, vp]),
    "mpg_csr_multiply_transpose": (_I, [vp, vp, vp]),
    "mpg_csr_transpose": (_I, [vp, C.POINTER(vp)]),
    "mpg_csr_frobenius_norm": (_D, [vp]),
    "mpg_op_create": (_I, [vp, vp, C.POINTER(vp)]),
    "mpg_op_destroy": (None, [vp]),
    "mpg_op_dim": (_L, [vp]),
    "mpg_op_apply": (_I, [vp, _D, _D, _I, vp, vp]),
    "mpg_op_explicit": (_I, [vp, _D, _D, _I, C.POINTER(vp)]),
    "mpg_spai_build": (_I, [vp, C.POINTER(SpaiCfg), C.POINTER(vp), vp, i64p, dp]),
    "mpg_spai_column_solve": (_I, [vp, _L, _L, vp, vp, dp, ip]),
    "mpg_update_build": (_I, [vp, vp, C.POINTER(SpaiCfg), C.POINTER(vp), dp, dp, i64p, dp]),
    "mpg_chain_create": (_I, [vp, C.POINTER(vp)]),
    "mpg_chain_extend": (_I, [vp, vp, C.POINTER(vp)]),
    "mpg_chain_destroy": (None, [vp]),
    "mpg_chain_length": (_I, [vp]),
    "mpg_chain_factor_id": (vp, [vp, _I]),
    "mpg_chain_apply": (_I, [vp, vp, vp]),
    "mpg_standard_residual": (_I, [vp, vp, dp]),
    "mpg_gmres_csr": (_I, [vp, vp, vp, vp, C.POINTER(GmresCfg), C.POINTER(GmresRep), vp]),
    "mpg_gmres_shifted": (_I, [vp, _D, _D, _I, vp, vp, vp, C.POINTER(GmresCfg), C.POINTER(GmresRep), vp]),
    "mpg_gmres_batch": (_I, [vp, _I, vp, vp, vp, vp, vp, vp, C.POINTER(GmresCfg), vp]),
    "mpg_irka_reduce": (_I, [vp, vp, _I, vp, _I, C.POINTER(IrkaCfg), _I, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                             ip, ip, vp, _I, ip]),
    "mpg_irka_reduce_from": (_I, [vp, vp, _I, vp, _I, C.POINTER(IrkaCfg), _I, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                  ip, ip, vp, _I, ip]),
    "mpg_birka_reduce": (_I, [vp, vp, vp, _I, vp, _I, C.POINTER(IrkaCfg), _I] + [vp] * 8
                          + [ip, ip, vp, _I, ip, C.POINTER(C.c_void_p)]),
    "mpg_irka_reduce_sharded": (_I, [vp, vp, _I, vp, _I, C.POINTER(IrkaCfg), _I, vp, _I, _I, ALLGATHER_FN, vp, vp,
                                     vp, vp, vp, vp, ip, ip, vp, _I, ip]),
    "mpg_qbihomm_reduce": (_I, [vp, vp, _L, vp, vp, vp, vp, vp, _I, vp, C.POINTER(QbCfg), _I, _I, ip] + [vp] * 8
                           + [_I, ip]),
    "mpg_project": (_I, [vp, vp, vp, _I, vp, vp]),
    "mpg_spai_bench": (_I, [vp, vp, _I, vp, C.POINTER(SpaiCfg), C.POINTER(GmresCfg), _I, _I, vp, vp, _I, ip, ip]),
    "mpg_airga_reduce": (_I, [vp, vp, vp, vp, _I, vp, _I, _D, _D, vp, _I, C.POINTER(AirgaCfg), _I, ip] + [vp] * 7
                         + [ip, ip, vp, _I, ip, C.POINTER(C.c_void_p)]),
    "mpg_update_expansion_points": (_I, [vp, vp, vp, _I, vp, _I, vp]),
    "mpg_h2_norm": (_I, [vp, vp, vp, _I, _I, _I, C.POINTER(C.c_double)]),
    "mpg_transfer_function_error": (_I, [vp, vp, vp, vp, _I, vp, _I, vp, vp, vp, vp, vp, _I, vp, _I,
                                         C.POINTER(GmresCfg), C.POINTER(SpaiCfg), _I, _I, vp, C.POINTER(C.c_longlong)]),
    "mpg_mm_read_file": (_I, [C.c_char_p, _I, C.POINTER(C.POINTER(HostCsr))]),
    "mpg_mm_read_buffer": (_I, [C.c_char_p, _L, C.c_char_p, _I, C.POINTER(C.POINTER(HostCsr))]),
    "mpg_mm_write_file": (_I, [C.c_char_p, C.POINTER(HostCsr), _I]),
    "mpg_mm_write_buffer": (_I, [C.POINTER(HostCsr), _I, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "mpg_mm_write_dense_buffer": (_I, [_L, _L, vp, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "mpg_report_csv": (_I, [vp, _I, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "mpg_buffer_free": (None, [vp]),
    "mpg_shard_cost": (_D, [_I, _I]),
    "mpg_shard_plan": (_I, [_I, vp, vp, _I, vp]),
    "mpg_comm_unique_id": (_I, [vp, _I]),
    "mpg_comm_create": (_I, [_I, _I, _I, vp, C.POINTER(C.c_void_p)]),
    "mpg_comm_destroy": (_I, [vp]),
    "mpg_comm_allgather": (_I, [vp, vp, vp, _L]),
    "mpg_comm_stats": (_I, [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_double)]),
    "mpg_nccl_version": (_I, [C.POINTER(C.c_int)]),
    "mpg_host_csr_free": (None, [C.POINTER(HostCsr)]),
    "mpg_host_csr_from_triplets": (_I, [_L, _L, _L, vp, vp, vp, C.POINTER(C.POINTER(HostCsr))]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def i64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int64)
