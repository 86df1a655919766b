"""B200-native preconditioned shifted-solve engine for IRKA / moment matching
(the hot path of arXiv 2003.12759, reference `morprec`, /root/reference/proj).

The compute path is libmpg.so (hand-written sm_100a CUDA + C++ drivers behind
the C ABI in include/mpg.h); this package is the Python mirror of the
reference's API (morprec.py) and the synthetic-input generators (gen.py).
"""
from ._lib import ConfigError, CudaError, IoError, SolverError, lib  # noqa: F401  (fails loudly if libmpg.so is missing)
from . import gen  # noqa: F401
from .morprec import *  # noqa: F401,F403


def device_count() -> int:
    import ctypes
    n = ctypes.c_int()
    lib.mpg_device_count(ctypes.byref(n))
    return n.value


def profile_enable(on: bool = True) -> None:
    """Per-kernel-class event timing + algorithmic bytes inside the GMRES engine."""
    lib.mpg_profile_enable(int(on))


def profile_read() -> dict:
    import ctypes
    out = {}
    for k in range(lib.mpg_profile_count()):
        name = ctypes.c_char_p()
        n, ms, by = ctypes.c_longlong(), ctypes.c_double(), ctypes.c_double()
        lib.mpg_profile_read(k, ctypes.byref(name), ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by))
        out[name.value.decode()] = {"launches": n.value, "ms": ms.value, "bytes": by.value}
    return out


def launch_count() -> int:
    """Kernels launched by libmpg.so in this process."""
    return int(lib.mpg_launch_count())
