"""Seeded synthetic inputs for the CPU side (test infrastructure, like the rest of oracle/).

Executes the generator wrapper paper_2003_12759_b200/gen.py (pure Python; it
imports nothing from its package) bound to oracle/liboracle.so, which compiles
the same generator source (oracle/Makefile). The inputs are therefore
identical to the GPU arm's, and the CPU reference arm of bench.py maps no
library outside oracle/.
"""
import importlib.util as _ilu
import os as _os
import sys as _sys

_here = _os.path.dirname(_os.path.abspath(__file__))
_spec = _ilu.spec_from_file_location("oracle._gen_impl",
                                     _os.path.join(_os.path.dirname(_here), "paper_2003_12759_b200", "gen.py"))
_impl = _ilu.module_from_spec(_spec)
_sys.modules["oracle._gen_impl"] = _impl
_spec.loader.exec_module(_impl)
_impl.LIBPATH = _os.path.join(_here, "liboracle.so")

for _k in dir(_impl):
    if not _k.startswith("__"):
        globals()[_k] = getattr(_impl, _k)
