"""Time one SPAI build on C3 (tuning aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
N = int(sys.argv[1]) if len(sys.argv) > 1 else 106
s = gen.config3(N)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
m = op.explicit(float(s.shifts[0]), False)
mpg.spai_build(m)
for rep in range(2):
    mpg.lib.mpg_synchronize(0)
    t = time.perf_counter()
    r = mpg.spai_build(m)
    mpg.lib.mpg_synchronize(0)
    print(f"N={N} n={s.n} spai_build {time.perf_counter() - t:.3f} s  fallbacks={r.fallback_count} wps={os.environ.get('MPG_SPAI_WPS', '16')}")
