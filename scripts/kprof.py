"""Per-kernel-class profile of one batched solve (tuning aid, not the bench)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12759_b200 as mpg
from paper_2003_12759_b200 import gen
N = int(sys.argv[1]) if len(sys.argv) > 1 else 80
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = gen.config3(N)
dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
op = mpg.ShiftedOperator(dev(s.a), dev(s.e))
sig = [float(x) for x in s.shifts[:S]]
P = mpg.PrecondChain(mpg.spai_build(op.explicit(sig[0])).p)
cfg = mpg.GmresConfig(1e-8, 1000)
mpg.gmres_batch(op, sig, [s.b[:, 0]] * S, chains=[P] * S, cfg=cfg)
t = time.time()
res = mpg.gmres_batch(op, sig, [s.b[:, 0]] * S, chains=[P] * S, cfg=cfg)
el = time.time() - t
mpg.profile_enable(True)
mpg.gmres_batch(op, sig, [s.b[:, 0]] * S, chains=[P] * S, cfg=cfg)
prof = mpg.profile_read()
mpg.profile_enable(False)
tot = sum(v["ms"] for v in prof.values())
print(f"N={N} n={s.n} S={S} its={[r.report.iterations for r in res]} reorth={[r.report.reorth_passes for r in res]} graph_time={el:.3f}s prof_total={tot/1e3:.3f}s vec={os.environ.get('MPG_VEC_WIDTH','auto')}")
for k, v in prof.items():
    if v["launches"]:
        gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 and v["bytes"] > 0 else 0
        print(f"  {k:16s} launches={v['launches']:6d} ms={v['ms']:9.2f} share={v['ms']/tot*100:5.1f}% GB/s={gbs:8.1f}")
