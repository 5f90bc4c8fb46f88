"""Per-call wall time of bench.py's e2e step (public API from host arrays) (diagnostic):
  python tools/e2e_breakdown.py [cfg3]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
npcg.workloads = workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else 'cfg3'
ctx = npcg.Context(0)
w = workloads.make(cfg, npcg.Rng, npcg.splitmix64)
for rep in range(3):
    T = {}
    t0 = t = time.perf_counter()
    def lap(k):
        global t
        ctx.sync(); n = time.perf_counter(); T[k] = (n - t) * 1e3; t = n
    op = workloads.build_operator(npcg, w, ctx=ctx, streamed=True); lap("operator")
    pair = npcg.make_empty_sketch(op); lap("empty")
    pair = npcg.extend_sketch_with(pair, op, w.omega); lap("sketch (Omega H2D + Y = A Omega)")
    ap = npcg.nystrom_from_sketch(pair); lap("factor")
    pre = npcg.build_preconditioner(ap, w.mu); lap("preconditioner")
    rep_ = npcg.nystrom_pcg(op, w.b, w.mu, pre, eta=w.eta, max_iter=w.max_iter, relative=w.relative); lap("pcg (b H2D, x D2H)")
    print("rep %d total %.1f ms: " % (rep, (time.perf_counter() - t0) * 1e3) + ", ".join("%s %.1f" % kv for kv in T.items()), flush=True)
    del op, pair, ap, pre, rep_
