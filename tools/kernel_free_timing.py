"""Matrix-free RBF operator: apply time for k = 1 (fused) and k = 400 (row blocks on DMMA) (diagnostic)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2110_02820_b200 as npcg
ctx = npcg.Context(0)
n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 50000, 32
pts = np.random.default_rng(0).random((n, d))
op = npcg.KernelOperator(pts, 0.5, dense_cap=1000, ctx=ctx)
for k in (1, 400):
    V = np.random.default_rng(1).standard_normal((n, k))
    op.apply_block(V)
    ctx.prof_enable(True)
    t = time.perf_counter(); op.apply_block(V); ctx.sync(); dt = time.perf_counter() - t
    prof = ctx.prof_report(); ctx.prof_enable(False)
    print("n=%d k=%d %.3f s" % (n, k, dt), {kk: (v[0], round(v[1], 2)) for kk, v in prof.items()})
