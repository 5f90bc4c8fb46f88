"""Per-kernel times (library CUDA events) of one matrix-free K V at n, d, k (diagnostic).
usage: python tools/kf_prof.py n d k"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2110_02820_b200 as npcg
n, d, k = (int(a) for a in sys.argv[1:4])
ctx = npcg.Context(0)
op = npcg.KernelOperator(np.random.default_rng(0).random((n, d)), 0.5, dense_cap=1000, ctx=ctx)
V = np.random.default_rng(1).standard_normal((n, k))
op.apply_block(V)
ctx.sync()
ctx.prof_enable(True)
t = time.perf_counter()
op.apply_block(V)
ctx.sync()
dt = time.perf_counter() - t
rep = ctx.prof_report()
ctx.prof_enable(False)
print("n=%d d=%d k=%d wall %.4f s, kernels %.3f ms, %d launches" % (n, d, k, dt, sum(v[1] for v in rep.values()),
                                                                  sum(v[0] for v in rep.values())))
for name, v in sorted(rep.items(), key=lambda kv: -kv[1][1]):
    print("  %-50s %4d launches %9.3f ms" % (name, v[0], v[1]))
