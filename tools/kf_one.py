"""One fused matrix-free RBF matvec (n = 50000, d = 32) for ncu (diagnostic)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2110_02820_b200 as npcg
ctx = npcg.Context(0)
n, d = 50000, 32
op = npcg.KernelOperator(np.random.default_rng(0).random((n, d)), 0.5, dense_cap=1000, ctx=ctx)
v = np.random.default_rng(1).standard_normal(n)
op.matvec(v)
ctx.sync()
print("ok")
