"""Host-buffer Gram operator construction: synchronous vs streamed (+ first
sketch product), cfg2 sizes, pinned host memory (diagnostic)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
ctx = npcg.Context(0)
m, n, l = 20000, 4000, 400
t = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
x = t.numpy().T
x[:] = np.random.default_rng(0).standard_normal((m, n))
om = np.asfortranarray(np.random.default_rng(1).standard_normal((n, l)))
dom = torch.from_numpy(om.T.copy()).cuda().T  # device Omega (n x l col-major)
for rep in range(3):
    t0 = time.perf_counter(); op = npcg.GramRidgeOperator(x, ctx=ctx); ctx.sync(); t1 = time.perf_counter()
    y = op.apply_block(om); t2 = time.perf_counter()
    del op
    t3 = time.perf_counter(); op = npcg.GramRidgeOperator(x, ctx=ctx, streamed=True); t4 = time.perf_counter()
    y2 = op.apply_block(om); t5 = time.perf_counter()
    del op
    print("sync create %.2f ms, sketch %.2f ms | streamed create %.2f ms, create+sketch %.2f ms  (rel diff %.1e)"
          % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t4 - t3) * 1e3, (t5 - t3) * 1e3,
             np.abs(y - y2).max() / np.abs(y).max()), flush=True)
