"""Matrix-free RBF kernel, one sketch-block product K V (n x k) with device
buffers: FP64 DMMA vs INT8 digit planes, per-kernel breakdown (diagnostic).
  python tools/kfree_sketch_timing.py n k [kblock_bytes]"""
import ctypes as C, os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
n, k = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    os.environ['NPCG_KBLOCK_BYTES'] = sys.argv[3]
ctx = npcg.Context(0)
pts = np.random.default_rng(0).random((n, 32))
op = npcg.KernelOperator(pts, 0.5, dense_cap=1, ctx=ctx)
V = torch.randn(n, k, dtype=torch.float64, device='cuda').T.contiguous().T  # col-major n x k
Y = torch.empty(k, n, dtype=torch.float64, device='cuda').T
L = npcg.lib(); vp = C.c_void_p; i64 = C.c_int64
def run():
    ctx.sync(); t = time.perf_counter()
    npcg._check(L.npcg_op_apply(vp(op.h), i64(n), i64(k), vp(V.data_ptr()), i64(n), vp(Y.data_ptr()), i64(n), npcg.DEVICE))
    ctx.sync(); return time.perf_counter() - t
run()
ctx.prof_enable(True)
dt = run()
rep = ctx.prof_report()
ctx.prof_enable(False)
print("OZAKI=%s n=%d k=%d: %.3f s" % (os.environ.get('NPCG_OZAKI', '1'), n, k, dt))
for name, v in sorted(rep.items(), key=lambda kv: -kv[1][1])[:8]:
    print("   %-40s %6d %9.1f ms" % (name[:40], v[0], v[1]))
