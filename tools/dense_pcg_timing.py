"""Persistent dense PCG: time per iteration and A-stream bandwidth for 1-4
right-hand sides (n = 50000: A is 20 GB), no preconditioner, fixed 40
iterations (diagnostic)."""
import ctypes as C, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
import bench
npcg.workloads = workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
ctx = npcg.Context(0)
w = workloads.make('cfg5', npcg.Rng, npcg.splitmix64, n=n, r=500, ell=100, nrhs=4, nmu=2)
path = bench.DevicePath(npcg, torch, w, ctx)
L = npcg.lib(); vp = C.c_void_p; i64 = C.c_int64
for s in ([int(v) for v in sys.argv[2].split(',')] if len(sys.argv) > 2 else (1, 2, 4)):
    reports = (npcg._SolveReport * s)()
    opts = npcg._SolveOpts(1e-300, 40, 0, 0)
    for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
        ctx.sync(); t0 = time.perf_counter()
        rc = L.npcg_pcg(vp(path.op.h), None, C.c_double(1e-3), i64(s), vp(path.b.data_ptr()), i64(n), None, i64(n),
                        C.byref(opts), vp(path.x.data_ptr()), i64(n), reports, None, None, npcg.DEVICE)
        ctx.sync(); dt = time.perf_counter() - t0
    it = reports[0].iterations
    print("S=%d: %d iterations, %.3f ms/iteration, A stream %.0f GB/s" % (s, it, dt / it * 1e3, 8.0 * n * n / (dt / it) / 1e9),
          flush=True)
