"""Persistent dense PCG with the Nystrom preconditioner at n = 1e5, ell = 2000:
time per iteration for 4 and 8 columns (fixed 30 iterations; diagnostic).
NPCG_PCG_TRACE=1 prints CTA 0's phase times."""
import ctypes as C, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
import bench
npcg.workloads = workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
ctx = npcg.Context(0)
w = workloads.make('cfg5', npcg.Rng, npcg.splitmix64, n=n, r=500, ell=ell, nrhs=8, nmu=2)
path = bench.DevicePath(npcg, torch, w, ctx)
L = npcg.lib(); vp = C.c_void_p; i64 = C.c_int64
nys, pre = vp(), vp()
npcg._check(L.npcg_nys_create(vp(path.op.h), C.byref(nys)))
npcg._check(L.npcg_nys_extend(nys, i64(ell), vp(path.omega.data_ptr()), i64(n), npcg.DEVICE))
npcg._check(L.npcg_nys_factor(nys))
mu = 1e-3
npcg._check(L.npcg_pre_create(nys, C.c_double(mu), C.byref(pre)))
for s in ([int(v) for v in sys.argv[3].split(',')] if len(sys.argv) > 3 else (4, 8)):
    reports = (npcg._SolveReport * s)()
    opts = npcg._SolveOpts(1e-300, 30, 0, 0)
    for rep in range(2):
        ctx.sync(); t0 = time.perf_counter()
        rc = L.npcg_pcg(vp(path.op.h), pre, C.c_double(mu), i64(s), vp(path.b.data_ptr()), i64(n), None, i64(n),
                        C.byref(opts), vp(path.x.data_ptr()), i64(n), reports, None, None, npcg.DEVICE)
        ctx.sync(); dt = time.perf_counter() - t0
    it = reports[0].iterations
    print("S=%d: %d iterations, %.3f ms/iteration; rc %d; per column (iterations, status, history_len): %s" % (
        s, it, dt / it * 1e3, rc, [(r.iterations, r.status, r.history_len) for r in reports]), flush=True)
