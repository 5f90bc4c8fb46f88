"""Host wall-clock per phase of one config-2 (default) or config-3 (--cfg3) solve (diagnostic)."""
import ctypes as C, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
import bench
npcg.workloads = workloads
ctx = npcg.Context(0)
small = '--small' in sys.argv
if '--cfg3' in sys.argv:
    w = workloads.make('cfg3', npcg.Rng, npcg.splitmix64)
else:
    w = workloads.make('cfg2', npcg.Rng, npcg.splitmix64, gemm=lambda a, b, transa=False: npcg.gemm(a, b, transa=transa, ctx=ctx), **(dict(m=4000, n=800, ell=100) if small else {}))
path = bench.DevicePath(npcg, torch, w, ctx)
L = npcg.lib(); vp = C.c_void_p; i64 = C.c_int64
for rep in range(4):
    t = [time.perf_counter()]
    nys, pre = vp(), vp()
    npcg._check(L.npcg_nys_create(vp(path.op.h), C.byref(nys))); t.append(time.perf_counter())
    npcg._check(L.npcg_nys_extend(nys, i64(w.ell), vp(path.omega.data_ptr()), i64(w.n), npcg.DEVICE)); ctx.sync(); t.append(time.perf_counter())
    npcg._check(L.npcg_nys_factor(nys)); ctx.sync(); t.append(time.perf_counter())
    npcg._check(L.npcg_pre_create(nys, C.c_double(w.mu), C.byref(pre))); ctx.sync(); t.append(time.perf_counter())
    npcg._check(L.npcg_pcg(vp(path.op.h), pre, C.c_double(w.mu), i64(1), vp(path.b.data_ptr()), i64(w.n), None, i64(w.n), C.byref(path.opts), vp(path.x.data_ptr()), i64(w.n), path.reports, None, None, npcg.DEVICE)); t.append(time.perf_counter())
    L.npcg_pre_destroy(pre); L.npcg_nys_destroy(nys); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("create %.2f extend %.2f factor %.2f pre %.2f pcg %.2f destroy %.2f total %.2f ms  iters %d" % (*d, sum(d), path.reports[0].iterations))
ctx.prof_enable(True); path.step(); prof = ctx.prof_report(); ctx.prof_enable(False)
tot = 0
for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    tot += v[1]
    print("%-40s %5d %9.3f ms  %.3e flop %.3e B" % (k[:40], *v))
print("kernel total %.2f ms" % tot)
