"""Config-5 PCG timing (first mu values of the path; 4 RHS) (diagnostic)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
import bench
npcg.workloads = workloads
ctx = npcg.Context(0)
w = workloads.make('cfg5', npcg.Rng, npcg.splitmix64, nmu=20)
w.mus = w.mus[:int(sys.argv[1]) if len(sys.argv) > 1 else 1]
if len(sys.argv) > 2:
    w.b = w.b[:, :int(sys.argv[2])].copy(order='F')
path = bench.DevicePath(npcg, torch, w, ctx)
ctx.prof_enable(True)
t = time.perf_counter(); info = path.step(); ctx.sync(); dt = time.perf_counter() - t
prof = ctx.prof_report()
print("mus", len(w.mus), "iters", info, "%.2f s" % dt)
for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:5]:
    print("%-40s %5d %10.1f ms  %.3e B  %.2f TB/s" % (k[:40], v[0], v[1], v[3], v[3] / (v[1] / 1e3) / 1e12 if v[1] else 0))
