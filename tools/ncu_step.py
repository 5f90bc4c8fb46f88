"""One config-2 solve step bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists (diagnostic). --cfg3 etc not supported."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
import bench
npcg.workloads = workloads
ctx = npcg.Context(0)
w = workloads.make('cfg2', npcg.Rng, npcg.splitmix64, gemm=lambda a, b, transa=False: npcg.gemm(a, b, transa=transa, ctx=ctx))
path = bench.DevicePath(npcg, torch, w, ctx)
for _ in range(2):
    path.step()
ctx.sync()
torch.cuda.cudart().cudaProfilerStart()
path.step()
ctx.sync()
torch.cuda.cudart().cudaProfilerStop()
print("iters", path.reports[0].iterations)
