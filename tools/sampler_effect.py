import sys, time; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
import bench
npcg.workloads = workloads
ctx = npcg.Context(0)
w = workloads.make('cfg2', npcg.Rng, npcg.splitmix64, gemm=lambda a, b, transa=False: npcg.gemm(a, b, transa=transa, ctx=ctx))
path = bench.DevicePath(npcg, torch, w, ctx)
for _ in range(2): path.step()
def timed(k, sampler=None, interval=None):
    t0 = time.perf_counter()
    if sampler:
        with bench.ClockSampler(0) as c:
            for _ in range(k): path.step()
    else:
        for _ in range(k): path.step()
    return (time.perf_counter() - t0) / k * 1e3
print("no sampler   %.1f ms" % timed(4))
print("nvidia-smi   %.1f ms" % timed(4, True))
import pynvml, threading
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False; samples = []
def loop():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.1)
th = threading.Thread(target=loop); th.start()
print("pynvml 100ms %.1f ms (%d samples)" % (timed(4), len(samples)))
stop = True; th.join()
print("no sampler   %.1f ms" % timed(4))
