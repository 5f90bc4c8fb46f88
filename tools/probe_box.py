"""Probe the GPU box: host cores/RAM, GPU props, cuBLAS DGEMM and copy bandwidth."""
import json, os, subprocess, time
import torch

out = {}
out["nproc"] = os.cpu_count()
try:
    out["meminfo_gb"] = int(open("/proc/meminfo").readline().split()[1]) / 1e6
except Exception as e:
    out["meminfo_gb"] = str(e)
out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].strip()
p = torch.cuda.get_device_properties(0)
out["gpu"] = dict(name=p.name, sms=p.multi_processor_count, mem_gb=p.total_memory / 1e9,
                  l2=getattr(p, "L2_cache_size", None))
dev = torch.device("cuda:0")
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        s.record(); c = a @ b; e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    out[f"cublas_dgemm_{n}_tflops"] = 2 * n ** 3 / best / 1e12
x = torch.empty(1 << 30, dtype=torch.float64, device=dev)
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s.record(); y.copy_(x); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
out["copy_gbs"] = 2 * x.numel() * 8 / best / 1e9
print(json.dumps(out, indent=1))
