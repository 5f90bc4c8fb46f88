"""Pinned host->device copy bandwidth, one vs two streams (diagnostic)."""
import time, torch
n = 640 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device='cuda')
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = n // streams
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(streams, "streams: %.1f GB/s" % (n * 8 / dt / 1e9))
