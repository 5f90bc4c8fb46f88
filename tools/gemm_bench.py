"""DMMA GEMM throughput (device-resident) vs cuBLAS DGEMM, several shapes/layouts."""
import ctypes as C, sys, json
sys.path.insert(0, '.')
import torch
import paper_2110_02820_b200 as npcg
ctx = npcg.Context(0)
L = npcg.lib()
stream = torch.cuda.ExternalStream(ctx.stream)
def run(m, n, k, ak, bk, reps=5):
    a = torch.randn((m, k) if ak else (k, m), dtype=torch.float64, device='cuda')  # row-major torch (r,c) == col-major (c,r)
    b = torch.randn((n, k) if bk else (k, n), dtype=torch.float64, device='cuda')
    c = torch.zeros((n, m), dtype=torch.float64, device='cuda')
    torch.cuda.synchronize()
    lda = k if ak else m
    ldb = k if bk else n
    def call():
        npcg._check(L.npcg_gemm(C.c_void_p(ctx.h), C.c_int64(m), C.c_int64(n), C.c_int64(k), C.c_double(1.0),
                                C.c_void_p(a.data_ptr()), C.c_int64(lda), C.c_int(ak), C.c_void_p(b.data_ptr()),
                                C.c_int64(ldb), C.c_int(bk), C.c_double(0.0), C.c_void_p(c.data_ptr()), C.c_int64(m), 1))
    call()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        s.record(stream); call(); e.record(stream); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return 2 * m * n * k / best / 1e12
out = {}
for (m, n, k) in [(8192, 8192, 8192), (20000, 400, 4000), (4000, 400, 20000), (50000, 1000, 50000), (4000, 400, 400), (400, 400, 4000), (20000, 400, 400), (400, 400, 20000), (20000, 64, 64), (336, 336, 64)]:
    for ak, bk in [(1, 1), (0, 1), (1, 0), (0, 0)]:
        if m * k > 3e9: 
            if (ak, bk) != (1, 1): continue
        out[f"{m}x{n}x{k} ak{ak} bk{bk}"] = round(run(m, n, k, ak, bk), 2)
        print(list(out.items())[-1], flush=True)
a = torch.randn(8192, 8192, dtype=torch.float64, device='cuda'); b = torch.randn_like(a)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
a @ b; torch.cuda.synchronize(); best = 1e9
for _ in range(5):
    s.record(); a @ b; e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
print("cublas 8192^3", 2 * 8192 ** 3 / best / 1e12)
