"""One emulated GEMM at a given shape with device buffers (diagnostic / ncu target):
  python tools/ozaki_shape.py M N K a_kmajor(0/1) [reps]"""
import ctypes as C, sys, time
sys.path.insert(0, '.')
import torch
import paper_2110_02820_b200 as npcg
M, N, K, ak = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
ctx = npcg.default_context()
A = torch.rand((M, K) if ak else (K, M), dtype=torch.float64, device='cuda')  # row-major torch = col-major (K x M) / (M x K)
B = torch.randn(N, K, dtype=torch.float64, device='cuda')
Cm = torch.zeros(N, M, dtype=torch.float64, device='cuda')
L = npcg.lib(); vp = C.c_void_p; i64 = C.c_int64
for r in range(reps):
    ctx.sync(); t = time.perf_counter()
    npcg._check(L.npcg_gemm_ozaki(vp(ctx.h), i64(M), i64(N), i64(K), vp(A.data_ptr()), i64(K if ak else M), C.c_int(ak),
                                  vp(B.data_ptr()), i64(K), C.c_int(1), vp(Cm.data_ptr()), i64(M), npcg.DEVICE))
    ctx.sync(); dt = time.perf_counter() - t
    print("M=%d N=%d K=%d kmajor=%d: %.2f ms, %.1f TF/s fp64-eq" % (M, N, K, ak, dt * 1e3, 2.0 * M * N * K / dt / 1e12), flush=True)
