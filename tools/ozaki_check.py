"""INT8 tcgen05 GEMM + Ozaki FP64 emulation: correctness on small shapes and
timing at the config-3 sketch shape against the FP64 DMMA GEMM (diagnostic)."""
import ctypes as C, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
rng = np.random.default_rng(5)
ctx = npcg.default_context()
for (m, n, kp) in [(128, 256, 128), (300, 520, 384), (1000, 77, 1024), (129, 257, 2048)]:
    a8 = rng.integers(-64, 65, size=(m, kp), dtype=np.int8)
    b8 = rng.integers(-64, 65, size=(n, kp), dtype=np.int8)
    ref = a8.astype(np.int64) @ b8.astype(np.int64).T
    got = npcg.gemm_i8(a8, b8)
    print("i8 %dx%dx%d exact=%s maxdiff=%d" % (m, n, kp, np.array_equal(ref, got), np.abs(ref - got).max()), flush=True)
for (m, n, k, spread) in [(200, 300, 500, 0), (513, 77, 1000, 6), (1000, 260, 3000, 30)]:
    a = rng.standard_normal((k, m)) * np.exp(rng.uniform(-spread, spread, (k, m)))
    b = rng.standard_normal((k, n))
    ref = a.T @ b
    got = npcg.gemm_ozaki(a, b)
    dm = npcg.gemm(a, b, transa=True)
    bound = np.abs(a.T) @ np.abs(b)
    print("ozaki %dx%dx%d spread %d: max |err|/(|A||B|) ozaki %.2e dmma %.2e" % (
        m, n, k, spread, np.max(np.abs(got - ref) / bound), np.max(np.abs(dm - ref) / bound)), flush=True)
# timing at the config-3 sketch shape (device buffers)
L = npcg.lib(); vp = C.c_void_p; i64 = C.c_int64
M = N = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
A = torch.randn(M, M, dtype=torch.float64, device='cuda')
A = (A + A.T) * 0.5
Om = torch.randn(ell, M, dtype=torch.float64, device='cuda')  # Omega^T rows = K-major Omega
Y1 = torch.empty(ell, M, dtype=torch.float64, device='cuda')
Y2 = torch.empty(ell, M, dtype=torch.float64, device='cuda')
def run(f):
    torch.cuda.synchronize(); t = time.perf_counter(); f(); ctx.sync(); torch.cuda.synchronize(); return time.perf_counter() - t
dmma = lambda: L.npcg_gemm(vp(ctx.h), i64(M), i64(ell), i64(M), C.c_double(1.0), vp(A.data_ptr()), i64(M), C.c_int(1),
                           vp(Om.data_ptr()), i64(M), C.c_int(1), C.c_double(0.0), vp(Y1.data_ptr()), i64(M), npcg.DEVICE)
oz = lambda: L.npcg_gemm_ozaki(vp(ctx.h), i64(M), i64(ell), i64(M), vp(A.data_ptr()), i64(M), C.c_int(1), vp(Om.data_ptr()), i64(M), C.c_int(1),
                               vp(Y2.data_ptr()), i64(M), npcg.DEVICE)
for f, name in ((dmma, "dmma"), (oz, "ozaki")):
    run(f)
    ts = [run(f) for _ in range(3)]
    print("%s %dx%dx%d: %.2f ms (%.1f TF/s fp64-equivalent)" % (name, M, ell, M, min(ts) * 1e3, 2.0 * M * M * ell / min(ts) / 1e12), flush=True)
d = (Y1 - Y2).abs().max().item() / Y1.abs().max().item()
print("ozaki vs dmma max rel diff %.2e" % d)
