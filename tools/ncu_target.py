"""Small, deterministic launch sequence for ncu captures of the config-2 hot
kernels: the sketch DMMA GEMM (X Omega: 20000x400x4000), the single-pass Gram
matvec (X^T X v / m over X 20000x4000) and a preconditioner apply (U 4000x400)."""
import ctypes as C, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
ctx = npcg.Context(0)
L = npcg.lib()
m, n, ell = 20000, 4000, 400
g = torch.Generator(device='cuda').manual_seed(0)
X = torch.randn((m, n), dtype=torch.float64, device='cuda', generator=g)          # row-major == X^T col-major
Om = torch.randn((ell, n), dtype=torch.float64, device='cuda', generator=g)       # Omega col-major n x ell
Z = torch.zeros((ell, m), dtype=torch.float64, device='cuda')
torch.cuda.synchronize()
# 1) sketch GEMM: Z (m x ell) = X (m x n) Omega  -- A K-major (row-major X), B K-major
npcg._check(L.npcg_gemm(C.c_void_p(ctx.h), C.c_int64(m), C.c_int64(ell), C.c_int64(n), C.c_double(1.0),
                        C.c_void_p(X.data_ptr()), C.c_int64(n), C.c_int(1), C.c_void_p(Om.data_ptr()), C.c_int64(n),
                        C.c_int(1), C.c_double(0.0), C.c_void_p(Z.data_ptr()), C.c_int64(m), 1))
# 2) Gram operator matvec with device pointers (X col-major m x n from the row-major tensor's transpose)
Xc = X.t().contiguous().t()  # same values, column-major storage
Xcm = torch.empty((n, m), dtype=torch.float64, device='cuda'); Xcm.copy_(X.t())  # (n, m) row-major == X col-major
torch.cuda.synchronize()
op = C.c_void_p()
npcg._check(L.npcg_op_gram_create(C.c_void_p(ctx.h), C.c_int64(m), C.c_int64(n), C.c_void_p(Xcm.data_ptr()),
                                  C.c_int64(m), 1, C.byref(op)))
v = torch.randn(n, dtype=torch.float64, device='cuda', generator=g)
out = torch.empty(n, dtype=torch.float64, device='cuda')
torch.cuda.synchronize()
for _ in range(2):
    npcg._check(L.npcg_op_apply(op, C.c_int64(n), C.c_int64(1), C.c_void_p(v.data_ptr()), C.c_int64(n),
                                C.c_void_p(out.data_ptr()), C.c_int64(n), 1))
# 3) preconditioner apply with U 4000 x 400
U = np.linalg.qr(np.random.default_rng(0).standard_normal((n, ell)))[0]
approx = npcg.make_approximation(U, np.linspace(1, 1e-3, ell), 1e-16, ctx=ctx)
pre = npcg.build_preconditioner(approx, 1e-3)
r = np.random.default_rng(1).standard_normal(n)
for _ in range(2):
    pre.apply_inverse(r)
ctx.sync()
L.npcg_op_destroy(op)
print("ok")
