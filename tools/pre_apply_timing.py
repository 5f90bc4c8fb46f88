"""Standalone Nystrom preconditioner apply P^{-1} R (npcg_pre_apply_inverse,
device buffers) at the config-3 and config-5 shapes: kernel times from the
library's CUDA events and HBM fraction of U read twice (diagnostic)."""
import ctypes as C, json, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import lib, _vp, _i64
ctx = npcg.Context(0)
peak = 6546.6
out = []
for n, ell, s in ((50000, 1000, 1), (100000, 2000, 1), (100000, 2000, 4)):
    rng = np.random.default_rng(0)
    u = np.asfortranarray(rng.standard_normal((n, ell)) / np.sqrt(n))
    lam = np.sort(rng.random(ell))[::-1].copy()
    pre = npcg.build_preconditioner(npcg.make_approximation(u, lam, ctx=ctx), 1e-3)
    r = torch.randn(s, n, dtype=torch.float64, device='cuda').t()  # column-major n x s
    z = torch.empty(s, n, dtype=torch.float64, device='cuda').t()
    def call():
        npcg._check(lib().npcg_pre_apply_inverse(_vp(pre.h), _i64(s), C.c_void_p(r.data_ptr()), _i64(n),
                                                 C.c_void_p(z.data_ptr()), _i64(n), 1))
    for _ in range(3):
        call()
    ctx.sync()
    ctx.prof_enable(True)
    reps = 20
    for _ in range(reps):
        call()
    ctx.sync()
    rep = ctx.prof_report()
    ctx.prof_enable(False)
    ms = sum(v[1] for v in rep.values()) / reps
    alg = 2 * 8.0 * n * ell + 3 * 8.0 * n * s  # U twice + r, z, r
    line = {"n": n, "ell": ell, "s": s, "us_per_apply": round(ms * 1e3, 1), "GBps": round(alg / (ms * 1e-3) / 1e9, 1),
            "frac_of_hbm": round(alg / (ms * 1e-3) / 1e9 / peak, 3),
            "kernels": {k: round(v[1] / reps * 1e3, 1) for k, v in rep.items()}}
    print(json.dumps(line), flush=True)
    out.append(line)
    del pre
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
