"""BASELINE config 4 at full size on one B200: matrix-free Gaussian KRR,
n = 1e6 points in [0,1]^32, sigma = 0.5, mu = 1e-7 n, adaptive rank search
(error strategy, ell0 = 50 doubling to ell_max = 3200, tau = 10, q = 5), PCG to
rel-res 1e-8. One solve (the CPU oracle cannot run this size; see the reduced
config-4 parity tests). Writes profiles/cfg4_full_r01.json (diagnostic)."""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
import bench
npcg.workloads = workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ctx = npcg.Context(0)
t0 = time.perf_counter()
w = workloads.make('cfg4', npcg.Rng, npcg.splitmix64, n=n)
t1 = time.perf_counter()
path = bench.DevicePath(npcg, torch, w, ctx)
t2 = time.perf_counter()
print("inputs %.1f s, operator %.1f s" % (t1 - t0, t2 - t1), flush=True)
prof = len(sys.argv) > 2 and sys.argv[2] == 'prof'
if prof:
    ctx.prof_enable(True)
s0 = time.perf_counter()
iters = path.step()
ctx.sync()
s1 = time.perf_counter()
kernels = {}
if prof:
    rep = ctx.prof_report()
    ctx.prof_enable(False)
    fam = {}
    for name, v in rep.items():
        key = name.split('[')[0]
        f = fam.setdefault(key, [0, 0.0, 0.0])
        f[0] += v[0]; f[1] += v[1]; f[2] += v[2]
    for name, v in sorted(fam.items(), key=lambda kv: -kv[1][1])[:16]:
        kernels[name] = {"launches": v[0], "s": round(v[1] / 1e3, 3),
                         "tflops": round(v[2] / (v[1] * 1e-3) / 1e12, 2) if v[2] and v[1] else None}
    kernels["_total_kernel_s"] = round(sum(v[1] for v in rep.values()) / 1e3, 3)
# residual check: || (K + mu I) x - b || / || b || with one more matvec
x = path.x[0].cpu().numpy()
r = path.op.matvec(x) + w.mu * x - w.b
rel = float(np.linalg.norm(r) / np.linalg.norm(w.b))
out = {"workload": w.name, "n": n, "d": 32, "sigma": 0.5, "mu": w.mu, "eta": w.eta,
       "adaptive_ell_final_doublings_hitcap": list(path.adaptive_outcome), "pcg_iterations": iters[0][0],
       "converged": iters[0][1], "solve_seconds": s1 - s0, "true_relative_residual": rel,
       "note": "one full solve (adaptive sketch + factorisations + PCG) on one B200; host Rng draws included",
       "kernels": kernels}
print(json.dumps(out), flush=True)
if n == 1_000_000:
    with open(sys.argv[3] if len(sys.argv) > 3 else "profiles/cfg4_full_r01.json", "w") as f:
        json.dump(out, f, indent=1)
