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
s0 = time.perf_counter()
iters = path.step()
ctx.sync()
s1 = time.perf_counter()
# residual check: || (K + mu I) x - b || / || b || with one more matvec
x = path.x[0].cpu().numpy()
r = path.op.matvec(x) + w.mu * x - w.b
rel = float(np.linalg.norm(r) / np.linalg.norm(w.b))
out = {"workload": w.name, "n": n, "d": 32, "sigma": 0.5, "mu": w.mu, "eta": w.eta,
       "adaptive_ell_final_doublings_hitcap": list(path.adaptive_outcome), "pcg_iterations": iters[0][0],
       "converged": iters[0][1], "solve_seconds": s1 - s0, "true_relative_residual": rel,
       "note": "one full solve (adaptive sketch + factorisations + PCG) on one B200; host Rng draws included"}
print(json.dumps(out), flush=True)
if n == 1_000_000:
    with open("profiles/cfg4_full_r01.json", "w") as f:
        json.dump(out, f, indent=1)
