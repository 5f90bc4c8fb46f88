"""Diagnose PCG iteration differences on config 5 at n = 20000 (mu = 4.6e-5):
batched 4-RHS persistent kernel vs single RHS vs the multi-kernel loop vs the
oracle, with residual histories."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

mode = sys.argv[1] if len(sys.argv) > 1 else "driver"
if mode == "driver":
    out = {}
    for tag, env in (("default", {}), ("classic", {"NPCG_PCG": "classic"}), ("full", {"NPCG_DENSE_FULL": "1"})):
        r = subprocess.run([sys.executable, __file__, "run"], env={**os.environ, **env}, capture_output=True, text=True)
        print(tag, r.stdout[-3000:], r.stderr[-2000:], flush=True)
    sys.exit(0)

from oracle import oracle as orc
from oracle.workload_ops import build_oracle_operator
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
w = workloads.make("cfg5", orc.Rng, orc.splitmix64, n=20000, r=1000, ell=400, nmu=4)
op = npcg.LowRankOperator(w.data["g"], w.data["lambda"])
ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, w.omega))
mu = w.mus[1]
pre = npcg.build_preconditioner(ap, mu)
reps = npcg.nystrom_pcg(op, w.b, mu, pre, eta=w.eta, relative=True)
singles = [npcg.nystrom_pcg(op, w.b[:, j], mu, pre, eta=w.eta, relative=True) for j in range(4)]
print("batched", [r.iterations for r in reps], "single", [r.iterations for r in singles])
oop = build_oracle_operator(orc, w)
ao = orc.nystrom_from_sketch(orc.extend_sketch_with(orc.make_empty_sketch(w.n), oop, w.omega))
keep = ao.lam >= 1e-6 * ao.lam[0]
print("lam err", np.max(np.abs(ap.lam[keep] - ao.lam[keep]) / ao.lam[keep]))
ro = orc.nystrom_pcg(oop, w.b[:, 0], mu, orc.build_preconditioner(ao, mu), eta=w.eta, relative=True)
print("oracle", ro.iterations)
h, hs, ho = reps[0].residual_history, singles[0].residual_history, ro.residual_history
for t in range(0, max(len(h), len(ho)), 4):
    print(t, h[t] if t < len(h) else None, hs[t] if t < len(hs) else None, ho[t] if t < len(ho) else None)
v = np.random.default_rng(0).standard_normal(w.n)
print("matvec rel diff", np.linalg.norm(op.matvec(v) - oop.matvec(v)) / np.linalg.norm(oop.matvec(v)))
