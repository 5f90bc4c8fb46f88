"""Repeated cold-start regularisation paths (8-column persistent solves) over several sizes; each must
reproduce the per-mu solves' iteration counts (diagnostic: catches intermittent synchronisation faults)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
ok = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    for n, r, ell, s in ((3000, 200, 100, 4), (5200, 300, 333, 4), (9000, 300, 150, 2), (1500, 100, 64, 1), (20000, 400, 400, 4)):
        w = workloads.make('cfg5', npcg.Rng, npcg.splitmix64, n=n, r=r, ell=ell, nrhs=4, nmu=4)
        op = npcg.LowRankOperator(w.data["g"], w.data["lambda"])
        ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, w.omega))
        b = np.asfortranarray(w.b[:, :s])
        cold = npcg.regularization_path(op, b, w.mus, ap, warm_start=False, eta=w.eta, relative=True)
        for k, mu in enumerate(w.mus):
            reps = npcg.nystrom_pcg(op, b, mu, npcg.build_preconditioner(ap, mu), eta=w.eta, relative=True)
            reps = reps if isinstance(reps, list) else [reps]
            for j, rp in enumerate(reps):
                assert abs(cold[k][1][j].iterations - rp.iterations) <= 1, (n, mu, j)
        ok += 1
print("stress ok:", ok, "paths")
