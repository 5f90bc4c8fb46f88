"""One small cold-start regularisation path (one 8-column persistent solve); for compute-sanitizer runs."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
w = workloads.make('cfg5', npcg.Rng, npcg.splitmix64, n=n, r=200, ell=100, nrhs=4, nmu=2)
op = npcg.LowRankOperator(w.data["g"], w.data["lambda"])
ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, w.omega))
cold = npcg.regularization_path(op, w.b, w.mus, ap, warm_start=False, eta=w.eta, relative=True, max_iter=int(sys.argv[2]) if len(sys.argv) > 2 else 500)
print([[r.iterations for r in reps] for _, reps in cold])
