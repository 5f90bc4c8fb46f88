import sys, time
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
npcg.workloads = workloads
import dist_worker
probs = dist_worker._problems(npcg)
ctx = npcg.Context(0)
for name in sys.argv[1:]:
    w = probs[name]
    t = time.time()
    op = workloads.build_operator(npcg, w, ctx=ctx)
    pair = npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, w.omega)
    ap = npcg.nystrom_from_sketch(pair)
    b = w.b.reshape(w.n, -1, order="F")
    print(name, "sketch ok", b.shape, flush=True)
    for mu in (w.mus or [w.mu]):
        pre = npcg.build_preconditioner(ap, mu)
        reps = npcg.nystrom_pcg(op, b, mu, pre, eta=w.eta, relative=True)
        reps = reps if isinstance(reps, list) else [reps]
        print(name, mu, [r.iterations for r in reps], "%.2f s" % (time.time() - t), flush=True)
    if name == "cfg5":
        br = npcg.block_nystrom_pcg(op, b, w.mus[-1], npcg.build_preconditioner(ap, w.mus[-1]), eta=w.eta, relative=True)
        print("block", br.iterations, flush=True)
