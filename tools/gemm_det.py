"""GEMM determinism / correctness probe across forced tile plans (diagnostic)."""
import os, sys, subprocess
sys.path.insert(0, os.environ.get('NPCG_ROOT', '.'))
if len(sys.argv) > 1:
    import numpy as np
    import paper_2110_02820_b200 as npcg
    rng = np.random.default_rng(3)
    for (m, n, k) in [(200, 200, 4000), (256, 256, 4000), (400, 400, 4000), (130, 90, 2000)]:
        a = rng.standard_normal((k, m)); b = rng.standard_normal((k, n))
        ref = a.T @ b
        g = [npcg.gemm(a, b, transa=True) for _ in range(4)]
        same = all(np.array_equal(g[0], x) for x in g[1:])
        err = max(np.abs(x - ref).max() for x in g)
        print(os.environ.get("NPCG_GEMM_FORCE", "auto"), (m, n, k), "deterministic" if same else "NONDET", "maxerr %.2e" % err, flush=True)
else:
    for f in ["", "w:1", "w:8", "w:41", "n:1", "n:8", "n:41"]:
        env = dict(os.environ)
        if f: env["NPCG_GEMM_FORCE"] = f
        subprocess.run([sys.executable, __file__, "x"], env=env)
