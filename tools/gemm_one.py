"""One GEMM through the C-ABI for sanitizer runs (diagnostic)."""
import os, sys
sys.path.insert(0, os.environ.get('NPCG_ROOT', '.'))
import numpy as np
import paper_2110_02820_b200 as npcg
rng = np.random.default_rng(3)
m, n, k = (int(x) for x in sys.argv[1:4])
a = rng.standard_normal((k, m)); b = rng.standard_normal((k, n))
g = npcg.gemm(a, b, transa=True)
print("maxerr %.3e" % np.abs(g - a.T @ b).max())
