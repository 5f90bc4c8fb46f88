"""chol_fused_kernel time vs grid size / n, via orthonormal_columns (diagnostic)."""
import os, sys, subprocess
sys.path.insert(0, '.')
if len(sys.argv) > 1:
    import numpy as np
    import paper_2110_02820_b200 as npcg
    ctx = npcg.Context(0)
    for (m, n) in [(4000, 100), (4000, 400), (8000, 1000)]:
        g = np.random.default_rng(0).standard_normal((m, n))
        npcg.orthonormal_columns(g, ctx=ctx)
        ctx.prof_enable(True)
        npcg.orthonormal_columns(g, ctx=ctx)
        prof = ctx.prof_report()
        ctx.prof_enable(False)
        v = prof.get('chol_fused_kernel')
        print(os.environ.get('NPCG_CHOL_GRID', 'auto'), (m, n), 'chol_fused %d launches %.1f us each' % (v[0], v[1] * 1e3 / v[0]) if v else prof.keys(), flush=True)
else:
    for gsz in ['', '1', '4', '16', '48']:
        env = dict(os.environ)
        if gsz: env['NPCG_CHOL_GRID'] = gsz
        subprocess.run([sys.executable, __file__, 'x'], env=env)
