"""Matrix-free RBF operator: time and agreement of the fused (k <= 2), row-block and scalar paths (diagnostic)."""
import os, subprocess, sys, time
sys.path.insert(0, '.')
if len(sys.argv) > 2:
    import numpy as np
    import paper_2110_02820_b200 as npcg
    ctx = npcg.Context(0)
    n, d = int(sys.argv[1]), int(sys.argv[2])
    pts = np.random.default_rng(0).random((n, d))
    op = npcg.KernelOperator(pts, 0.5, dense_cap=1000, ctx=ctx)
    for k in ((1, 2, 400) if n <= 50000 else (1, 2)):
        V = np.random.default_rng(1).standard_normal((n, k))
        r = op.apply_block(V)
        ctx.sync(); t = time.perf_counter(); op.apply_block(V); ctx.sync(); dt = time.perf_counter() - t
        np.save('/tmp/kf_%s_%d.npy' % (os.environ.get('NPCG_KFREE', 'auto'), k), r)
        print(os.environ.get('NPCG_KFREE', 'auto'), "n=%d d=%d k=%d %.4f s" % (n, d, k, dt), flush=True)
else:
    import numpy as np
    n, d = (sys.argv[1] if len(sys.argv) > 1 else '50000'), '32'
    for mode in ['', 'rowwise', 'blocked']:
        env = dict(os.environ)
        if mode: env['NPCG_KFREE'] = mode
        subprocess.run([sys.executable, __file__, n, d], env=env)
    for k in (1, 2):
        a, b = np.load('/tmp/kf_auto_%d.npy' % k), np.load('/tmp/kf_blocked_%d.npy' % k)
        r = np.load('/tmp/kf_rowwise_%d.npy' % k)
        print('k=%d symmetric vs blocked max rel diff %.2e, rowwise vs blocked %.2e' % (
            k, np.abs(a - b).max() / np.abs(b).max(), np.abs(r - b).max() / np.abs(b).max()))
