"""Throughput of forced GEMM plans on a few shapes (diagnostic)."""
import os, sys, subprocess
sys.path.insert(0, '.')
if len(sys.argv) > 1:
    import ctypes as C, torch
    import paper_2110_02820_b200 as npcg
    ctx = npcg.Context(0); L = npcg.lib(); stream = torch.cuda.ExternalStream(ctx.stream)
    m, n, k = (int(x) for x in sys.argv[1:4])
    a = torch.randn((m, k), dtype=torch.float64, device='cuda'); b = torch.randn((n, k), dtype=torch.float64, device='cuda')
    c = torch.zeros((n, m), dtype=torch.float64, device='cuda'); torch.cuda.synchronize()
    def call():
        npcg._check(L.npcg_gemm(C.c_void_p(ctx.h), C.c_int64(m), C.c_int64(n), C.c_int64(k), C.c_double(1.0),
                                C.c_void_p(a.data_ptr()), C.c_int64(k), C.c_int(1), C.c_void_p(b.data_ptr()),
                                C.c_int64(k), C.c_int(1), C.c_double(0.0), C.c_void_p(c.data_ptr()), C.c_int64(m), 1))
    call(); s, e = torch.cuda.Event(True), torch.cuda.Event(True); best = 1e9
    for _ in range(5):
        s.record(stream); call(); e.record(stream); e.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
    print(os.environ.get('NPCG_GEMM_FORCE', 'auto'), (m, n, k), '%.2f TF/s' % (2 * m * n * k / best / 1e12), flush=True)
else:
    for shape in [('20000', '400', '4000'), ('4000', '400', '20000'), ('8192', '8192', '8192')]:
        for f in ['', 't:1', 't:2', 't:3', 't:5', 't:9', 'n:3', 'w:1']:
            env = dict(os.environ)
            if f: env['NPCG_GEMM_FORCE'] = f
            if shape[0] == '8192' and f not in ('', 't:1', 'w:1'): continue
            subprocess.run([sys.executable, __file__, *shape], env=env)
