"""Run tests/dist_worker.solve_all on an unsharded context with a traceback dump
if it stalls (diagnostic)."""
import faulthandler, sys, time
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
faulthandler.dump_traceback_later(90, exit=True)
import paper_2110_02820_b200 as npcg
from paper_2110_02820_b200 import workloads
npcg.workloads = workloads
import dist_worker
t = time.time()
out = dist_worker.solve_all(npcg, npcg.Context(0), lambda n: (0, n))
print("done %.1f s" % (time.time() - t), sorted(out))
