"""Spawn the GPU dist-test workers repeatedly with a stall watchdog (diagnostic):
  python tools/repro_dist.py <reps>"""
import faulthandler, multiprocessing as mp, os, socket, sys, time
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import dist_worker


def port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def guarded(fn, args):
    faulthandler.enable()
    faulthandler.dump_traceback_later(100, exit=True)
    fn(*args)


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        for name, fn, argsets in (("ref", dist_worker.gpu_reference, [()]),):
            q = ctx.Queue()
            pt = port()
            if argsets is None:
                argsets = [(r, 2, pt) for r in range(2)] if name == "world2" else [(pt,)]
            procs = [ctx.Process(target=guarded, args=(fn, (*a, q))) for a in argsets]
            t = time.time()
            for p in procs:
                p.start()
            got = 0
            try:
                for _ in procs:
                    r, v = q.get(timeout=110)
                    got += 1
                    if isinstance(v, str):
                        print(name, "ERROR", v[-500:], flush=True)
            except Exception as e:  # noqa: BLE001
                print(name, "TIMEOUT", repr(e), flush=True)
            for p in procs:
                p.join(timeout=20)
                if p.is_alive():
                    p.kill()
            print(rep, name, "results", got, "/", len(procs), "%.1f s" % (time.time() - t),
                  "exitcodes", [p.exitcode for p in procs], flush=True)
