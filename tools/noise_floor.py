"""Noise floor of the parity bar: the oracle run with 1
OpenBLAS thread and with all host cores on identical inputs, and the B200
library on the same inputs. Reports, per config, the iteration counts and the
lambda / x relative deviations of every pair, so the GPU-vs-oracle deltas can
be read against the oracle's own 1-vs-N-thread spread.

    python tools/noise_floor.py [out.json]      (needs the GPU for the b200 leg)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from oracle.workload_ops import build_oracle_operator  # noqa: E402
from paper_2110_02820_b200 import workloads  # noqa: E402

CASES = [("cfg1", {}), ("cfg2", {}), ("cfg3", {"n": 20000, "ell": 1000}),
         ("cfg5", {"n": 10000, "r": 1000, "ell": 400, "nmu": 2})]


def lam_rel(a, b):
    keep = b >= 1e-6 * b[0]
    return float(np.max(np.abs(a[keep] - b[keep]) / b[keep]))


def x_rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_run(w, threads):
    orc.set_threads(threads)
    op = build_oracle_operator(orc, w)
    t0 = time.perf_counter()
    ap = orc.nystrom_from_sketch(orc.extend_sketch_with(orc.make_empty_sketch(w.n), op, w.omega))
    pre = orc.build_preconditioner(ap, w.mu)
    b = w.b.reshape(w.n, -1, order="F")[:, 0]
    rep = orc.nystrom_pcg(op, b, w.mu, pre, eta=w.eta, max_iter=w.max_iter, relative=w.relative)
    return {"lam": ap.lam, "x": rep.x, "iterations": rep.iterations, "seconds": time.perf_counter() - t0}


def b200_run(w):
    import paper_2110_02820_b200 as npcg
    npcg.workloads = workloads
    op = workloads.build_operator(npcg, w)
    ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, w.omega))
    pre = npcg.build_preconditioner(ap, w.mu)
    b = w.b.reshape(w.n, -1, order="F")[:, 0]
    rep = npcg.nystrom_pcg(op, b, w.mu, pre, eta=w.eta, max_iter=w.max_iter, relative=w.relative)
    return {"lam": ap.lam, "x": rep.x, "iterations": rep.iterations}


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "profiles/noise_floor_r02.json"
    ncores = os.cpu_count() or 1
    rows = []
    for name, kw in CASES:
        w = workloads.make(name, orc.Rng, orc.splitmix64, **kw)
        r1 = oracle_run(w, 1)
        rn = oracle_run(w, ncores)
        rg = b200_run(w)
        row = {"workload": w.name, "iterations": {"oracle_1t": r1["iterations"], f"oracle_{ncores}t": rn["iterations"],
                                                  "b200": rg["iterations"]},
               "lambda_rel": {"oracle_1t_vs_Nt": lam_rel(rn["lam"], r1["lam"]), "b200_vs_1t": lam_rel(rg["lam"], r1["lam"]),
                              "b200_vs_Nt": lam_rel(rg["lam"], rn["lam"])},
               "x_rel": {"oracle_1t_vs_Nt": x_rel(rn["x"], r1["x"]), "b200_vs_1t": x_rel(rg["x"], r1["x"]),
                         "b200_vs_Nt": x_rel(rg["x"], rn["x"])},
               "oracle_seconds": {"1t": r1["seconds"], f"{ncores}t": rn["seconds"]}}
        print(json.dumps(row), flush=True)
        rows.append(row)
    with open(out_path, "w") as f:
        json.dump({"threads": ncores, "openblas_core": orc.corename(), "rows": rows,
                   "note": "lambda_rel over lambda_j >= 1e-6 lambda_1; x_rel = ||x - x_ref|| / ||x_ref||"}, f, indent=1)


if __name__ == "__main__":
    main()
