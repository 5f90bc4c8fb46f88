"""The reference's benchmark harness over the B200 library:
bench.hpp / bench.cpp restated -- ProblemSpec, the FNV-1a spec hash,
run_benchmark / run_benchmark_trials producing BenchRecord JSON lines,
summarize(), random_features(). Every solve runs through this package's
C-ABI (libnpcg_b200.so); only the orchestration is Python, as the reference's
is host C++.

Reference: /root/reference/proj/core/src/bench.cpp (file:line per function).
"""
from __future__ import annotations

import json
import math
import struct
import time
from dataclasses import dataclass, field

import numpy as np

import paper_2110_02820_b200 as npcg
from . import matrix_io

SOLVERS = ("cg", "nystrom_pcg", "sketch_and_solve", "block_pcg")          # bench.hpp SolverKind order
POLICIES = ("fixed", "adaptive_error", "adaptive_ratio")                   # RankPolicy order
CONVENTIONS = ("mu", "n_mu")                                               # RegularizerConvention order
FORMATS = ("matrix_market", "csv_dense", "raw_f64")                        # io::MatrixFormat order


@dataclass
class FileSource:
    path: str
    format: str = "matrix_market"


@dataclass
class RidgeSource:
    design: np.ndarray  # G, n_rows x d; operator (1/n_rows) G^T G


@dataclass
class KrrSource:
    points: np.ndarray  # one row per point
    sigma: float = 1.0
    convention: str = "n_mu"


@dataclass
class ProblemSpec:
    """bench.hpp:44-63: everything needed to run (and re-run) one problem."""
    problem_id: str = "problem"
    file: FileSource | None = None
    synthetic: np.ndarray | None = None  # SpectrumProfile eigenvalues
    ridge: RidgeSource | None = None
    krr: KrrSource | None = None
    solver: str = "nystrom_pcg"
    policy: str = "fixed"
    mu: float = 0.0
    eta: float = 1e-10
    relative_tol: bool = False
    max_iter: int = 500
    rank: int = 0
    ell0: int = 10
    ell_max: int = 0
    tau: float | None = None
    rhs: np.ndarray | None = None
    seed: int = 0


@dataclass
class PhaseTimes:
    sketch: float = 0.0
    precondition: float = 0.0
    solve: float = 0.0
    total: float = 0.0


@dataclass
class BenchRecord:
    """bench.hpp:74-93: one trial's metrics."""
    problem_id: str = ""
    n: int = 0
    d: int = 0
    mu: float = 0.0
    ell_final: int = 0
    iterations: int = 0
    times: PhaseTimes = field(default_factory=PhaseTimes)
    residual: float = 0.0
    error_estimate: float | None = None
    posterior_condition: float | None = None
    converged: bool = False
    failure: str = ""
    seed: int = 0
    spec_hash: str = ""

    def json_line(self) -> str:  # bench.cpp:323-345
        j = {"problem_id": self.problem_id, "n": self.n, "d": self.d, "mu": self.mu, "ell_final": self.ell_final,
             "iterations": self.iterations, "sketch_time": self.times.sketch,
             "precondition_time": self.times.precondition, "solve_time": self.times.solve,
             "total_time": self.times.total, "residual": self.residual}
        if self.error_estimate is not None:
            j["error_estimate"] = self.error_estimate
        if self.posterior_condition is not None:
            j["posterior_condition"] = self.posterior_condition
        j["converged"] = self.converged
        if self.failure:
            j["failure"] = self.failure
        j["seed"] = self.seed
        j["spec_hash"] = self.spec_hash
        return json.dumps(j)


class Fnv1a:
    """bench.cpp:30-72: 64-bit FNV-1a over the fields' byte images (the
    reference's offset basis 1469598103934665603 is kept as written)."""
    MASK = (1 << 64) - 1

    def __init__(self):
        self.h = 1469598103934665603

    def bytes(self, data: bytes):
        h = self.h
        for c in data:
            h ^= c
            h = (h * 1099511628211) & self.MASK
        self.h = h

    def add_str(self, s: str):
        self.bytes(s.encode() + b"\0")

    def add_u64(self, v: int):
        self.bytes(struct.pack("<Q", v & self.MASK))

    def add_f64(self, v: float):
        self.bytes(struct.pack("<d", float(v)))

    def add_vector(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64).ravel()
        self.add_u64(v.size)
        self.bytes(v.astype("<f8").tobytes())

    def add_matrix(self, m):
        m = np.asarray(m, dtype=np.float64)
        self.add_u64(m.shape[0])
        self.add_u64(m.shape[1])
        self.bytes(np.asfortranarray(m).ravel(order="F").astype("<f8").tobytes())

    def hex(self) -> str:
        return "%016x" % self.h


def spec_hash(spec: ProblemSpec) -> str:  # bench.cpp:143-178
    f = Fnv1a()
    f.add_str(spec.problem_id)
    if spec.file is not None:
        f.add_str("file")
        f.add_str(spec.file.path)
        f.add_u64(FORMATS.index(spec.file.format))
    elif spec.synthetic is not None:
        f.add_str("synthetic")
        f.add_vector(spec.synthetic)
    elif spec.ridge is not None:
        f.add_str("ridge")
        f.add_matrix(spec.ridge.design)
    elif spec.krr is not None:
        f.add_str("krr")
        f.add_matrix(spec.krr.points)
        f.add_f64(spec.krr.sigma)
        f.add_u64(CONVENTIONS.index(spec.krr.convention))
    else:
        f.add_str("none")
    f.add_u64(SOLVERS.index(spec.solver))
    f.add_u64(POLICIES.index(spec.policy))
    f.add_f64(spec.mu)
    f.add_f64(spec.eta)
    f.add_u64(int(spec.relative_tol))
    f.add_u64(spec.max_iter)
    f.add_u64(spec.rank)
    f.add_u64(spec.ell0)
    f.add_u64(spec.ell_max)
    f.add_u64(int(spec.tau is not None))
    if spec.tau is not None:
        f.add_f64(spec.tau)
    f.add_u64(int(spec.rhs is not None))
    if spec.rhs is not None:
        f.add_vector(spec.rhs)
    return f.hex()


def synthetic_operator_seed(seed: int) -> int:  # bench.cpp:180-185
    return npcg.splitmix64(seed)


def _recommended_sketch_size(lam, mu) -> int:  # diagnostics.cpp:31-35
    deff = float(np.sum(lam / (lam + mu)))
    return min(2 * int(math.ceil(1.5 * deff)) + 1, len(lam))


def build_problem(spec: ProblemSpec, ctx=None):  # bench.cpp:80-111
    sources = sum(x is not None for x in (spec.file, spec.synthetic, spec.ridge, spec.krr))
    if sources != 1:
        raise npcg.InvalidArgument("run_benchmark: exactly one problem source required")
    if spec.mu < 0.0:
        raise npcg.InvalidArgument("run_benchmark: mu must be >= 0")
    shift = spec.mu
    if spec.file is not None:
        m = matrix_io.require_symmetric(matrix_io.load_matrix(spec.file.path, spec.file.format.replace("_", "-")),
                                        "run_benchmark")
        return npcg.DenseOperator(m, ctx=ctx), shift, m.shape[0]
    if spec.synthetic is not None:
        lam = np.asarray(spec.synthetic, dtype=np.float64)
        return npcg.synthesize_operator(lam, synthetic_operator_seed(spec.seed), ctx=ctx), shift, lam.size
    if spec.ridge is not None:
        g = np.asarray(spec.ridge.design, dtype=np.float64)
        return npcg.GramRidgeOperator(g, ctx=ctx), shift, g.shape[0]
    pts = np.asarray(spec.krr.points, dtype=np.float64)
    op = npcg.KernelOperator(pts, spec.krr.sigma, ctx=ctx)
    if spec.krr.convention == "n_mu":
        shift = spec.mu * op.dim()
    return op, shift, pts.shape[1]


def _resolve_fixed_rank(spec, shift, n) -> int:  # bench.cpp:113-124
    if spec.rank > 0:
        if spec.rank > n:
            raise npcg.InvalidArgument("run_benchmark: rank exceeds problem dimension")
        return spec.rank
    if spec.synthetic is not None and shift > 0.0:
        return _recommended_sketch_size(np.asarray(spec.synthetic, dtype=np.float64), shift)
    raise npcg.InvalidArgument("run_benchmark: fixed rank policy needs an explicit rank for this source")


def run_benchmark(spec: ProblemSpec, ctx=None) -> BenchRecord:  # bench.cpp:187-290
    rec = BenchRecord(problem_id=spec.problem_id, mu=spec.mu, seed=spec.seed, spec_hash=spec_hash(spec))
    try:
        op, shift, data_dim = build_problem(spec, ctx)
        n = op.dim()
        rec.n, rec.d = n, data_dim
        rng = npcg.Rng(spec.seed)
        if spec.rhs is not None:
            b = np.asarray(spec.rhs, dtype=np.float64)
            if b.size != n:
                raise npcg.InvalidArgument("run_benchmark: right-hand side length mismatch")
        else:
            b = rng.gaussian_vector(n)
        opts = dict(eta=spec.eta, max_iter=spec.max_iter, relative=spec.relative_tol)
        run_start = time.perf_counter()
        if spec.solver == "cg":
            t0 = time.perf_counter()
            rep = npcg.cg(npcg.regularize(op, shift), b, **opts)
            rec.times.solve = time.perf_counter() - t0
            rec.iterations, rec.residual, rec.converged = rep.iterations, float(rep.residual_history[-1]), \
                rep.converged
        else:
            t0 = time.perf_counter()
            if spec.policy == "fixed":
                approx = npcg.randomized_nystrom(op, _resolve_fixed_rank(spec, shift, n), rng)
            else:
                out = npcg.adaptive(op, rng, mode="ratio" if spec.policy == "adaptive_ratio" else "error",
                                    ell0=spec.ell0, ell_max=spec.ell_max if spec.ell_max > 0 else n, mu=shift,
                                    tau=spec.tau, sketch="column" if spec.krr is not None else "gaussian")
                approx = out.approximation
                rec.error_estimate = out.error_estimate
                rec.posterior_condition = out.posterior_condition_estimate
            rec.times.sketch = time.perf_counter() - t0
            rec.ell_final = approx.size()
            if spec.solver == "sketch_and_solve":
                t0 = time.perf_counter()
                x = npcg.woodbury_inverse_apply(approx, shift, b)
                rec.times.solve = time.perf_counter() - t0
                r = b - op.matvec(x)
                r -= shift * x
                rec.residual = float(np.linalg.norm(r))
                rec.iterations = 0
                rec.converged = rec.residual <= (spec.eta * np.linalg.norm(b) if spec.relative_tol else spec.eta)
            else:
                t0 = time.perf_counter()
                pre = npcg.build_preconditioner(approx, shift)
                rec.times.precondition = time.perf_counter() - t0
                t0 = time.perf_counter()
                if spec.solver == "block_pcg":
                    brep = npcg.block_nystrom_pcg(op, b.reshape(-1, 1), shift, pre, **opts)
                    rec.times.solve = time.perf_counter() - t0
                    rec.iterations, rec.residual = brep.iterations, float(brep.residual_history[0][-1])
                    rec.converged = brep.converged[0]
                else:
                    rep = npcg.nystrom_pcg(op, b, shift, pre, **opts)
                    rec.times.solve = time.perf_counter() - t0
                    rec.iterations, rec.residual, rec.converged = rep.iterations, \
                        float(rep.residual_history[-1]), rep.converged
        rec.times.total = time.perf_counter() - run_start
    except npcg.SolveDivergenceError as e:
        rec.failure = str(e)
        rep = e.report
        if rep is not None:
            rec.iterations = rep.iterations
            if len(rep.residual_history):
                rec.residual = float(rep.residual_history[-1])
        rec.converged = False
    except Exception as e:  # noqa: BLE001 - failures are recorded, never thrown (bench.cpp:276-283)
        rec.failure = str(e) or type(e).__name__
        rec.converged = False
    return rec


def run_benchmark_trials(spec: ProblemSpec, trials: int, ctx=None) -> list[BenchRecord]:  # bench.cpp:292-321
    """Per-trial seeds seed + 0 .. seed + trials - 1, records in trial order.
    (The device serialises the trials; the reference's NPCG_THREADS host
    threads give the same records.)"""
    if trials < 1:
        raise npcg.InvalidArgument("run_benchmark_trials: trials must be >= 1")
    out = []
    for i in range(trials):
        t = ProblemSpec(**{**spec.__dict__, "seed": spec.seed + i})
        out.append(run_benchmark(t, ctx))
    return out


def summarize(records: list[BenchRecord]) -> str:  # bench.cpp:347-393
    def stats(get):
        vals = [v for v in (get(r) for r in records) if v is not None]
        if not vals:
            return None
        mean = sum(vals) / len(vals)
        var = sum((v - mean) ** 2 for v in vals)
        return {"mean": mean, "std": math.sqrt(var / (len(vals) - 1)) if len(vals) > 1 else 0.0}
    j = {"trials": len(records), "converged": sum(r.converged for r in records),
         "failures": sum(bool(r.failure) for r in records),
         "iterations": stats(lambda r: float(r.iterations)), "ell_final": stats(lambda r: float(r.ell_final)),
         "residual": stats(lambda r: r.residual), "solve_time": stats(lambda r: r.times.solve),
         "total_time": stats(lambda r: r.times.total),
         "posterior_condition": stats(lambda r: r.posterior_condition)}
    return json.dumps(j)


def random_features(x, m_rf: int, sigma: float, rng: "npcg.Rng") -> np.ndarray:  # bench.cpp:395-407
    """sqrt(2/m_rf) cos(X W + 1 phase^T), W ~ N(0, 1/sigma^2) from rng, then the
    phases 2 pi u; the product X W runs on the device DMMA GEMM."""
    if m_rf < 1:
        raise npcg.InvalidArgument("random_features: m_rf must be >= 1")
    if not sigma > 0.0:
        raise npcg.InvalidArgument("random_features: sigma must be > 0")
    x = np.asarray(x, dtype=np.float64)
    w = rng.gaussian_matrix(x.shape[1], m_rf) / sigma
    phase = np.array([2.0 * math.pi * rng.uniform() for _ in range(m_rf)])
    z = npcg.gemm(np.asfortranarray(x), np.asfortranarray(w))
    z = z + phase[None, :]
    return math.sqrt(2.0 / m_rf) * np.cos(z)
