"""Synthetic stand-ins for the BASELINE.json configs.

The reference's paper benchmarks run on real datasets that are not in this
container; these generators reproduce the shapes, sizes and value
distributions BASELINE.json names, drawing every random number from the
reference's own generator (mt19937_64 + Box-Muller, random.cpp:11-32) with the
bench.cpp seed convention: data stream Rng(splitmix64(k)), solve stream Rng(k)
(b first when it is random, then the raw Gaussian test matrix Omega).

`make(name, rng_factory, gemm)` is implementation-agnostic so the tests can
build bit-identical inputs with the oracle's Rng.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    kind: str                 # "dense" | "gram" | "kernel" | "lowrank" | "synth"
    n: int                    # operator dimension
    mu: float
    ell: int                  # fixed sketch size (adaptive: ell_max)
    eta: float = 1e-10
    relative: bool = True
    max_iter: int = 500
    data: dict = field(default_factory=dict)  # operator inputs
    b: np.ndarray | None = None               # n or n x s
    omega: np.ndarray | None = None           # raw Gaussian n x ell (fixed-rank configs)
    adaptive: dict | None = None
    mus: list | None = None                   # config 5 regularisation path

    def describe(self) -> dict:
        d = {"workload": self.name, "n": self.n, "mu": self.mu, "ell": self.ell, "eta": self.eta,
             "relative": self.relative}
        if self.kind == "gram":
            d["m"] = self.data["x"].shape[0]
        if self.kind in ("kernel",):
            d["d"] = self.data["points"].shape[1]
            d["sigma"] = self.data["sigma"]
        return d


def _np_gemm(a, b, transa=False, transb=False):
    return (a.T if transa else a) @ (b.T if transb else b)


def cfg1(Rng, splitmix64, n=2000, ell=100, **_):
    """Dense synthetic psd: A = Q diag(j^-2) Q^T (synthesize_operator), mu=1e-4."""
    lam = np.array([(j + 1.0) ** -2.0 for j in range(n)])
    rng = Rng(1)
    b = rng.gaussian_vector(n)
    omega = rng.gaussian_matrix(n, ell)
    return Workload("cfg1_dense_poly_n%d_l%d" % (n, ell), "synth", n, 1e-4, ell,
                    data={"lambda": lam, "seed": splitmix64(1)}, b=b, omega=omega)


def cfg2(Rng, splitmix64, m=20000, n=4000, ell=400, gemm=_np_gemm, **_):
    """Ridge: A = X^T X / m, X_ij = N(0,1) j^-0.5; b = X^T y / m, y = X w* + 0.1 N(0,1); mu=1e-3."""
    data = Rng(splitmix64(2))
    x = data.gaussian_matrix(m, n)
    x *= np.array([(j + 1.0) ** -0.5 for j in range(n)])[None, :]
    w = data.gaussian_vector(n)
    noise = data.gaussian_vector(m)
    y = gemm(x, w.reshape(-1, 1))[:, 0] + 0.1 * noise
    b = gemm(x, y.reshape(-1, 1), transa=True)[:, 0] / m
    rng = Rng(2)  # b comes from the data: the solve stream starts at Omega
    omega = rng.gaussian_matrix(n, ell)
    return Workload("cfg2_ridge_m%d_n%d_l%d" % (m, n, ell), "gram", n, 1e-3, ell, data={"x": x}, b=b, omega=omega)


def cfg3(Rng, splitmix64, n=50000, d=64, ell=1000, **_):
    """Gaussian KRR, stored kernel: 10-component mixture in d=64, sigma=8, mu=1e-6 n."""
    data = Rng(splitmix64(3))
    means = 2.0 * data.gaussian_matrix(10, d)
    pts = np.empty((n, d), order="F")
    comps = np.empty(n, dtype=np.int64)
    for i in range(n):
        comps[i] = data.integer(10)
        pts[i, :] = means[comps[i]] + data.gaussian_vector(d)
    rng = Rng(3)
    b = rng.gaussian_vector(n)
    omega = rng.gaussian_matrix(n, ell)
    return Workload("cfg3_krr_stored_n%d_d%d_l%d" % (n, d, ell), "kernel", n, 1e-6 * n, ell,
                    data={"points": pts, "sigma": 8.0, "dense_cap": max(n, 20000)}, b=b, omega=omega)


def cfg4(Rng, splitmix64, n=1_000_000, d=32, ell0=50, ell_max=3200, **_):
    """Matrix-free RBF KRR: uniform [0,1]^32, sigma=0.5, mu=1e-7 n, adaptive error strategy, tol 1e-8."""
    data = Rng(splitmix64(4))
    pts = np.asfortranarray(data.uniform_fill(n * d).reshape(n, d))
    rng = Rng(4)
    b = rng.gaussian_vector(n)
    return Workload("cfg4_rbf_free_n%d_d%d" % (n, d), "kernel", n, 1e-7 * n, ell_max, eta=1e-8,
                    data={"points": pts, "sigma": 0.5, "dense_cap": 20000}, b=b,
                    adaptive={"ell0": ell0, "ell_max": ell_max, "tau": 10.0, "q": 5})


def cfg5(Rng, splitmix64, n=100_000, r=5000, ell=2000, nrhs=4, nmu=20, **_):
    """Regularisation path: A = G diag(exp(-j/500)) G^T / r, one sketch, 20 mu in [1e-6, 1e-1], 4 RHS."""
    data = Rng(splitmix64(5))
    g = data.gaussian_matrix(n, r)
    lam = np.exp(-np.arange(1, r + 1) / 500.0)
    rng = Rng(5)
    b = rng.gaussian_matrix(n, nrhs)
    omega = rng.gaussian_matrix(n, ell)
    mus = [10.0 ** (-6 + 5 * k / (nmu - 1)) for k in range(nmu)]
    return Workload("cfg5_regpath_n%d_r%d_l%d" % (n, r, ell), "lowrank", n, mus[0], ell,
                    data={"g": g, "lambda": lam}, b=b, omega=omega, mus=mus)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def make(name: str, Rng, splitmix64, **kw) -> Workload:
    return CONFIGS[name](Rng, splitmix64, **kw)


def build_operator(npcg, w: Workload, ctx=None, streamed=False):
    """The product operator for a workload (device-resident). On a row-sharded
    context (dist.nccl_context / dist.exchange_context) the same constructors
    keep this rank's share: the column block A[:, R_g] of the dense / stored
    kernel / low-rank operators, the rows of X for the ridge Gram operator, a
    share of the matrix-free kernel work. `streamed` overlaps the upload of a
    ridge design with the sketch (npcg_op_gram_create_streamed)."""
    if w.kind == "synth":
        return npcg.synthesize_operator(w.data["lambda"], w.data["seed"], ctx=ctx)
    if w.kind == "dense":
        return npcg.DenseOperator(w.data["a"], ctx=ctx)
    if w.kind == "gram":
        return npcg.GramRidgeOperator(w.data["x"], ctx=ctx, streamed=streamed)
    if w.kind == "kernel":
        return npcg.KernelOperator(w.data["points"], w.data["sigma"], w.data["dense_cap"], ctx=ctx)
    if w.kind == "lowrank":
        return npcg.LowRankOperator(w.data["g"], w.data["lambda"], ctx=ctx)
    raise ValueError(w.kind)
