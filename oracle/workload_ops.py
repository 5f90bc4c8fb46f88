"""TEST INFRASTRUCTURE ONLY: the oracle's operator for a product Workload
(same input arrays), used by tests/ and bench.py's CPU-baseline legs."""
import numpy as np


def build_oracle_operator(orc, w):
    if w.kind == "synth":
        return orc.synthesize_operator(w.data["lambda"], w.data["seed"])
    if w.kind == "dense":
        return orc.DenseOperator(w.data["a"])
    if w.kind == "gram":
        return orc.GramRidgeOperator(w.data["x"])
    if w.kind == "kernel":
        return orc.KernelOperator(w.data["points"], w.data["sigma"], w.data["dense_cap"])
    if w.kind == "lowrank":
        g, lam = w.data["g"], w.data["lambda"]
        a = (g * lam) @ g.T / g.shape[1]
        return orc.DenseOperator((a + a.T) / 2)
    raise ValueError(w.kind)
