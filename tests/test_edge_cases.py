"""Edge cases of the B200 path against the CPU oracle: ragged sizes (not
multiples of the 16/32/80/128 tiles), n = 1, l = n, wide designs, zero and
non-finite inputs, mixed per-column convergence, max_iter, the persistent vs
the multi-kernel PCG drivers, and the matrix-free kernel paths (fused k <= 2,
row blocks k > 2) at odd d and n. Same tolerances as the config parity."""
import os
import subprocess
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_parity_configs import X_RTOL, compare_approx, compare_solve  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def npcg():
    import paper_2110_02820_b200 as m
    return m


def psd(rng, n, decay=2.0):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (q * (np.arange(1, n + 1) ** -decay)) @ q.T
    return 0.5 * (a + a.T)


def both(npcg, orc, a):
    return npcg.DenseOperator(a), orc.DenseOperator(a)


@pytest.mark.parametrize("n,ell", [(37, 13), (129, 81), (1, 1), (16, 16), (300, 300)])
def test_ragged_and_extreme_sketch_sizes(npcg, orc, n, ell):
    rng = np.random.default_rng(n + ell)
    a = psd(rng, n)
    op, oop = both(npcg, orc, a)
    omega = npcg.Rng(7).gaussian_matrix(n, ell)
    ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, omega))
    ao = orc.nystrom_from_sketch(orc.extend_sketch_with(orc.make_empty_sketch(n), oop, omega))
    compare_approx(ap, ao)
    b = rng.standard_normal(n)
    mu = 1e-4
    compare_solve(npcg.nystrom_pcg(op, b, mu, npcg.build_preconditioner(ap, mu), eta=1e-10, relative=True),
                  orc.nystrom_pcg(oop, b, mu, orc.build_preconditioner(ao, mu), eta=1e-10, relative=True))


def test_wide_gram_design(npcg, orc):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((50, 83))  # m < n: A is rank deficient
    op, oop = npcg.GramRidgeOperator(x), orc.GramRidgeOperator(x)
    v = rng.standard_normal(83)
    assert np.allclose(op.matvec(v), oop.matvec(v), rtol=1e-13, atol=1e-14)
    omega = npcg.Rng(2).gaussian_matrix(83, 20)
    ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, omega))
    ao = orc.nystrom_from_sketch(orc.extend_sketch_with(orc.make_empty_sketch(83), oop, omega))
    compare_approx(ap, ao)


def test_non_finite_inputs_are_rejected(npcg):
    a = np.eye(4)
    op = npcg.DenseOperator(a)
    with pytest.raises(ValueError):
        op.matvec(np.array([1.0, np.nan, 0.0, 0.0]))
    x = np.ones((5, 3))
    x[2, 1] = np.inf
    with pytest.raises(ValueError):
        npcg.GramRidgeOperator(x)
    with pytest.raises(npcg.SolveDivergenceError):  # solvers.cpp: non-finite initial residual
        npcg.nystrom_pcg(op, np.array([1.0, 2.0, np.inf, 0.0]), 1.0, None)


def test_mixed_columns_zero_rhs_and_max_iter(npcg, orc):
    rng = np.random.default_rng(11)
    n = 200
    a = psd(rng, n, 1.0)
    op, oop = both(npcg, orc, a)
    B = rng.standard_normal((n, 3))
    B[:, 1] = 0.0  # converges at iteration 0
    reps = npcg.nystrom_pcg(op, B, 1e-1, None, eta=1e-10, relative=False)  # well conditioned: counts are robust
    for j in (0, 2):
        compare_solve(reps[j], orc.nystrom_pcg(oop, B[:, j], 1e-1, None, eta=1e-10, relative=False))
    assert reps[1].iterations == 0 and reps[1].converged and np.array_equal(reps[1].x, np.zeros(n))
    capped = npcg.nystrom_pcg(op, B[:, 0], 1e-6, None, eta=1e-14, max_iter=3, relative=True)
    ocapped = orc.nystrom_pcg(oop, B[:, 0], 1e-6, None, eta=1e-14, max_iter=3, relative=True)
    assert capped.iterations == ocapped.iterations == 3 and not capped.converged
    assert np.linalg.norm(capped.x - ocapped.x) <= X_RTOL * np.linalg.norm(ocapped.x)


_DRIVER_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2110_02820_b200 as npcg
rng = np.random.default_rng(5)
x = rng.standard_normal((3000, 700)) * (np.arange(1, 701) ** -0.5)
q, _ = np.linalg.qr(rng.standard_normal((900, 900)))
a = (q * (np.arange(1, 901) ** -1.5)) @ q.T
a = 0.5 * (a + a.T)
out = {}
for name, op, n in (("gram", npcg.GramRidgeOperator(x), 700), ("dense", npcg.DenseOperator(a), 900)):
    omega = npcg.Rng(3).gaussian_matrix(n, 60)
    ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, omega))
    b = rng.standard_normal((n, 2)) if name == "dense" else rng.standard_normal(n)
    r = npcg.nystrom_pcg(op, b, 1e-3, npcg.build_preconditioner(ap, 1e-3), eta=1e-10, relative=True)
    r = r if isinstance(r, list) else [r]
    out[name] = [(rr.iterations, rr.x) for rr in r]
np.save(sys.argv[2], np.array([out], dtype=object), allow_pickle=True)
"""


def test_persistent_and_multikernel_pcg_agree(tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("persistent", "classic"):
        env = dict(os.environ)
        if mode == "classic":
            env["NPCG_PCG"] = "classic"
        f = tmp_path / f"{mode}.npy"
        r = subprocess.run([sys.executable, "-c", _DRIVER_SCRIPT, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        res[mode] = np.load(f, allow_pickle=True)[0]
    for name in ("gram", "dense"):
        for (ip, xp), (ic, xc) in zip(res["persistent"][name], res["classic"][name]):
            assert abs(ip - ic) <= 1
            assert np.linalg.norm(xp - xc) <= 1e-10 * np.linalg.norm(xc)


_SYM_DRIVER = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2110_02820_b200 as npcg
rng = np.random.default_rng(11)
n = 9001  # several row blocks of the symmetric persistent path (4096 / 2048 rows), ragged last block
g = rng.standard_normal((n, 300))
a = (g * np.exp(-np.arange(300) / 40.0)) @ g.T / 300.0
a = 0.5 * (a + a.T)
op = npcg.DenseOperator(a)
omega = npcg.Rng(7).gaussian_matrix(n, 200)
ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, omega))
out = {}
for s in (1, 2, 3, 4):
    b = rng.standard_normal((n, s)) if s > 1 else rng.standard_normal(n)
    r = npcg.nystrom_pcg(op, b, 1e-3, npcg.build_preconditioner(ap, 1e-3), eta=1e-10, relative=True)
    r = r if isinstance(r, list) else [r]
    out[s] = [(rr.iterations, rr.x) for rr in r]
np.save(sys.argv[2], np.array([out], dtype=object), allow_pickle=True)
"""


@pytest.mark.gpu
def test_symmetric_dense_pcg_matches_multikernel(tmp_path):
    """The persistent dense PCG reads only the block-upper part of A (row axpy
    + mirrored column dots); it must agree with the multi-kernel loop, which
    reads all of A (coldot), for 1-4 right-hand sides over several row blocks."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("persistent", "classic"):
        env = dict(os.environ)
        if mode == "classic":
            env["NPCG_PCG"] = "classic"
        f = tmp_path / f"{mode}.npy"
        r = subprocess.run([sys.executable, "-c", _SYM_DRIVER, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stderr
        res[mode] = np.load(f, allow_pickle=True)[0]
    for s in (1, 2, 3, 4):
        for (ip, xp), (ic, xc) in zip(res["persistent"][s], res["classic"][s]):
            assert ip > 5 and abs(ip - ic) <= 1, (s, ip, ic)
            assert np.linalg.norm(xp - xc) <= 1e-9 * np.linalg.norm(xc), s


@pytest.mark.parametrize("n,d", [(1300, 3), (700, 7), (257, 32), (5000, 32), (4099, 17)])
def test_matrix_free_kernel_paths(npcg, n, d):
    """Fused symmetric (k <= 2; n = 5000 / 4099 give several block pairs per
    CTA and row-block changes inside a CTA), row-block (k > 2) and column paths
    against the stored kernel; the fused product is deterministic."""
    rng = np.random.default_rng(n + d)
    pts = rng.random((n, d))
    free = npcg.KernelOperator(pts, 0.6, dense_cap=1)       # matrix-free
    stored = npcg.KernelOperator(pts, 0.6, dense_cap=n)     # stored
    for k in (1, 2, 5, 12):  # fused (k <= 2) and row-block (k > 2) paths
        V = rng.standard_normal((n, k))
        got, want = free.apply_block(V), stored.apply_block(V)
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max(), k
        if k <= 2:
            assert np.array_equal(free.apply_block(V), got)
    j = n // 3
    assert np.allclose(free.column(j), stored.column(j), rtol=1e-13, atol=1e-15)


def test_streamed_gram_upload(npcg, orc, monkeypatch):
    """npcg_op_gram_create_streamed: the block-by-block sketch as X lands
    matches the synchronous operator and the oracle; the non-finite check
    moves from the constructor to the first product (same message)."""
    monkeypatch.setenv("NPCG_STREAM_ROWS", "208")  # several row blocks, a ragged last one
    rng = np.random.default_rng(17)
    x = rng.standard_normal((1000, 90)) * (np.arange(1, 91) ** -0.5)
    sync, streamed, oop = npcg.GramRidgeOperator(x), npcg.GramRidgeOperator(x, streamed=True), \
        orc.GramRidgeOperator(x)
    omega = npcg.Rng(4).gaussian_matrix(90, 24)
    ap = npcg.nystrom_from_sketch(npcg.extend_sketch_with(npcg.make_empty_sketch(streamed), streamed, omega))
    ao = orc.nystrom_from_sketch(orc.extend_sketch_with(orc.make_empty_sketch(90), oop, omega))
    compare_approx(ap, ao)
    v = rng.standard_normal(90)
    assert np.array_equal(streamed.matvec(v), sync.matvec(v))
    b = rng.standard_normal(90)
    compare_solve(npcg.nystrom_pcg(streamed, b, 1e-3, npcg.build_preconditioner(ap, 1e-3), eta=1e-10, relative=True),
                  orc.nystrom_pcg(oop, b, 1e-3, orc.build_preconditioner(ao, 1e-3), eta=1e-10, relative=True))
    x[555, 7] = np.nan
    bad = npcg.GramRidgeOperator(x, streamed=True)
    with pytest.raises(ValueError, match="non-finite"):
        bad.apply_block(rng.standard_normal((90, 24)))
    with pytest.raises(ValueError, match="non-finite"):
        bad.matvec(v)
