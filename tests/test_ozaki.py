"""INT8 tcgen05 GEMM and the FP64 GEMM emulated on it by digit-plane splitting
(csrc/ozaki.cu). The emulation replaces the FP64 DMMA GEMM in the sketch
Y = A Omega of large stored operators (nystrom.cpp:56 via operators.cpp:76-78).
Its error bound: every entry of row i of A (column j of B) is represented to
2^-55 of that row's (column's) largest magnitude, so
    |C - AB|_ij <= c eps (max_k|a_ik| sum_k|b_kj| + sum_k|a_ik| max_k|b_kj|),
which is the FP64 GEMM bound eps |A||B| when a row's entries are of one
magnitude (measured ratio to DMMA's error ~1-4 on Gaussian data)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def npcg():
    import paper_2110_02820_b200 as m
    return m

EPS = np.finfo(np.float64).eps


@pytest.mark.parametrize("m,n,kp", [(128, 256, 128), (300, 520, 384), (1000, 77, 1024), (129, 257, 2048)])
def test_int8_gemm_exact(npcg, m, n, kp):
    rng = np.random.default_rng(m + n + kp)
    a8 = rng.integers(-128, 128, size=(m, kp), dtype=np.int8)
    b8 = rng.integers(-128, 128, size=(n, kp), dtype=np.int8)
    ref = a8.astype(np.int64) @ b8.astype(np.int64).T
    assert np.array_equal(npcg.gemm_i8(a8, b8), ref)


def scheme_bound(a, b):
    """max_k|a_ik| sum_k|b_kj| + sum_k|a_ik| max_k|b_kj| for a (K x M), b (K x N)."""
    aa, bb = np.abs(a), np.abs(b)
    return np.outer(aa.max(axis=0), bb.sum(axis=0)) + np.outer(aa.sum(axis=0), bb.max(axis=0))


@pytest.mark.parametrize("m,n,k,spread", [(200, 300, 500, 0), (513, 77, 1000, 6), (1000, 260, 3000, 30),
                                          (256, 192, 70000, 2)])  # K > one int32-safe chunk (65408)
def test_ozaki_gemm_fp64_accuracy(npcg, m, n, k, spread):
    rng = np.random.default_rng(k + spread)
    a = rng.standard_normal((k, m)) * np.exp(rng.uniform(-spread, spread, (k, m)))
    b = rng.standard_normal((k, n)) * np.exp(rng.uniform(-spread, spread, (k, n)))
    ref = a.T @ b
    got = npcg.gemm_ozaki(a, b)
    assert np.max(np.abs(got - ref) / scheme_bound(a, b)) <= 4 * EPS
    if spread == 0:  # one magnitude per row: within a small factor of the FP64 GEMM bound
        assert np.max(np.abs(got - ref) / (np.abs(a.T) @ np.abs(b))) <= 16 * EPS
    assert np.array_equal(got, npcg.gemm_ozaki(a, b))  # deterministic


@pytest.mark.parametrize("m,n,k", [(300, 260, 500), (77, 513, 2000), (1000, 300, 70000)])
def test_ozaki_gemm_m_major_operand(npcg, m, n, k):
    """A stored M x K (rows of A strided): the transposing splitter."""
    rng = np.random.default_rng(m * k)
    a = rng.standard_normal((m, k)) * np.exp(rng.uniform(-3, 3, (m, 1)))
    b = rng.standard_normal((k, n))
    ref = a @ b
    got = npcg.gemm_ozaki(a, b, transa=False)
    assert np.max(np.abs(got - ref) / scheme_bound(a.T, b)) <= 4 * EPS
    assert np.array_equal(got, npcg.gemm_ozaki(np.ascontiguousarray(a).copy(order="F"), b, transa=False))


@pytest.mark.parametrize("m,n,k", [(1000, 1000, 50000), (3000, 520, 1000)])
def test_ozaki_gemm_factorisation_shapes(npcg, m, n, k):
    """The factorisation's shapes: a Gram (few output tiles: K split into
    parallel chunks) and Y L^-T with an N-major B (transposing splits of both)."""
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((k, m)) if m == n else rng.standard_normal((m, k))
    b = rng.standard_normal((k, n)) if m == n else rng.standard_normal((n, k))
    transa, transb = (True, False) if m == n else (False, True)
    ref = (a.T if transa else a) @ (b.T if transb else b)
    got = npcg.gemm_ozaki(a, b, transa=transa, transb=transb)
    aa = a if transa else a.T
    bb = b.T if transb else b
    assert np.max(np.abs(got - ref) / scheme_bound(aa, bb)) <= 4 * EPS


def test_ozaki_gemm_zero_and_extreme_rows(npcg):
    rng = np.random.default_rng(3)
    k, m, n = 640, 300, 260
    a = rng.standard_normal((k, m))
    a[:, 7] = 0.0                 # zero row of A
    a[:, 11] *= 1e-300            # tiny row (exponent near the subnormal range)
    a[:, 13] *= 1e300             # huge row
    a[5, 17] = 1e-310             # a subnormal entry
    b = rng.standard_normal((k, n))
    b[:, 3] = 0.0
    ref = a.T @ b
    got = npcg.gemm_ozaki(a, b)
    bound = scheme_bound(a, b)
    ok = bound > 0
    assert np.all(got[~ok] == 0.0)
    assert np.max(np.abs(got[ok] - ref[ok]) / bound[ok]) <= 4 * EPS


def test_dense_sketch_uses_int8_path_and_matches_dmma(npcg):
    """A stored symmetric operator's sketch block (k >= 192, n >= 4096) runs on
    the emulated GEMM: it agrees with the DMMA GEMM to the FP64 error bound."""
    rng = np.random.default_rng(9)
    n, k = 4500, 200
    g = rng.standard_normal((n, 64))
    a = g @ g.T / 64.0 + np.eye(n)
    a = 0.5 * (a + a.T)
    v = rng.standard_normal((n, k))
    op = npcg.DenseOperator(a)
    got = op.apply_block(v)
    dm = npcg.gemm(a, v)
    bound = np.abs(a) @ np.abs(v)
    assert np.max(np.abs(got - dm) / bound) <= 16 * EPS


def test_matrix_free_kernel_sketch_block_int8(npcg, monkeypatch):
    """Matrix-free RBF kernel, a sketch-width block (k = 256) over several
    column blocks of K: both symmetric products (K[r0:n,R]^T V and its mirror
    K[r0+rb:n,R] V_R) run on the emulated GEMM with V split once. Checked on
    sampled rows against numpy FP64 (operators.cpp:166-177's entry formula)."""
    monkeypatch.setenv("NPCG_KBLOCK_BYTES", str(1 << 30))  # 1 GB blocks: R = 3328 columns, 12 blocks at n = 40000
    rng = np.random.default_rng(21)
    n, d, k, sigma = 40000, 32, 256, 0.5
    pts = rng.random((n, d))
    v = rng.standard_normal((n, k))
    op = npcg.KernelOperator(pts, sigma, dense_cap=1)
    y = op.apply_block(v)
    rows = rng.choice(n, 24, replace=False)
    sq = ((pts[rows, None, :] - pts[None, :, :]) ** 2).sum(axis=2)
    kr = np.exp(-sq / (2 * sigma * sigma))
    kr[np.arange(len(rows)), rows] = 1.0
    ref = kr @ v
    bound = np.abs(kr) @ np.abs(v) + np.outer(kr.sum(axis=1), np.abs(v).max(axis=0)) + np.abs(v).sum(axis=0)[None, :]
    assert np.max(np.abs(y[rows] - ref) / bound) <= 16 * EPS
