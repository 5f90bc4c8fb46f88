"""GPU unit tests of the hand-written kernels against numpy fp64 / the oracle:
DMMA+TMA GEMM in all four operand layouts (incl. ragged edges and split-K),
Cholesky-QR orthonormalisation, thin SVD, skinny GEMVs via the operators."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def npcg():
    import paper_2110_02820_b200 as m
    return m


@pytest.mark.parametrize("transa", [False, True])
@pytest.mark.parametrize("transb", [False, True])
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 5, 3), (128, 128, 16), (130, 67, 45), (300, 129, 257),
                                   (64, 64, 5000), (513, 20, 40)])
def test_gemm_layouts(npcg, transa, transb, shape):
    m, n, k = shape
    rng = np.random.default_rng(m * 1000 + n * 10 + k)
    a = rng.standard_normal((k, m) if transa else (m, k))
    b = rng.standard_normal((n, k) if transb else (k, n))
    c = rng.standard_normal((m, n))
    want = 1.5 * ((a.T if transa else a) @ (b.T if transb else b)) - 0.5 * c
    got = npcg.gemm(a, b, transa, transb, alpha=1.5, beta=-0.5, c=c)
    scale = np.abs(a).max() * np.abs(b).max() * k + np.abs(c).max()
    assert np.abs(got - want).max() <= 1e-14 * scale


def test_gemm_is_deterministic(npcg):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((4000, 200))
    g1 = npcg.gemm(a, a, transa=True)
    g2 = npcg.gemm(a, a, transa=True)
    assert np.array_equal(g1, g2)


@pytest.mark.parametrize("m,n", [(50, 7), (2000, 100), (3000, 300)])
def test_orthonormal_columns(npcg, m, n):
    g = np.random.default_rng(m + n).standard_normal((m, n))
    q = npcg.orthonormal_columns(g)
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-13
    assert np.abs(q @ (q.T @ g) - g).max() < 1e-11 * np.abs(g).max() * np.sqrt(n)


def test_orthonormal_columns_ill_conditioned(npcg):
    # kappa ~ 1e12 forces the shifted CholeskyQR3 path
    rng = np.random.default_rng(5)
    u, _ = np.linalg.qr(rng.standard_normal((400, 40)))
    v, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    g = (u * np.logspace(0, -12, 40)) @ v.T
    q = npcg.orthonormal_columns(g)
    assert np.abs(q.T @ q - np.eye(40)).max() < 1e-12


@pytest.mark.parametrize("m,n", [(12, 5), (300, 64), (1000, 200)])
def test_thin_svd(npcg, m, n):
    b = np.random.default_rng(m).standard_normal((m, n)) * np.logspace(0, -6, n)
    u, s = npcg.thin_svd(b)
    uo, so, _ = np.linalg.svd(b, full_matrices=False)
    assert np.all(np.diff(s) <= 0)
    assert np.abs(s - so).max() < 1e-13 * so[0]
    assert np.abs(u.T @ u - np.eye(n)).max() < 1e-12
    recon = (u * s) @ (u.T @ b) / np.where(s > 0, s, 1)[None, :] if False else None
    # left singular vectors up to sign on well-separated values
    for j in range(n):
        assert abs(abs(u[:, j] @ uo[:, j]) - 1.0) < 1e-8


@pytest.mark.parametrize("k", [1, 3, 8, 9])
def test_dense_apply_blocks(npcg, k):
    rng = np.random.default_rng(k)
    g = rng.standard_normal((500, 500))
    a = (g + g.T) / 2
    op = npcg.DenseOperator(a)
    v = rng.standard_normal((500, k))
    assert np.abs(op.apply_block(v) - a @ v).max() < 1e-12 * np.abs(a @ v).max()


@pytest.mark.parametrize("k", [1, 2, 8, 12])
def test_gram_apply_blocks(npcg, k):
    rng = np.random.default_rng(10 + k)
    x = rng.standard_normal((777, 130))
    op = npcg.GramRidgeOperator(x)
    v = rng.standard_normal((130, k))
    want = x.T @ (x @ v) / 777
    assert np.abs(op.apply_block(v) - want).max() < 1e-12 * np.abs(want).max()
