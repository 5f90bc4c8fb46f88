"""KATs of /root/reference/proj/tests/operators_test.cpp (oracle: CPU suite;
B200 product: GPU suite)."""
import numpy as np
import pytest

from support import poly_spectrum, random_psd, rel_diff, min_eigenvalue, sym_eigenvalues


def check_dense_agreement(impl, op, seed):  # operators_test.cpp:28-40
    n = op.dim()
    m = op.apply_block(np.eye(n))
    rng = impl.Rng(seed)
    for _ in range(20):
        v = rng.gaussian_vector(n)
        assert rel_diff(op.matvec(v), m @ v) < 1e-12
    probe = rng.gaussian_matrix(n, 5)
    assert rel_diff(op.apply_block(probe), m @ probe) < 1e-12


def test_identity_operator_returns_its_input(impl):  # :44-48
    op = impl.DenseOperator(np.eye(3))
    assert np.array_equal(op.matvec(np.array([1.0, 2, 3])), [1, 2, 3])
    assert op.dim() == 3


def test_zero_operator(impl):  # :50-53
    op = impl.DenseOperator(np.zeros((2, 2)))
    assert np.array_equal(op.matvec(np.array([5.0, -1])), [0, 0])


def test_dense_matvec_2x2(impl):  # :55-62
    op = impl.DenseOperator(np.array([[2.0, 1], [1, 2]]))
    assert np.array_equal(op.matvec(np.array([1.0, 0])), [2, 1])
    assert np.array_equal(op.column(1), [1, 2])


def test_matvec_validates_dimension_and_finiteness(impl):  # :64-70
    op = impl.DenseOperator(np.eye(3))
    with pytest.raises(ValueError):
        op.matvec(np.array([1.0, 2]))
    with pytest.raises(ValueError):
        op.matvec(np.array([1.0, 2, np.nan]))
    with pytest.raises(ValueError):
        op.column(3)


def test_dense_operator_rejects_nonsquare_and_asymmetric(impl):  # :72-77
    with pytest.raises(ValueError):
        impl.DenseOperator(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        impl.DenseOperator(np.array([[0.0, 1], [-1, 0]]))


def test_gram_ridge(impl):  # :111-131
    op = impl.GramRidgeOperator(np.eye(2))
    assert np.array_equal(op.matvec(np.array([2.0, 4])), [1, 2])
    op = impl.GramRidgeOperator(np.diag([1.0, 2.0]))
    assert np.array_equal(op.matvec(np.array([1.0, 1])), [0.5, 2.0])
    rng = impl.Rng(9)
    g = rng.gaussian_matrix(6, 3)
    op = impl.GramRidgeOperator(g)
    v = rng.gaussian_vector(3)
    assert rel_diff(op.matvec(v), (g.T @ g / 6.0) @ v) < 1e-12
    with pytest.raises(ValueError):
        impl.GramRidgeOperator(np.zeros((0, 0)))


def test_gram_eigenvalues_are_squared_singular_values_over_rows(impl):  # :133-141
    g = impl.Rng(13).gaussian_matrix(20, 8)
    op = impl.GramRidgeOperator(g)
    eig = sym_eigenvalues(op.apply_block(np.eye(8)))
    want = np.linalg.svd(g, compute_uv=False) ** 2 / 20.0
    assert np.abs(eig - want).max() < 1e-12 * want[0]


def test_gaussian_kernel_entries(impl):  # :143-170
    pts = np.array([[1.0, -2.0, 0.5], [1.0, -2.0, 0.5]])
    k = impl.KernelOperator(pts, 1.0).apply_block(np.eye(2))
    assert np.array_equal(k, np.ones((2, 2)))
    k = impl.KernelOperator(np.array([[0.0], [2.0]]), 1.0).apply_block(np.eye(2))
    assert abs(k[0, 1] - np.exp(-2.0)) <= 1e-15 * np.exp(-2.0)
    assert k[1, 0] == k[0, 1] and k[0, 0] == 1.0 and k[1, 1] == 1.0
    pts = impl.Rng(3).gaussian_matrix(40, 4)
    k = impl.KernelOperator(pts, 1.5).apply_block(np.eye(40))
    assert np.all(np.diag(k) == 1.0)
    with pytest.raises(ValueError):
        impl.KernelOperator(np.zeros((2, 1)), 0.0)


def test_gaussian_kernel_is_psd(impl):  # :172-178
    pts = impl.Rng(19).gaussian_matrix(120, 5)
    k = impl.KernelOperator(pts, 2.0).apply_block(np.eye(120))
    assert min_eigenvalue(k) > -1e-10


def test_blockwise_kernel_matches_dense(impl):  # :180-193
    rng = impl.Rng(23)
    pts = rng.gaussian_matrix(35, 3)
    dense_op = impl.KernelOperator(pts, 1.2)
    block_op = impl.KernelOperator(pts, 1.2, dense_cap=4)
    v = rng.gaussian_vector(35)
    assert rel_diff(block_op.matvec(v), dense_op.matvec(v)) < 1e-12
    for j in (0, 17, 34):
        assert rel_diff(block_op.column(j), dense_op.column(j)) < 1e-14


def test_synthesize_operator(impl):  # :203-225
    op = impl.synthesize_operator(np.ones(12), 7)
    v = impl.Rng(1).gaussian_vector(12)
    assert rel_diff(op.matvec(v), v) < 1e-12
    op = impl.synthesize_operator(np.array([4.0, 2, 1]), 11)
    eig = sym_eigenvalues(op.apply_block(np.eye(3)))
    assert np.abs(eig - [4, 2, 1]).max() < 1e-10
    a = impl.synthesize_operator(np.array([3.0, 1, 0.5]), 99).apply_block(np.eye(3))
    b = impl.synthesize_operator(np.array([3.0, 1, 0.5]), 99).apply_block(np.eye(3))
    c = impl.synthesize_operator(np.array([3.0, 1, 0.5]), 100).apply_block(np.eye(3))
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    with pytest.raises(ValueError):
        impl.synthesize_operator(np.array([1.0, 2.0]), 1)


def test_every_operator_kind_agrees_with_its_materialized_copy(impl):  # :227-241
    rng = impl.Rng(77)
    a = random_psd(impl, rng, 15)
    check_dense_agreement(impl, impl.DenseOperator(a), 101)
    check_dense_agreement(impl, impl.GramRidgeOperator(rng.gaussian_matrix(20, 9)), 103)
    check_dense_agreement(impl, impl.KernelOperator(rng.gaussian_matrix(25, 4), 1.1), 104)
    check_dense_agreement(impl, impl.KernelOperator(rng.gaussian_matrix(25, 4), 1.1, dense_cap=4), 106)
    check_dense_agreement(impl, impl.synthesize_operator(poly_spectrum(10, 1.0), 5), 105)
