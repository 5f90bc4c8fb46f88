"""KATs of /root/reference/proj/tests/preconditioner_test.cpp."""
import numpy as np
import pytest

from support import random_psd, rel_diff, sym_eigenvalues


def basis_approx(impl, n, lam):  # preconditioner_test.cpp:13-19
    lam = np.asarray(lam, dtype=np.float64)
    return impl.make_approximation(np.eye(n)[:, : lam.size], lam, 1e-16)


def empty_approx(impl, n):  # :21-26
    return impl.make_approximation(np.zeros((n, 0)), np.zeros(0), 0.0)


def materialize(p, n):
    return np.column_stack([p.apply(e) for e in np.eye(n)])


def test_rank1_single_eigenvalue_is_identity(impl):  # :42-48
    p = impl.build_preconditioner(basis_approx(impl, 3, [3.0]), 1.0)
    assert np.array_equal(materialize(p, 3), np.eye(3))


def test_preconditioner_eigenvalues_3x3(impl):  # :50-56
    p = impl.build_preconditioner(basis_approx(impl, 3, [4.0, 2.0]), 1.0)
    eig = sym_eigenvalues(materialize(p, 3))
    assert np.allclose(eig, [5 / 3, 1, 1], rtol=1e-12, atol=0)


def test_materialized_preconditioner_equals_closed_form(impl):  # :58-71
    rng = impl.Rng(31)
    a = random_psd(impl, rng, 18)
    approx = impl.randomized_nystrom(impl.DenseOperator(a), 6, rng)
    mu = 0.37
    p = impl.build_preconditioner(approx, mu)
    u, lam = approx.u, approx.lam
    want = (u * (lam + mu)) @ u.T / (lam[-1] + mu) + (np.eye(18) - u @ u.T)
    assert np.abs(materialize(p, 18) - want).max() < 1e-12


def test_build_rejects_nonpositive_mu(impl):  # :73-78
    with pytest.raises(ValueError):
        impl.build_preconditioner(basis_approx(impl, 3, [1.0]), 0.0)
    with pytest.raises(ValueError):
        impl.build_preconditioner(basis_approx(impl, 3, [1.0]), -1.0)


def test_apply_inverse_worked_example(impl):  # :80-86  (5,3,7) -> (3,3,7)
    p = impl.build_preconditioner(basis_approx(impl, 3, [4.0, 2.0]), 1.0)
    out = p.apply_inverse(np.array([5.0, 3, 7]))
    assert np.allclose(out, [3, 3, 7], rtol=1e-14, atol=0)


def test_vectors_orthogonal_to_range_pass_through(impl):  # :88-93
    p = impl.build_preconditioner(basis_approx(impl, 3, [4.0, 2.0]), 1.0)
    r = np.array([0.0, 0, 7])
    assert np.array_equal(p.apply_inverse(r), r)
    assert np.array_equal(p.apply(r), r)


def test_apply_and_apply_inverse_agree_with_dense(impl):  # :103-124
    rng = impl.Rng(41)
    a = random_psd(impl, rng, 25)
    approx = impl.randomized_nystrom(impl.DenseOperator(a), 8, rng)
    p = impl.build_preconditioner(approx, 0.05)
    dp = materialize(p, 25)
    dpinv = np.linalg.inv(dp)
    for _ in range(10):
        v = rng.gaussian_vector(25)
        assert rel_diff(p.apply(v), dp @ v) < 1e-12
        assert rel_diff(p.apply_inverse(v), dpinv @ v) < 1e-10
        assert rel_diff(p.apply(p.apply_inverse(v)), v) < 1e-10
        assert v @ p.apply(v) >= (v @ v) * (1 - 1e-10)
    block = rng.gaussian_matrix(25, 4)
    got = p.apply_inverse(block)
    for j in range(4):
        assert rel_diff(got[:, j], p.apply_inverse(block[:, j])) < 1e-12


def test_empty_preconditioner_is_identity(impl):  # :126-134
    p = impl.build_preconditioner(empty_approx(impl, 4), 0.5)
    v = impl.Rng(51).gaussian_vector(4)
    assert np.array_equal(p.apply(v), v)
    assert np.array_equal(p.apply_inverse(v), v)


def test_constant_eigenvalues_reduce_to_identity(impl):  # :136-143
    p = impl.build_preconditioner(basis_approx(impl, 6, [2.5, 2.5, 2.5]), 0.3)
    v = impl.Rng(52).gaussian_vector(6)
    assert np.array_equal(p.apply_inverse(v), v)
    assert np.array_equal(p.apply(v), v)


# ---- preconditioner_test.cpp:186-252: woodbury_inverse_apply / sketch_and_solve
def test_woodbury_worked_example(impl):  # :187-194
    approx = impl.make_approximation(np.eye(2)[:, :1], np.array([3.0]), 0.0)
    out = impl.woodbury_inverse_apply(approx, 1.0, np.array([4.0, 2.0]))
    assert abs(out[0] - 1.0) <= 1e-14 and abs(out[1] - 2.0) <= 1e-14


def test_woodbury_empty_divides_by_mu(impl):  # :195-199
    approx = impl.make_approximation(np.zeros((2, 0)), np.zeros(0), 0.0)
    assert np.array_equal(impl.woodbury_inverse_apply(approx, 0.5, np.array([4.0, 2.0])), [8.0, 4.0])


def test_woodbury_matches_dense_inverse(impl):  # :200-210
    rng = impl.Rng(71)
    a = random_psd(impl, rng, 20)
    approx = impl.randomized_nystrom(impl.DenseOperator(a), 7, rng)
    mu = 0.2
    b = rng.gaussian_vector(20)
    want = np.linalg.solve(approx.materialize() + mu * np.eye(20), b)
    assert np.linalg.norm(impl.woodbury_inverse_apply(approx, mu, b) - want) < 1e-10 * np.linalg.norm(want)
    with pytest.raises(ValueError):
        impl.woodbury_inverse_apply(approx, 0.0, b)


def test_sketch_and_solve(impl):  # :213-252
    rng = impl.Rng(81)
    g = rng.gaussian_matrix(12, 3)
    a = g @ g.T
    a = (a + a.T) / 2
    b = rng.gaussian_vector(12)
    x = impl.sketch_and_solve(impl.DenseOperator(a), b, 0.4, 5, rng)
    want = np.linalg.solve(a + 0.4 * np.eye(12), b)
    assert np.linalg.norm(x - want) < 1e-8 * np.linalg.norm(want)
    rng = impl.Rng(82)
    for trial in range(8):
        a = random_psd(impl, rng, 30)
        b = rng.gaussian_vector(30)
        x = impl.sketch_and_solve(impl.DenseOperator(a), b, 0.5, 6, impl.Rng(1000 + trial))
        approx = impl.randomized_nystrom(impl.DenseOperator(a), 6, impl.Rng(1000 + trial))
        err = np.abs(np.linalg.eigvalsh(a - approx.materialize())).max()
        star = np.linalg.solve(a + 0.5 * np.eye(30), b)
        assert np.linalg.norm(x - star) / np.linalg.norm(star) <= err / 0.5 + 1e-12
    d = np.full(10, 1e-6)
    d[0] = 1.0
    rng = impl.Rng(83)
    b = rng.gaussian_vector(10)
    x = impl.sketch_and_solve(impl.DenseOperator(np.diag(d)), b, 1.0, 3, rng)
    star = np.linalg.solve(np.diag(d) + np.eye(10), b)
    assert np.linalg.norm(x - star) / np.linalg.norm(star) <= 1e-5
