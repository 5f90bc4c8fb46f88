"""KATs of /root/reference/proj/tests/nystrom_test.cpp (Gaussian sketch rows)."""
import numpy as np
import pytest

from support import (logspace_spectrum, min_eigenvalue, nystrom_definitional, random_psd,
                     sym_eigenvalues)


def test_zero_matrix_yields_exactly_zero_eigenvalues(impl):  # nystrom_test.cpp:12-20
    approx = impl.randomized_nystrom(impl.DenseOperator(np.zeros((10, 10))), 3, impl.Rng(1))
    assert approx.lam.shape == (3,)
    assert np.array_equal(approx.lam, np.zeros(3))
    assert approx.lambda_min == 0.0


def test_rank_deficient_matrix_is_reconstructed(impl):  # :22-29
    d = np.diag([1.0, 1, 0, 0])
    approx = impl.randomized_nystrom(impl.DenseOperator(d), 3, impl.Rng(2))
    assert np.linalg.norm(approx.materialize() - d) < 1e-8


def test_stable_pipeline_matches_definitional_oracle(impl):  # :31-45
    a = random_psd(impl, impl.Rng(3), 20, 1e2)
    approx = impl.randomized_nystrom(impl.DenseOperator(a), 6, impl.Rng(42))
    omega = impl.Rng(42).gaussian_matrix(20, 6)
    assert np.linalg.norm(approx.materialize() - nystrom_definitional(a, omega)) < 1e-8 * np.linalg.norm(a)


def test_out_of_range_sketch_sizes_rejected(impl):  # :47-55
    op = impl.DenseOperator(np.eye(5))
    rng = impl.Rng(4)
    with pytest.raises(ValueError):
        impl.randomized_nystrom(op, 0, rng)
    with pytest.raises(ValueError):
        impl.randomized_nystrom(op, 6, rng)
    full = impl.randomized_nystrom(op, 5, rng)
    assert np.linalg.norm(full.materialize() - np.eye(5)) < 1e-10


def test_extend_sketch_grows_without_touching_old_columns(impl):  # :136-154
    a = random_psd(impl, impl.Rng(10), 15)
    op = impl.DenseOperator(a)
    draw = impl.Rng(11)
    pair = impl.make_empty_sketch(15)
    with pytest.raises(ValueError):
        impl.extend_sketch(pair, op, 0, draw)
    pair = impl.extend_sketch(pair, op, 4, draw)
    om4, y4 = pair.arrays(15)
    pair = impl.extend_sketch(pair, op, 3, draw)
    om, y = pair.arrays(15)
    assert pair.size() == 7
    assert np.array_equal(om[:, :4], om4) and np.array_equal(y[:, :4], y4)
    assert np.abs(om.T @ om - np.eye(7)).max() < 1e-10
    for j in range(7):
        assert np.linalg.norm(y[:, j] - a @ om[:, j]) < 1e-12 * max(1.0, np.linalg.norm(y[:, j]))


def test_extending_a_sketch_replays_the_oneshot_run(impl):  # :156-171
    a = random_psd(impl, impl.Rng(12), 40, 1e2)
    op = impl.DenseOperator(a)
    grow = impl.Rng(2024)
    pair = impl.extend_sketch(impl.make_empty_sketch(40), op, 5, grow)
    pair = impl.extend_sketch(pair, op, 7, grow)
    extended = impl.nystrom_from_sketch(pair)
    oneshot = impl.randomized_nystrom(op, 12, impl.Rng(2024))
    assert np.linalg.norm(extended.materialize() - oneshot.materialize()) < 1e-8 * np.linalg.norm(a)


def test_loewner_order_and_majorization(impl):  # :223-246
    rng = impl.Rng(14)
    for _ in range(10):
        n = 20 + rng.integer(81)
        a = random_psd(impl, rng, n)
        lam = sym_eigenvalues(a)
        ell = 3 + rng.integer(n // 2)
        approx = impl.randomized_nystrom(impl.DenseOperator(a), ell, rng)
        tol = 1e-8 * lam[0]
        assert min_eigenvalue(a - approx.materialize()) > -tol
        assert np.all(approx.lam <= lam[: ell] + tol)
        assert np.abs(approx.u.T @ approx.u - np.eye(ell)).max() < 1e-10
        assert approx.shift_used > 0.0
        assert np.all(np.diff(approx.lam) <= 0)


def test_stable_pipeline_survives_sixteen_decades(impl):  # :265-282
    n, ell = 30, 10
    op = impl.synthesize_operator(logspace_spectrum(n, 0.0, -16.0), 23)
    a = op.apply_block(np.eye(n))
    approx = impl.randomized_nystrom(op, ell, impl.Rng(77))
    ahat = approx.materialize()
    assert np.all(np.isfinite(ahat))
    assert min_eigenvalue(ahat) > -1e-14
    omega = impl.Rng(77).gaussian_matrix(n, ell)
    assert np.linalg.norm(ahat - nystrom_definitional(a, omega)) < 1e-6 * np.linalg.norm(a)


# ---- column-sampling Nyström (nystrom.cpp:60-94,150-184) ----

def test_column_sampling_on_diagonal_matrices(impl):  # nystrom_test.cpp:84-103
    d = np.diag([5.0, 0, 0])
    approx = impl.column_sampling_nystrom(impl.DenseOperator(d), [0])
    assert np.abs(approx.materialize() - d).max() < 1e-12
    approx = impl.column_sampling_nystrom(impl.DenseOperator(np.eye(4)), [0, 2])
    assert np.abs(approx.materialize() - np.diag([1.0, 0, 1, 0])).max() < 1e-12
    op = impl.DenseOperator(np.eye(4))
    with pytest.raises(ValueError):
        impl.column_sampling_nystrom(op, [1, 1])
    with pytest.raises(ValueError):
        impl.column_sampling_nystrom(op, [4])


def test_column_sampling_matches_definitional_oracle(impl):  # :105-121
    rng = impl.Rng(8)
    pts = rng.gaussian_matrix(30, 3)
    op = impl.KernelOperator(pts, 1.5)
    k = op.dense()
    approx = impl.column_sampling_nystrom(op, 10, impl.Rng(1234))
    idx = impl.Rng(1234).sample_without_replacement(30, 10)
    x = np.zeros((30, 10))
    for i, j in enumerate(idx):
        x[j, i] = 1.0
    assert np.linalg.norm(approx.materialize() - nystrom_definitional(k, x)) < 1e-8 * np.linalg.norm(k)


def test_column_sampling_requires_column_access(impl):  # :123-127
    rng = impl.Rng(9)
    op = impl.GramRidgeOperator(rng.gaussian_matrix(10, 6))
    with pytest.raises(RuntimeError):
        impl.column_sampling_nystrom(op, 2, rng)


def test_extend_sketch_columns_draws_unused_indices(impl):  # :173-189
    op = impl.DenseOperator(np.eye(6))
    rng = impl.Rng(13)
    used = []
    pair = impl.extend_sketch_columns(impl.make_empty_sketch(6), op, 2, used, rng)
    assert len(used) == 2
    pair = impl.extend_sketch_columns(pair, op, 3, used, rng)
    assert len(used) == 5 and len(set(used)) == 5
    om, y = pair.arrays(6)
    for i in range(5):
        assert om[:, i].sum() == 1.0
        assert np.array_equal(y[:, i], op.column(used[i]))
    with pytest.raises(ValueError):
        impl.extend_sketch_columns(pair, op, 2, used, rng)


def test_column_sampling_draws_match_the_oracle(impl, orc):
    # the same Rng stream picks the same columns in both implementations
    op = impl.DenseOperator(np.diag(np.arange(1.0, 13.0)))
    used = []
    impl.extend_sketch_columns(impl.make_empty_sketch(12), op, 4, used, impl.Rng(21))
    ref = []
    orc.extend_sketch_columns(orc.make_empty_sketch(12), orc.DenseOperator(np.diag(np.arange(1.0, 13.0))), 4, ref,
                              orc.Rng(21))
    assert used == ref


def test_extend_sketch_leaves_its_input_unchanged(impl):
    """extend_sketch returns a new SketchPair (nystrom.cpp:36-58): extending the
    same pair twice (a branch) must not disturb either result, and an
    approximation / preconditioner built earlier is unaffected by later
    extends and refactors (value semantics of nystrom.hpp:19-48)."""
    a = random_psd(impl, impl.Rng(20), 30, 1e2)
    op = impl.DenseOperator(a)
    base = impl.extend_sketch(impl.make_empty_sketch(30), op, 4, impl.Rng(21))
    om4, y4 = base.arrays(30)
    approx4 = impl.nystrom_from_sketch(base)
    pre = impl.build_preconditioner(approx4, 0.1)
    r = impl.Rng(22).gaussian_vector(30)
    z_before = pre.apply_inverse(r)
    lam4 = approx4.lam.copy()
    longer = impl.extend_sketch(base, op, 3, impl.Rng(23))
    om7, y7 = longer.arrays(30)
    branch = impl.extend_sketch(base, op, 2, impl.Rng(24))  # appends behind `longer`'s columns
    assert base.size() == 4 and longer.size() == 7 and branch.size() == 6
    om4b, y4b = base.arrays(30)
    assert np.array_equal(om4b, om4) and np.array_equal(y4b, y4)
    om7b, y7b = longer.arrays(30)
    assert np.array_equal(om7b, om7) and np.array_equal(y7b, y7)
    om6, _ = branch.arrays(30)
    assert np.array_equal(om6[:, :4], om4)
    impl.nystrom_from_sketch(longer)
    impl.nystrom_from_sketch(branch)
    assert np.array_equal(approx4.lam, lam4)
    assert np.array_equal(pre.apply_inverse(r), z_before)
    again = impl.nystrom_from_sketch(base)
    assert np.array_equal(again.lam, lam4)
