"""KATs of /root/reference/proj/tests/solvers_test.cpp."""
import numpy as np
import pytest

from support import energy_norm, logspace_spectrum, random_psd, rel_diff, spectral_norm


def identity_preconditioner(impl, n, mu):  # solvers_test.cpp:13-18
    return impl.build_preconditioner(impl.make_approximation(np.zeros((n, 0)), np.zeros(0), 0.0), mu)


def direct_solve(a, mu, b):
    return np.linalg.solve(a + mu * np.eye(a.shape[0]), b)


def test_cg_identity_one_iteration(impl):  # :28-39
    b = impl.Rng(1).gaussian_vector(6)
    rep = impl.cg(impl.DenseOperator(np.eye(6)), 0.0, b)
    assert np.array_equal(rep.x, b)
    assert rep.iterations == 1 and rep.converged and rep.matvec_count == 2
    assert len(rep.residual_history) == 2 and rep.residual_history[1] == 0.0


def test_cg_three_eigenvalues(impl):  # :41-54
    d = np.array([4.0, 2, 1])
    b = impl.Rng(2).gaussian_vector(3)
    rep = impl.cg(impl.DenseOperator(np.diag(d)), 0.0, b, eta=1e-10, max_iter=50)
    assert rep.converged and rep.iterations <= 3
    assert rel_diff(rep.x, b / d) < 1e-10
    assert len(rep.residual_history) == rep.iterations + 1
    assert rep.matvec_count == rep.iterations + 1


def test_cg_zero_rhs_stops_immediately(impl):  # :56-63
    rep = impl.cg(impl.DenseOperator(np.eye(4)), 0.0, np.zeros(4))
    assert np.array_equal(rep.x, np.zeros(4))
    assert rep.iterations == 0 and rep.converged and rep.matvec_count == 1


def test_cg_honors_warm_start(impl):  # :65-74
    rng = impl.Rng(3)
    a = random_psd(impl, rng, 20)
    b = rng.gaussian_vector(20)
    star = direct_solve(a, 0.0, b)
    rep = impl.cg(impl.DenseOperator(a), 0.0, b, eta=1e-8, max_iter=100, x0=star)
    assert rep.converged and rep.iterations == 0


def test_cg_reports_breakdown_on_indefinite(impl):  # :76-90
    a = np.diag([1.0, -1.0])
    with pytest.raises(impl.SolveDivergenceError) as ei:
        impl.cg(impl.DenseOperator(a), 0.0, np.array([1.0, 1.0]))
    rep = ei.value.report
    assert rep.iterations == 1 and not rep.converged and len(rep.residual_history) >= 1


def test_pcg_exact_preconditioner_two_iterations(impl):  # :92-110
    rng = impl.Rng(4)
    g = rng.gaussian_matrix(20, 3)
    a = g @ g.T
    a = (a + a.T) / 2
    op = impl.DenseOperator(a)
    mu = 0.1
    approx = impl.randomized_nystrom(op, 3, rng)
    assert spectral_norm(a - approx.materialize()) < 1e-10
    p = impl.build_preconditioner(approx, mu)
    b = rng.gaussian_vector(20)
    rep = impl.nystrom_pcg(op, b, mu, p, eta=1e-9, max_iter=50, relative=True)
    assert rep.converged and rep.iterations <= 2


def test_pcg_recovers_known_solution(impl):  # :112-127
    rng = impl.Rng(5)
    a = random_psd(impl, rng, 50)
    op = impl.DenseOperator(a)
    mu = 0.01
    star = rng.gaussian_vector(50)
    b = op.matvec(star) + mu * star
    approx = impl.randomized_nystrom(op, 10, rng)
    p = impl.build_preconditioner(approx, mu)
    rep = impl.nystrom_pcg(op, b, mu, p, eta=1e-10, max_iter=500, relative=True)
    assert rep.converged and rel_diff(rep.x, star) < 1e-8
    assert abs(rep.eta_used - 1e-10 * np.linalg.norm(b)) <= 1e-14 * rep.eta_used


def test_pcg_empty_preconditioner_matches_cg_bitwise(impl):  # :129-147
    rng = impl.Rng(6)
    a = random_psd(impl, rng, 30)
    op = impl.DenseOperator(a)
    mu = 0.1
    b = rng.gaussian_vector(30)
    plain = impl.cg(op, mu, b, eta=1e-9, max_iter=200)
    pre = impl.nystrom_pcg(op, b, mu, identity_preconditioner(impl, 30, mu), eta=1e-9, max_iter=200)
    assert np.array_equal(plain.x, pre.x)
    assert plain.iterations == pre.iterations
    assert np.array_equal(plain.residual_history, pre.residual_history)


def test_pcg_validates_preconditioner_mu(impl):  # :149-157
    rng = impl.Rng(7)
    a = random_psd(impl, rng, 10)
    op = impl.DenseOperator(a)
    p = impl.build_preconditioner(impl.randomized_nystrom(op, 3, rng), 0.1)
    with pytest.raises(ValueError):
        impl.nystrom_pcg(op, rng.gaussian_vector(10), 0.2, p)


def test_energy_norm_error_is_monotone(impl):  # :159-198 (monotonicity part)
    rng = impl.Rng(8)
    a = random_psd(impl, rng, 60, 1e3)
    op = impl.DenseOperator(a)
    mu = 1e-3
    a_mu = a + mu * np.eye(60)
    b = rng.gaussian_vector(60)
    star = direct_solve(a, mu, b)
    denom = energy_norm(a_mu, star)
    p = impl.build_preconditioner(impl.randomized_nystrom(op, 12, rng), mu)
    rep = impl.nystrom_pcg(op, b, mu, p, eta=1e-7, max_iter=500, relative=True, record_iterates=True)
    cg_rep = impl.cg(op, mu, b, eta=1e-7, max_iter=500, relative=True)
    assert rep.iterates.shape[0] == rep.iterations + 1
    prev = np.inf
    for it in rep.iterates:
        err = energy_norm(a_mu, it - star) / denom
        assert err <= prev * (1 + 1e-9) + 1e-15
        prev = err
    assert rep.iterations < cg_rep.iterations


def test_block_pcg_one_column_reduces_to_pcg(impl):  # :232-248
    rng = impl.Rng(10)
    a = random_psd(impl, rng, 25)
    op = impl.DenseOperator(a)
    mu = 0.05
    p = impl.build_preconditioner(impl.randomized_nystrom(op, 6, rng), mu)
    b = rng.gaussian_vector(25)
    single = impl.nystrom_pcg(op, b, mu, p, eta=1e-11, max_iter=300)
    block = impl.block_nystrom_pcg(op, b.reshape(-1, 1), mu, p, eta=1e-11, max_iter=300)
    assert block.converged[0] and not block.deflated
    assert np.linalg.norm(block.x[:, 0] - single.x) < 1e-10 * np.linalg.norm(single.x)


def test_block_pcg_deflates_duplicate_rhs(impl):  # :250-266
    rng = impl.Rng(11)
    a = random_psd(impl, rng, 20)
    op = impl.DenseOperator(a)
    b = np.empty((20, 2), order="F")
    b[:, 0] = rng.gaussian_vector(20)
    b[:, 1] = b[:, 0]
    rep = impl.block_nystrom_pcg(op, b, 0.1, identity_preconditioner(impl, 20, 0.1))
    assert rep.deflated == [1] and rep.converged == [True, True]
    assert np.linalg.norm(rep.x[:, 0] - rep.x[:, 1]) < 1e-12 * np.linalg.norm(rep.x[:, 0])


def test_block_pcg_matches_independent_solves(impl):  # :268-290
    op = impl.synthesize_operator(logspace_spectrum(200, 0.0, -4.0), 33)
    mu = 1e-3
    rng = impl.Rng(12)
    p = impl.build_preconditioner(impl.randomized_nystrom(op, 30, rng), mu)
    b = rng.gaussian_matrix(200, 4)
    block = impl.block_nystrom_pcg(op, b, mu, p, eta=1e-11, max_iter=400, relative=True)
    max_single = 0
    for j in range(4):
        assert block.converged[j]
        single = impl.nystrom_pcg(op, b[:, j], mu, p, eta=1e-11, max_iter=400, relative=True)
        max_single = max(max_single, single.iterations)
        assert np.linalg.norm(block.x[:, j] - single.x) < 1e-8 * np.linalg.norm(single.x)
    assert block.iterations <= max_single + 1
    assert block.fallback_count == 0


def test_block_pcg_zero_block(impl):  # :292-301
    rep = impl.block_nystrom_pcg(impl.DenseOperator(np.eye(8)), np.zeros((8, 3)), 1.0,
                                 identity_preconditioner(impl, 8, 1.0))
    assert np.array_equal(rep.x, np.zeros((8, 3)))
    assert rep.iterations == 0 and len(rep.deflated) == 3 and all(rep.converged)


def test_iteration_bound(impl):  # :303-320
    assert impl.iteration_bound(1.0, 1e-6) == 1
    assert impl.iteration_bound(56.0, 1e-2) == 20
    assert impl.iteration_bound(56.0, 1e-6) == 54
    for kappa, eps in ((10.0, 1e-4), (400.0, 1e-8)):
        r = np.sqrt(kappa)
        assert impl.iteration_bound(kappa, eps) == int(np.ceil(np.log(2 / eps) / np.log((r + 1) / (r - 1))))
    for bad in ((0.5, 1e-2), (2.0, 0.0), (2.0, 1.0)):
        with pytest.raises(ValueError):
            impl.iteration_bound(*bad)
