"""Acceptance criteria c1, c2, c7, c9, c10, c12, c13, c14 of the reference
(/root/reference/proj/tests/acceptance/acceptance.cpp), same trials, same
seeds, same pass thresholds. On the CPU suite they pin the oracle; on the GPU
suite they run through the B200 library (c7, the costly one, on the GPU only).
The dense O(n^3) diagnostics they use (definitional formula, exact condition
number, eigenvalues) are numpy restatements in tests/support.py."""
import math

import numpy as np
import pytest

from support import (effective_dimension, exact_condition_number, geo_spectrum, min_eigenvalue, nystrom_definitional,
                     poly_spectrum, preconditioner_matrix, psd_from_spectrum, random_psd, recommended_sketch_size,
                     rel_diff, spectral_norm, sym_eigenvalues)


def nystrom_trials(impl):  # acceptance.cpp:57-86
    trials = []
    for t in range(50):
        seed = 1000 + t
        setup = impl.Rng(seed * 7 + 1)
        n = 20 + setup.integer(81)
        if t % 3 == 0:
            lam = np.array([10.0 ** (-4.0 * setup.uniform()) for _ in range(n)])
        elif t % 3 == 1:
            lam = poly_spectrum(n, 2.0)
        else:
            lam = geo_spectrum(n, 0.7)
            lam[n - n // 4:] = 0.0  # rank-deficient inputs
        a = psd_from_spectrum(impl, lam, setup)
        ell = 2 + setup.integer(n // 2)
        approx = impl.randomized_nystrom(impl.DenseOperator(a), ell, impl.Rng(seed))
        omega = impl.Rng(seed).gaussian_matrix(n, ell)
        trials.append((a, omega, approx))
    return trials


@pytest.fixture(scope="module")
def trials_by_impl():
    cache = {}

    def get(impl):
        key = impl.__name__
        if key not in cache:
            cache[key] = nystrom_trials(impl)
        return cache[key]
    return get


def test_c1_definitional_formula(impl, trials_by_impl):  # acceptance.cpp:88-97
    worst = 0.0
    for a, omega, approx in trials_by_impl(impl):
        err = np.linalg.norm(approx.materialize() - nystrom_definitional(a, omega)) / np.linalg.norm(a)
        worst = max(worst, err)
    assert worst <= 1e-8, f"max definitional mismatch {worst:.3e}"


def test_c2_loewner_order_and_majorisation(impl, trials_by_impl):  # acceptance.cpp:99-116
    worst_neg = worst_exc = 0.0
    for a, _, approx in trials_by_impl(impl):
        lam = sym_eigenvalues(a)
        top = lam[0]
        worst_neg = max(worst_neg, -min_eigenvalue(a - approx.materialize()) / top)
        for j in range(approx.lam.size):
            worst_exc = max(worst_exc, (approx.lam[j] - lam[j]) / top)
    assert worst_neg <= 1e-8 and worst_exc <= 1e-8, (worst_neg, worst_exc)


def run_condition_cell(impl, spectrum, mu, seed):  # acceptance.cpp:219-272 (solve = true)
    n = spectrum.size
    ell = recommended_sketch_size(spectrum, mu)
    a = np.asfortranarray(np.diag(spectrum))
    op = impl.DenseOperator(a)
    a_mu = a + mu * np.eye(n)
    a_mu_diag = spectrum + mu
    bound_iters = impl.iteration_bound(56.0, 1e-6)
    rng = impl.Rng(seed)
    envelope_ok, all_reached, worst_hit, solved = True, True, 0, 0
    for _ in range(20):
        approx = impl.randomized_nystrom(op, ell, rng)
        p = impl.build_preconditioner(approx, mu)
        kappa = exact_condition_number(preconditioner_matrix(approx, mu), a_mu)
        if kappa > 56.0:
            continue
        solved += 1
        x_star = rng.gaussian_vector(n)
        b = a_mu_diag * x_star
        run = impl.nystrom_pcg(op, b, mu, p, eta=1e-10, relative=True, max_iter=500, record_iterates=True)
        rho = (math.sqrt(kappa) - 1.0) / (math.sqrt(kappa) + 1.0)
        hit = -1
        den = math.sqrt(x_star @ (a_mu_diag * x_star))
        for t, xt in enumerate(run.iterates):
            e = xt - x_star
            delta = math.sqrt(e @ (a_mu_diag * e)) / den
            if hit < 0:
                envelope = 2.0 * rho ** t * (1.0 + 1e-9)
                if delta > max(envelope, 1e-6):
                    envelope_ok = False
                if delta <= 1e-6:
                    hit = t
        if hit < 0 or hit > bound_iters:
            all_reached = False
        else:
            worst_hit = max(worst_hit, hit)
    return envelope_ok, all_reached, worst_hit, solved


@pytest.mark.gpu
def test_c7_pcg_convergence_envelope():  # acceptance.cpp:307-323
    import paper_2110_02820_b200 as impl
    n = 1000
    cells = []
    for mu in (1e-2, 1e-4):
        cells += [(poly_spectrum(n, 1.0), mu), (poly_spectrum(n, 2.0), mu), (geo_spectrum(n, 0.9), mu)]
    seed, solved, worst = 600, 0, 0
    for spectrum, mu in cells:
        env, reached, hit, s = run_condition_cell(impl, spectrum, mu, seed)
        seed += 1
        assert env and reached, (mu, hit)
        solved += s
        worst = max(worst, hit)
    assert solved > 0 and worst <= impl.iteration_bound(56.0, 1e-6)


def test_c12_block_pcg_matches_single(impl):  # acceptance.cpp:498-527
    rng = impl.Rng(1212)
    n = 300
    a = psd_from_spectrum(impl, geo_spectrum(n, 0.85), rng)
    op = impl.DenseOperator(a)
    mu = 1e-2
    approx = impl.randomized_nystrom(op, 30, rng)
    p = impl.build_preconditioner(approx, mu)
    opt = dict(eta=1e-12, relative=True, max_iter=1000)
    b = rng.gaussian_matrix(n, 4)
    block = impl.block_nystrom_pcg(op, b, mu, p, **opt)
    worst = 0.0
    for j in range(4):
        single = impl.nystrom_pcg(op, b[:, j], mu, p, **opt)
        worst = max(worst, rel_diff(block.x[:, j], single.x))
    one = impl.block_nystrom_pcg(op, b[:, :1], mu, p, **opt)
    single0 = impl.nystrom_pcg(op, b[:, 0], mu, p, **opt)
    assert worst <= 1e-8 and rel_diff(one.x[:, 0], single0.x) <= 1e-10


def test_c14_krr_column_sampling_ratio(impl):  # acceptance.cpp:565-604
    rng = impl.Rng(1414)
    n = 1500
    centers = 2.0 * rng.gaussian_matrix(15, 3)
    points = np.empty((n, 3), order="F")
    for i in range(n):  # component index drawn before the offset (left-to-right)
        c = rng.integer(15)
        points[i, :] = centers[c] + 0.2 * rng.gaussian_vector(3)
    sigma, mu = 1.0, 1e-6
    shift = n * mu
    op = impl.KernelOperator(points, sigma)
    b = rng.gaussian_vector(n)
    out = impl.adaptive(op, rng, mode="ratio", ell0=100, ell_max=600, mu=shift, tau=0.5, sketch="column")
    p = impl.build_preconditioner(out.approximation, shift)
    opt = dict(eta=1e-6, relative=True, max_iter=500)
    pcg = impl.nystrom_pcg(op, b, shift, p, **opt)
    try:
        raw = impl.cg(impl.regularize(op, shift), b, **opt)
        cg_iters = raw.iterations if raw.converged else 500
    except impl.SolveDivergenceError:
        cg_iters = 500
    assert pcg.converged and pcg.iterations <= 60 and 4 * pcg.iterations <= cg_iters, \
        (out.ell_final, pcg.iterations, cg_iters)


def random_features(impl, x, m_rf, sigma, rng):  # bench.cpp:395-407, draws through impl's Rng
    w = rng.gaussian_matrix(x.shape[1], m_rf) / sigma
    phase = np.array([2.0 * math.pi * rng.uniform() for _ in range(m_rf)])
    return np.asfortranarray(math.sqrt(2.0 / m_rf) * np.cos(x @ w + phase[None, :]))


def test_c9_sketch_and_solve_bound_and_pcg_vs_cg(impl):  # acceptance.cpp:355-414
    n_pts, m_rf, ell, sigma = 500, 2000, 200, 1.0
    for seed in (1, 2):
        rng = impl.Rng(seed)
        centers = 2.5 * rng.gaussian_matrix(20, 3)
        x = np.empty((n_pts, 3))
        for i in range(n_pts):  # component index drawn before the offset
            c = rng.integer(20)
            x[i, :] = centers[c] + 0.2 * rng.gaussian_vector(3)
        z = random_features(impl, x, m_rf, sigma, rng)
        op = impl.GramRidgeOperator(z)
        a = z.T @ z / n_pts
        w, v = np.linalg.eigh((a + a.T) / 2)
        approx = impl.randomized_nystrom(op, ell, rng)
        err_norm = spectral_norm(a - approx.materialize())
        b = rng.gaussian_vector(m_rf)
        b = b / np.linalg.norm(b)
        prev_rel = -1.0
        for mu in (1e-2, 1e-4, 1e-6):
            x_star = v @ ((v.T @ b) / (w + mu))
            x_hat = impl.woodbury_inverse_apply(approx, mu, b)
            rel = np.linalg.norm(x_hat - x_star) / np.linalg.norm(x_star)
            assert rel > prev_rel, (seed, mu, rel, prev_rel)  # grows as mu decreases
            assert rel <= err_norm / mu * (1.0 + 1e-9), (seed, mu, rel, err_norm)
            prev_rel = rel
            pcg = impl.nystrom_pcg(op, b, mu, impl.build_preconditioner(approx, mu), eta=1e-10, max_iter=500)
            assert pcg.converged, (seed, mu, pcg.iterations)
            if mu == 1e-6:
                raw = impl.cg(impl.regularize(op, mu), b, eta=1e-10, max_iter=500)
                assert not raw.converged, (seed, raw.iterations)  # CG must fail at this scale


def test_c10_adaptive_doublings_size_and_iterations(impl):  # acceptance.cpp:416-471
    n, mu, tau, delta = 500, 1e-3, 44.0, 0.25
    lam = geo_spectrum(n, 0.7)
    op = impl.DenseOperator(np.asfortranarray(np.diag(lam)))
    a_mu_diag = lam + mu
    deff = effective_dimension(lam, delta * tau * mu / 11.0)
    ell_tilde = 2 * int(math.ceil(2.0 * deff)) + 1
    allowed_doublings = int(math.ceil(math.log2(ell_tilde / 10.0)))
    size_cap = 4 * int(math.ceil(2.0 * deff)) + 2
    iter_cap = impl.iteration_bound(1.0 + 12.0 * tau / 11.0, 1e-6)
    ok_doublings = ok_size = ok_iters = 0
    trials = 40
    rng = impl.Rng(1010)
    for _ in range(trials):
        out = impl.adaptive(op, rng, mode="error", ell0=10, ell_max=n, mu=mu, tau=tau)
        ok_doublings += out.doublings <= allowed_doublings
        ok_size += out.ell_final <= size_cap
        if out.hit_cap:
            continue
        p = impl.build_preconditioner(out.approximation, mu)
        x_star = rng.gaussian_vector(n)
        b = a_mu_diag * x_star
        run = impl.nystrom_pcg(op, b, mu, p, eta=1e-10, relative=True, max_iter=200, record_iterates=True)
        den = math.sqrt(x_star @ (a_mu_diag * x_star))
        for it, xt in enumerate(run.iterates):
            e = xt - x_star
            if math.sqrt(e @ (a_mu_diag * e)) / den <= 1e-6:  # diag_energy_error, acceptance.cpp:45-49
                ok_iters += it <= iter_cap
                break
    need = trials * 3 // 4
    assert ok_doublings >= need and ok_size >= need and ok_iters >= need, (ok_doublings, ok_size, ok_iters)


def test_c13_power_estimate_lower_bound_and_sharpness(impl):  # acceptance.cpp:529-563
    rng = impl.Rng(1313)
    violations = 0
    for _ in range(100):
        n = 20 + rng.integer(61)
        cond = 10.0 ** (1.0 + 3.0 * rng.uniform())
        a = random_psd(impl, rng, n, cond)
        ell = 1 + rng.integer(n // 2)
        q = 1 + rng.integer(8)
        approx = impl.randomized_nystrom(impl.DenseOperator(a), ell, rng)
        estimate = impl.estimate_error_power(impl.DenseOperator(a), approx, q, rng)
        exact = spectral_norm(a - approx.materialize())
        violations += estimate > exact + 1e-12 * np.linalg.norm(a)
    worst_ratio = 1.0
    for _ in range(20):
        n = 40
        lam = geo_spectrum(n, 0.45)
        ell = 3 + rng.integer(10)
        approx = impl.make_approximation(np.asfortranarray(np.eye(n)[:, :ell]), lam[:ell].copy())
        op = impl.DenseOperator(np.asfortranarray(np.diag(lam)))
        estimate = impl.estimate_error_power(op, approx, 20, rng)
        worst_ratio = min(worst_ratio, estimate / lam[ell])
    assert violations == 0 and worst_ratio >= 0.99, (violations, worst_ratio)
