"""KATs of /root/reference/proj/tests/adaptive_test.cpp (strategy 1 on the hot
path; strategies 2/3 share the doubling loop)."""
import numpy as np
import pytest

from support import geo_spectrum, poly_spectrum, random_psd, spectral_norm, sym_eigenvalues


def test_error_estimate_vanishes_when_exact(impl):  # adaptive_test.cpp:25-36
    rng = impl.Rng(1)
    g = rng.gaussian_matrix(15, 3)
    a = g @ g.T
    a = (a + a.T) / 2
    op = impl.DenseOperator(a)
    approx = impl.randomized_nystrom(op, 3, rng)
    est = impl.estimate_error_power(op, approx, 5, rng)
    assert abs(est) <= 1e-10 * sym_eigenvalues(a)[0]


def test_power_method_reaches_top_eigenvalue(impl):  # :38-46
    op = impl.DenseOperator(np.diag([3.0, 1.0]))
    empty = impl.make_approximation(np.zeros((2, 0)), np.zeros(0), 0.0)
    est = impl.estimate_error_power(op, empty, 20, impl.Rng(2))
    assert 3.0 * (1 - 1e-6) <= est <= 3.0


def test_power_estimate_never_exceeds_true_error(impl):  # :48-60 (25 of the 100 trials)
    rng = impl.Rng(3)
    for _ in range(25):
        n = 10 + rng.integer(51)
        a = random_psd(impl, rng, n)
        ell = 1 + rng.integer(n // 2)
        approx = impl.randomized_nystrom(impl.DenseOperator(a), ell, rng)
        err = spectral_norm(a - approx.materialize())
        q = 1 + rng.integer(8)
        est = impl.estimate_error_power(impl.DenseOperator(a), approx, q, rng)
        assert est <= err + 1e-12 * sym_eigenvalues(a)[0]


def test_adaptive_stops_immediately_on_tiny_tail(impl):  # :62-78
    d = np.full(100, 1e-12)
    d[0] = 1.0
    out = impl.adaptive(impl.DenseOperator(np.diag(d)), impl.Rng(4), mode="error", ell0=10,
                        ell_max=100, mu=0.05, tau=10.0)
    assert out.doublings == 0 and not out.hit_cap and out.ell_final == 10
    assert out.error_estimate is not None and out.error_estimate <= 0.5
    assert out.approximation.lambda_min <= 0.5 / 11


def test_flat_spectrum_forces_the_cap(impl):  # :80-91
    out = impl.adaptive(impl.DenseOperator(np.eye(100)), impl.Rng(5), mode="error", ell0=4,
                        ell_max=16, mu=0.05, tau=10.0)
    assert out.hit_cap and out.ell_final == 16 and out.doublings == 2
    assert out.error_estimate > 0.5


def test_strategy1_meets_its_tolerance(impl):  # :93-107
    op = impl.synthesize_operator(geo_spectrum(100, 0.7), 17)
    out = impl.adaptive(op, impl.Rng(6), mode="error", ell0=5, ell_max=100, mu=1e-3, tau=30.0)
    assert not out.hit_cap
    assert out.error_estimate <= 30e-3
    assert out.approximation.lambda_min <= 30e-3 / 11
    want = (out.approximation.lambda_min + 1e-3 + out.error_estimate) / 1e-3
    assert out.posterior_condition_estimate == pytest.approx(want)


def test_ratio_strategy(impl):  # :124-147
    op = impl.synthesize_operator(poly_spectrum(50, 2.0), 19)
    out = impl.adaptive(op, impl.Rng(8), mode="ratio", ell0=10, ell_max=50, mu=1e-2, tau=10.0)
    assert out.doublings == 0 and not out.hit_cap and out.error_estimate is None
    out = impl.adaptive(impl.DenseOperator(np.eye(100)), impl.Rng(9), mode="ratio", ell0=4,
                        ell_max=16, mu=1e-6, tau=10.0)
    assert out.hit_cap and out.ell_final == 16


def test_identical_seeds_reproduce_bitwise(impl):  # :164-178
    op = impl.synthesize_operator(geo_spectrum(80, 0.8), 20)
    a = impl.adaptive(op, impl.Rng(11), mode="error", ell0=6, ell_max=80, mu=1e-3, tau=30.0)
    b = impl.adaptive(op, impl.Rng(11), mode="error", ell0=6, ell_max=80, mu=1e-3, tau=30.0)
    assert a.ell_final == b.ell_final and a.doublings == b.doublings and a.hit_cap == b.hit_cap
    assert np.array_equal(a.approximation.u, b.approximation.u)
    assert np.array_equal(a.approximation.lam, b.approximation.lam)
    assert a.error_estimate == b.error_estimate


def test_fixed_rank_strategy(impl):  # :202-218
    op = impl.synthesize_operator(geo_spectrum(60, 0.85), 21)
    out = impl.adaptive(op, impl.Rng(13), mode="fixed", ell0=5, ell_max=24, mu=1e-3, tau=30.0)
    assert out.ell_final == 24 and out.doublings == 0 and not out.hit_cap
    want = (out.approximation.lambda_min + 1e-3 + max(0.0, out.error_estimate)) / 1e-3
    assert out.posterior_condition_estimate == pytest.approx(want)


def test_posterior_arithmetic(impl):  # :220-226
    assert impl.posterior_condition_estimate(0.0, 1.0, 0.0) == 1.0
    assert impl.posterior_condition_estimate(1.0, 1.0, 2.0) == 4.0
    for bad in ((1.0, 0.0, 1.0), (-1.0, 1.0, 0.0), (1.0, 1.0, -2.0)):
        with pytest.raises(ValueError):
            impl.posterior_condition_estimate(*bad)


def test_configuration_validation(impl):  # :250-277
    op = impl.DenseOperator(np.eye(10))
    rng = impl.Rng(15)
    for kw in (dict(ell0=0, ell_max=5, mu=1.0), dict(ell0=6, ell_max=5, mu=1.0),
               dict(ell0=2, ell_max=11, mu=1.0), dict(ell0=2, ell_max=5, mu=0.0),
               dict(ell0=2, ell_max=5, mu=1.0, tau=-3.0), dict(ell0=2, ell_max=5, mu=1.0, q=0)):
        kw.setdefault("tau", 10.0)
        with pytest.raises(ValueError):
            impl.adaptive(op, rng, mode="error", **kw)


def test_column_sampling_drives_the_adaptive_loop(impl):  # adaptive_test.cpp:180-199
    rng = impl.Rng(12)
    pts = rng.gaussian_matrix(60, 3)
    op = impl.KernelOperator(pts, 0.8)
    out = impl.adaptive(op, rng, mode="ratio", ell0=5, ell_max=60, mu=1e-2, tau=10.0, sketch="column_sampling")
    assert out.ell_final >= 5
    if not out.hit_cap:
        assert out.approximation.lambda_min <= 0.1
    u = out.approximation.u
    assert np.abs(u.T @ u - np.eye(out.ell_final)).max() < 1e-10
    gram = impl.GramRidgeOperator(rng.gaussian_matrix(30, 10))
    with pytest.raises(RuntimeError):
        impl.adaptive(gram, rng, mode="ratio", ell0=2, ell_max=10, mu=1e-2, tau=10.0, sketch="column_sampling")


@pytest.mark.gpu
@pytest.mark.parametrize("ell0,ell_max,diag", [(4, 16, "flat"), (5, 12, "flat"), (10, 100, "tail"), (3, 40, "poly")])
def test_adaptive_stream_position_matches_reference(orc, ell0, ell_max, diag):
    """The library's draw-ahead (next Omega block and power vector drawn on a
    host thread while the GPU works) must leave the caller's Rng exactly where
    the reference's sequential draws leave it (random.hpp:11-20), whether the
    loop stops on the estimate, on the cap after an estimate, or on the top-up."""
    import paper_2110_02820_b200 as npcg
    n = 100
    d = {"flat": np.ones(n), "tail": np.r_[1.0, np.full(n - 1, 1e-12)],
         "poly": np.arange(1, n + 1, dtype=float) ** -2.0}[diag]
    outs, rngs = [], []
    for impl in (npcg, orc):
        rng = impl.Rng(21)
        outs.append(impl.adaptive(impl.DenseOperator(np.diag(d)), rng, mode="error", ell0=ell0, ell_max=ell_max,
                                  mu=1e-3, tau=10.0))
        rngs.append(rng)
    assert (outs[0].ell_final, outs[0].doublings, outs[0].hit_cap) == (outs[1].ell_final, outs[1].doublings,
                                                                       outs[1].hit_cap)
    assert rngs[0].normal() == rngs[1].normal()
    assert np.array_equal(rngs[0].gaussian_vector(5), rngs[1].gaussian_vector(5))
