"""KATs of /root/reference/proj/tests/random_dense_test.cpp, run against the
CPU oracle (CPU suite) and the B200 product (GPU suite)."""
import numpy as np
import pytest

from support import random_orthogonal


def test_mt19937_64_standard_known_answer(impl):
    # C++ standard [rand.predef]: the 10000th output of a default-constructed
    # std::mt19937_64 (seed 5489) is 9981545732273789042. Pins the engine the
    # reference uses (random.hpp:37).
    rng = impl.Rng(5489)
    rng.discard(9999)
    assert rng.word() == 9981545732273789042


def test_rng_is_deterministic_in_the_seed(impl):  # random_dense_test.cpp:11-22
    a, b, c = impl.Rng(7), impl.Rng(7), impl.Rng(8)
    xs = [a.normal() for _ in range(100)]
    assert xs == [b.normal() for _ in range(100)]
    assert xs != [c.normal() for _ in range(100)]


def test_normal_moments(impl):  # :24-38
    rng = impl.Rng(123)
    x = rng.gaussian_vector(100000)
    assert np.all(np.isfinite(x))
    assert abs(x.mean()) < 0.02
    assert abs(x.var() - 1.0) < 0.05


def test_uniform_and_integer_stay_in_range(impl):  # :40-51
    rng = impl.Rng(5)
    for _ in range(1000):
        u = rng.uniform()
        assert 0.0 <= u < 1.0
        assert rng.integer(7) < 7
    with pytest.raises(ValueError):
        rng.integer(0)


def test_block_draws_align_with_column_stream(impl):  # :52-63
    n, a, b = 17, 4, 6
    split, joint = impl.Rng(99), impl.Rng(99)
    g1 = split.gaussian_matrix(n, a)
    g2 = split.gaussian_matrix(n, b)
    g = joint.gaussian_matrix(n, a + b)
    assert np.array_equal(g[:, :a], g1)
    assert np.array_equal(g[:, a:], g2)


def test_gaussian_vector_matches_first_column(impl):  # :65-70
    v = impl.Rng(3).gaussian_vector(11)
    g = impl.Rng(3).gaussian_matrix(11, 2)
    assert np.array_equal(v, g[:, 0])


def test_random_orthogonal_is_orthogonal(impl):  # :72-78
    q = random_orthogonal(impl, impl.Rng(17), 25)
    eye = np.eye(25)
    assert np.abs(q.T @ q - eye).max() < 1e-12
    assert np.abs(q @ q.T - eye).max() < 1e-12


def test_sample_without_replacement(impl):  # :80-96
    rng = impl.Rng(11)
    s = rng.sample_without_replacement(20, 8)
    assert len(set(s.tolist())) == 8 and s.min() >= 0 and s.max() < 20
    assert len(set(rng.sample_without_replacement(5, 5).tolist())) == 5
    with pytest.raises(ValueError):
        rng.sample_without_replacement(3, 4)


def test_orthonormal_columns_spans_the_input_range(impl):  # :134-142
    g = impl.Rng(41).gaussian_matrix(15, 6)
    q = impl.orthonormal_columns(g)
    assert np.abs(q.T @ q - np.eye(6)).max() < 1e-12
    assert np.abs(q @ (q.T @ g) - g).max() < 1e-11


def test_thin_svd_agrees_with_an_independent_svd(impl):  # :118-132
    b = impl.Rng(31).gaussian_matrix(12, 5)
    u, s = impl.thin_svd(b)
    uo, so, _ = np.linalg.svd(b, full_matrices=False)
    assert np.abs(s - so).max() < 1e-12
    for j in range(5):
        sign = -1.0 if u[:, j] @ uo[:, j] < 0 else 1.0
        assert np.linalg.norm(u[:, j] - sign * uo[:, j]) < 1e-10
    with pytest.raises(ValueError):
        impl.thin_svd(np.ones((3, 5)))


def test_ulp_spacing(impl):  # :158-164
    eps = np.finfo(np.float64).eps
    assert impl.ulp_spacing(1.0) == eps
    assert 0.0 < impl.ulp_spacing(0.0) < 1e-300
    assert impl.ulp_spacing(2.0) == 2 * eps
    assert impl.ulp_spacing(-8.0) == impl.ulp_spacing(8.0)


def test_splitmix64_seed_derivation(impl):  # bench.cpp:180-185
    # splitmix64 reference vector (first output for state 0): 0xe220a8397b1dcdaf
    assert impl.splitmix64(0) == 0xE220A8397B1DCDAF


# ---- the generator on the GPU ---------------------------
@pytest.mark.gpu
def test_device_engine_words_are_the_reference_stream(orc):
    import paper_2110_02820_b200 as npcg
    for seed, skip in ((0, 0), (5, 1), (42, 311), (7, 100001)):
        r, o = npcg.Rng(seed), orc.Rng(seed)
        for _ in range(skip):  # arbitrary stream positions, including mid-block
            assert r.word() == o.word()
        w = r.words_device(3 * 312 + 17)
        ref = np.array([o.word() for _ in range(w.size)], dtype=np.uint64)
        assert np.array_equal(w, ref)
        assert r.word() == o.word()  # the host engine continues exactly after the device draw


@pytest.mark.gpu
def test_device_gaussian_matches_host_draw(orc):
    import paper_2110_02820_b200 as npcg
    r, o = npcg.Rng(9), orc.Rng(9)
    r.gaussian_vector(77)
    o.gaussian_vector(77)  # odd word offset into a block
    g = r.gaussian_matrix_device(1000, 37)
    h = o.gaussian_matrix(1000, 37)
    ulp = np.abs(g - h) / np.spacing(np.maximum(np.abs(h), 1e-300))
    assert np.max(ulp) <= 4, np.max(ulp)  # CUDA log/cos vs libm
    assert np.median(ulp) == 0
    assert r.word() == o.word()
