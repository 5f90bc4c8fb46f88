"""The reference's benchmark harness over the library (bench.hpp / bench.cpp,
SURVEY §8f f4): cases of /root/reference/proj/tests/bench_test.cpp."""
import json
import math

import numpy as np
import pytest

from paper_2110_02820_b200 import benchmark as bm


def synthetic_spec(eigs, mu):
    return bm.ProblemSpec(synthetic=np.asarray(eigs, dtype=float), mu=mu)


def test_fnv1a_offset_and_byte_images():
    f = bm.Fnv1a()
    assert f.hex() == "%016x" % 1469598103934665603  # the reference's basis, kept as written (bench.cpp:71)
    f.add_str("")  # one NUL byte
    h = (1469598103934665603 ^ 0) * 1099511628211 % (1 << 64)
    assert f.hex() == "%016x" % h


def test_spec_hash_tracks_configuration_not_seed():  # bench_test.cpp:106-121
    a = synthetic_spec(np.ones(5), 0.5)
    b = bm.ProblemSpec(**{**a.__dict__, "seed": 999})
    assert bm.spec_hash(a) == bm.spec_hash(b)
    for change in ({"mu": 0.25}, {"problem_id": "other"}, {"max_iter": 321}, {"tau": 3.0},
                   {"solver": "cg"}, {"policy": "adaptive_ratio"}, {"rhs": np.ones(5)}):
        assert bm.spec_hash(a) != bm.spec_hash(bm.ProblemSpec(**{**a.__dict__, **change})), change
    k1 = bm.ProblemSpec(krr=bm.KrrSource(np.ones((4, 2)), 1.0, "n_mu"), mu=1e-3)
    k2 = bm.ProblemSpec(krr=bm.KrrSource(np.ones((4, 2)), 1.0, "mu"), mu=4e-3)
    assert bm.spec_hash(k1) != bm.spec_hash(k2)  # bench_test.cpp:235


def test_summarize_mean_and_std():  # bench_test.cpp:144-165
    a = bm.BenchRecord(iterations=10, residual=1e-3, converged=True)
    b = bm.BenchRecord(iterations=20, residual=3e-3, converged=False, failure="diverged")
    j = json.loads(bm.summarize([a, b]))
    assert j["trials"] == 2 and j["converged"] == 1 and j["failures"] == 1
    assert j["iterations"]["mean"] == 15.0
    assert abs(j["iterations"]["std"] - math.sqrt(50.0)) <= 1e-14 * math.sqrt(50.0)
    assert abs(j["residual"]["mean"] - 2e-3) <= 1e-14 * 2e-3
    assert j["posterior_condition"] is None


def test_invalid_specs_are_recorded_not_raised():  # bench_test.cpp:192-203 (no device work)
    rec = bm.run_benchmark(bm.ProblemSpec())
    assert rec.failure and not rec.converged


@pytest.mark.gpu
def test_cg_identity_converges_in_one_iteration():  # bench_test.cpp:46-58
    spec = synthetic_spec(np.ones(20), 0.0)
    spec.solver, spec.seed = "cg", 7
    rec = bm.run_benchmark(spec)
    assert not rec.failure and rec.converged and rec.iterations == 1
    assert rec.residual <= spec.eta and rec.n == 20 and rec.d == 20 and rec.ell_final == 0


@pytest.mark.gpu
def test_trials_use_per_trial_seeds_and_replay():  # bench_test.cpp:123-142
    spec = synthetic_spec(0.6 ** np.arange(1, 41), 1e-2)
    spec.rank, spec.seed = 8, 100
    recs = bm.run_benchmark_trials(spec, 4)
    for i, r in enumerate(recs):
        assert r.seed == 100 + i
        again = bm.run_benchmark(bm.ProblemSpec(**{**spec.__dict__, "seed": 100 + i}))
        assert (again.iterations, again.residual, again.ell_final, again.spec_hash) == \
            (r.iterations, r.residual, r.ell_final, r.spec_hash)


@pytest.mark.gpu
def test_records_serialize_to_json_lines():  # bench_test.cpp:167-178
    spec = synthetic_spec(np.ones(6), 1.0)
    spec.rank = 3
    rec = bm.run_benchmark(spec)
    j = json.loads(rec.json_line())
    assert j["n"] == 6 and j["mu"] == 1.0 and j["ell_final"] == 3 and j["seed"] == 0
    assert j["spec_hash"] == rec.spec_hash and j["total_time"] >= 0.0


@pytest.mark.gpu
def test_rank_zero_applies_deff_rule():  # bench_test.cpp:205-212
    spec = synthetic_spec(np.ones(10), 1.0)
    rec = bm.run_benchmark(spec)
    assert not rec.failure and rec.ell_final == 10


@pytest.mark.gpu
def test_krr_n_mu_matches_literal_shift():  # bench_test.cpp:214-236
    import paper_2110_02820_b200 as npcg
    pts = npcg.Rng(23).gaussian_matrix(40, 2)
    krr = bm.ProblemSpec(krr=bm.KrrSource(pts, 1.0, "n_mu"), mu=1e-3, rank=10, seed=5)
    lit = bm.ProblemSpec(**{**krr.__dict__, "krr": bm.KrrSource(pts, 1.0, "mu"), "mu": 40.0 * 1e-3})
    a, c = bm.run_benchmark(krr), bm.run_benchmark(lit)
    assert not a.failure and a.iterations == c.iterations and a.residual == c.residual
    assert a.d == 2 and a.n == 40


@pytest.mark.gpu
def test_sketch_and_solve_and_block_solvers_end_to_end():  # bench_test.cpp:238-256
    sas = synthetic_spec(0.3 ** np.arange(1, 31), 1e-2)
    sas.solver, sas.rank, sas.eta = "sketch_and_solve", 15, 1e-2
    rec = bm.run_benchmark(sas)
    assert not rec.failure and rec.iterations == 0 and rec.residual < 1e-2
    blk = synthetic_spec(0.3 ** np.arange(1, 31), 1e-2)
    blk.solver, blk.rank = "block_pcg", 10
    brec = bm.run_benchmark(blk)
    assert not brec.failure and brec.converged and brec.residual <= blk.eta


@pytest.mark.gpu
def test_solver_failure_is_recorded(tmp_path):  # bench_test.cpp:180-190
    from paper_2110_02820_b200 import matrix_io
    path = tmp_path / "negdef.csv"
    matrix_io.save_matrix(str(path), -np.eye(3), "csv-dense")
    spec = bm.ProblemSpec(file=bm.FileSource(str(path), "csv_dense"), solver="cg", mu=0.0)
    rec = bm.run_benchmark(spec)
    assert not rec.converged and rec.failure
