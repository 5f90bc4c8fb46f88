"""The drop-in boundary beyond the concrete operators: the reference's plug-in
point (a user subclass of LinearOperator, operators.hpp:25-47), the
RegularizedOperator / regularize pair (operators.hpp:69-94,153) and the
cg(op_mu, b[, x0]) entry point the reference bench calls (bench.cpp:218-220).

The user operator runs through the product's C-ABI callback operator
(npcg_op_callback_create); the oracle solves the same matrix as a
DenseOperator, so each library result is pinned to the reference algorithm."""
import numpy as np
import pytest

from support import random_psd


def tridiag(n):
    a = np.diag([2.0 + i / n for i in range(n)]) - np.eye(n, k=1) - np.eye(n, k=-1)
    return np.asfortranarray(a)


class Tridiag:
    """Mixin body of the user operator: only do_dim / do_matvec."""

    def __init__(self, n):
        self.n, self.calls = n, 0
        self.d = np.array([2.0 + i / n for i in range(n)])

    def do_dim(self):
        return self.n

    def do_matvec(self, v):
        self.calls += 1
        out = self.d * v
        out[1:] -= v[:-1]
        out[:-1] -= v[1:]
        return out


def user_op(npcg, n):
    cls = type("TridiagOperator", (Tridiag, npcg.UserOperator), {})
    return cls(n)


def test_regularize_adds_mu_identity(impl):  # operators_test.cpp:78-100
    zero = impl.DenseOperator(np.zeros((2, 2)))
    assert np.array_equal(impl.regularize(zero, 1.0).matvec(np.array([3.0, 4.0])), [3.0, 4.0])
    op = impl.RegularizedOperator(impl.DenseOperator(np.diag([2.0, 1.0])), 0.5)
    assert np.array_equal(op.matvec(np.ones(2)), [2.5, 1.5])
    assert op.mu == 0.5
    a = random_psd(impl, impl.Rng(2), 8)
    base = impl.DenseOperator(a)
    v = impl.Rng(3).gaussian_vector(8)
    assert np.array_equal(impl.RegularizedOperator(base, 0.0).matvec(v), base.matvec(v))
    with pytest.raises(ValueError):
        impl.regularize(base, -1.0)
    assert not impl.regularize(base, 1.0).has_column_access()


def test_cg_on_regularized_operator_equals_shifted_cg(impl):  # solvers.cpp:111-148
    a = random_psd(impl, impl.Rng(4), 40, 1e3)
    op = impl.DenseOperator(a)
    b = impl.Rng(5).gaussian_vector(40)
    r1 = impl.cg(impl.regularize(op, 1e-2), b, eta=1e-10, relative=True)
    r2 = impl.cg(op, 1e-2, b, eta=1e-10, relative=True)
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.x, r2.x)  # same products, same rounding order
    x0 = impl.Rng(6).gaussian_vector(40)
    r3 = impl.cg(impl.regularize(op, 1e-2), b, x0, eta=1e-10, relative=True)
    assert r3.converged and np.linalg.norm(r3.x - r1.x) <= 1e-8 * np.linalg.norm(r1.x)


@pytest.mark.gpu
def test_user_operator_through_every_entry_point(orc):
    import paper_2110_02820_b200 as npcg
    n, mu = 120, 0.05
    user = user_op(npcg, n)
    ref_op = orc.DenseOperator(tridiag(n))
    b = np.cos(0.1 * np.arange(n))
    # matvec / apply_block through the NVI default
    v = npcg.Rng(1).gaussian_vector(n)
    assert np.allclose(user.matvec(v), tridiag(n) @ v, rtol=0, atol=1e-14)
    # cg(regularize(user, mu), b): the reference bench's call
    r = npcg.cg(npcg.regularize(user, mu), b, eta=1e-10, relative=True)
    o = orc.cg(ref_op, mu, b, eta=1e-10, relative=True)
    assert abs(r.iterations - o.iterations) <= 1 and r.matvec_count == r.iterations + 1
    assert np.linalg.norm(r.x - o.x) <= 1e-8 * np.linalg.norm(o.x)
    calls = user.calls
    # randomized Nyström on the user operator (sketch Y = A Omega through the callback)
    approx = npcg.randomized_nystrom(user, 16, npcg.Rng(11))
    oapprox = orc.randomized_nystrom(ref_op, 16, orc.Rng(11))
    assert user.calls > calls
    keep = oapprox.lam >= 1e-6 * oapprox.lam[0]
    assert np.max(np.abs(approx.lam[keep] - oapprox.lam[keep]) / oapprox.lam[keep]) <= 1e-10
    pre, opre = npcg.build_preconditioner(approx, mu), orc.build_preconditioner(oapprox, mu)
    r = npcg.nystrom_pcg(user, b, mu, pre, eta=1e-10, relative=True)
    o = orc.nystrom_pcg(ref_op, b, mu, opre, eta=1e-10, relative=True)
    assert abs(r.iterations - o.iterations) <= 1
    assert np.linalg.norm(r.x - o.x) <= 1e-8 * np.linalg.norm(o.x)
    # block PCG with per-iteration histories
    B = np.column_stack([np.sin(0.05 * (np.arange(n) + 1) * (j + 1)) for j in range(3)])
    rb = npcg.block_nystrom_pcg(user, B, mu, pre, eta=1e-10, relative=True)
    ob = orc.block_nystrom_pcg(ref_op, B, mu, opre, eta=1e-10, relative=True)
    assert abs(rb.iterations - ob.iterations) <= 1
    assert np.linalg.norm(rb.x - ob.x) <= 1e-8 * np.linalg.norm(ob.x)
    assert all(len(h) == rb.iterations + 1 for h in rb.residual_history)
    # power estimate and the adaptive loop (Omega blocks drawn in reference order)
    e = npcg.estimate_error_power(user, approx, 5, npcg.Rng(12))
    oe = orc.estimate_error_power(ref_op, oapprox, 5, orc.Rng(12))
    assert abs(e - oe) <= 1e-8 * abs(oe)
    ad = npcg.adaptive(user, npcg.Rng(13), mode="error", ell0=4, ell_max=32, mu=mu, tau=10.0)
    oad = orc.adaptive(ref_op, orc.Rng(13), mode="error", ell0=4, ell_max=32, mu=mu, tau=10.0)
    assert (ad.ell_final, ad.doublings, ad.hit_cap) == (oad.ell_final, oad.doublings, oad.hit_cap)


@pytest.mark.gpu
def test_user_operator_exceptions_cross_the_library():
    import paper_2110_02820_b200 as npcg

    class Broken(npcg.UserOperator):
        def do_dim(self):
            return 4

        def do_matvec(self, v):
            raise ZeroDivisionError("user operator failed")

    with pytest.raises(ZeroDivisionError):
        npcg.cg(npcg.regularize(Broken(), 1.0), np.ones(4))
    with pytest.raises(ZeroDivisionError):
        npcg.randomized_nystrom(Broken(), 2, npcg.Rng(1))


@pytest.mark.gpu
def test_regularized_device_operator_is_a_device_operator():
    import paper_2110_02820_b200 as npcg
    lam = np.array([(j + 1.0) ** -2 for j in range(300)])
    op = npcg.synthesize_operator(lam, 3)
    reg = npcg.regularize(op, 1e-3)
    assert reg.h is not None and reg.kind == 5
    b = npcg.Rng(2).gaussian_vector(300)
    assert np.array_equal(reg.matvec(b), op.matvec(b) + 1e-3 * b) or \
        np.max(np.abs(reg.matvec(b) - (op.matvec(b) + 1e-3 * b))) == 0.0
    r1 = npcg.cg(reg, b, eta=1e-10, relative=True)
    r2 = npcg.nystrom_pcg(op, b, 1e-3, None, eta=1e-10, relative=True)
    assert r1.iterations == r2.iterations and np.array_equal(r1.x, r2.x)
