"""Port of /root/reference/proj/tests/support/test_support.hpp:15-75 — naive
dense helpers used as independent oracles by the KAT suites. Random draws go
through the implementation's own reference-compatible Rng."""
import numpy as np


def random_orthogonal(impl, rng, n):
    # random.cpp:40-42
    return impl.orthonormal_columns(rng.gaussian_matrix(n, n))


def psd_from_spectrum(impl, lambdas, rng):
    # test_support.hpp:15-20
    lam = np.asarray(lambdas, dtype=np.float64)
    q = random_orthogonal(impl, rng, lam.size)
    a = (q * lam) @ q.T
    return np.asfortranarray((a + a.T) / 2.0)


def poly_spectrum(n, power):
    return np.array([(j + 1.0) ** (-power) for j in range(n)])


def geo_spectrum(n, base):
    out, v = np.empty(n), base
    for j in range(n):
        out[j] = v
        v *= base
    return out


def logspace_spectrum(n, hi, lo):
    if n == 1:
        return np.array([10.0 ** hi])
    return np.array([10.0 ** (hi + (lo - hi) * j / (n - 1)) for j in range(n)])


def random_psd(impl, rng, n, cond=1.0e3):
    # test_support.hpp:51-57
    lo = -np.log10(cond)
    lam = np.array([10.0 ** (lo * rng.uniform()) for _ in range(n)])
    return psd_from_spectrum(impl, lam, rng)


def rel_diff(x, y):
    x, y = np.asarray(x), np.asarray(y)
    scale = np.linalg.norm(y)
    d = np.linalg.norm(x - y)
    return d / scale if scale > 0 else d


def min_eigenvalue(a):
    return float(np.linalg.eigvalsh((a + a.T) / 2).min())


def sym_eigenvalues(a):
    return np.sort(np.linalg.eigvalsh((a + a.T) / 2))[::-1]


def spectral_norm(a):
    v = np.linalg.eigvalsh((a + a.T) / 2)
    return float(max(abs(v[0]), abs(v[-1])))


def nystrom_definitional(a, x):
    # nystrom.cpp:186-200 (dense oracle; pseudo-inverse of the core)
    ax = a @ x
    core = x.T @ ax
    return ax @ np.linalg.pinv(core) @ ax.T


def energy_norm(m, v):
    return float(np.sqrt(v @ (m @ v)))


def effective_dimension(lam, mu):
    # diagnostics.cpp:12-18
    return float(sum(l / (l + mu) for l in lam))


def recommended_sketch_size(lam, mu):
    # diagnostics.cpp:31-35
    import math
    deff = effective_dimension(lam, mu)
    return min(2 * int(math.ceil(1.5 * deff)) + 1, len(lam))


def preconditioner_matrix(approx, mu):
    # NystromPreconditioner::materialize (preconditioner.cpp:47-54)
    u, lam = approx.u, approx.lam
    n = u.shape[0]
    p = np.eye(n)
    if lam.size == 0:
        return p
    gain = (lam + mu) / (lam[-1] + mu) - 1.0
    return p + (u * gain) @ u.T


def exact_condition_number(p, a_mu):
    # diagnostics.cpp:64-88 (dense O(n^3) oracle): cond(P^-1/2 A_mu P^-1/2)
    w, v = np.linalg.eigh((p + p.T) / 2)
    inv_sqrt = (v / np.sqrt(w)) @ v.T
    m = inv_sqrt @ a_mu @ inv_sqrt
    eig = np.linalg.eigvalsh((m + m.T) / 2)
    return float(eig[-1] / eig[0])
