"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

The oracle (oracle/npcg_oracle.cpp) is a line-by-line restatement of the
reference's hot path (/root/reference/proj/core/src/*.cpp, cited per function
there). Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` legs may import this module; the product package
(paper_2110_02820_b200) never does.

Arrays are numpy float64 in column-major (Fortran) order, matching the
reference's Eigen::MatrixXd layout.
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libnpcg_oracle.so"

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


def _cpu_has_avx512() -> bool:
    try:
        return "avx512f" in Path("/proc/cpuinfo").read_text()
    except OSError:
        return False


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (g++ + bundled OpenBLAS); make
    rebuilds only when a source changed."""
    if force or not LIB_PATH.exists() or shutil.which("make"):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


class OracleError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """reference std::invalid_argument"""


class SolveDivergenceError(RuntimeError):
    """reference npcg::SolveDivergenceError (solvers.hpp:51-57); carries the partial report."""

    def __init__(self, msg, report=None):
        super().__init__(msg)
        self.report = report


_lib = None


def lib():
    global _lib
    if _lib is None:
        # OpenBLAS 0.3.15 misdetects this CPU family as "Prescott" (4x slower
        # DGEMM); the core type is read once when the library loads.
        os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX" if _cpu_has_avx512() else "Haswell")
        build()
        L = C.CDLL(str(LIB_PATH))
        L.orc_last_error.restype = C.c_char_p
        L.orc_corename.restype = C.c_char_p
        L.orc_rng_new.restype = _vp
        L.orc_rng_new.argtypes = [C.c_uint64]
        L.orc_rng_clone.restype = _vp
        L.orc_rng_clone.argtypes = [_vp]
        L.orc_rng_free.argtypes = [_vp]
        L.orc_rng_normal.restype = C.c_double
        L.orc_rng_normal.argtypes = [_vp]
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_uniform.argtypes = [_vp]
        L.orc_rng_word.restype = C.c_uint64
        L.orc_rng_word.argtypes = [_vp]
        L.orc_rng_discard.argtypes = [_vp, C.c_uint64]
        L.orc_rng_integer.argtypes = [_vp, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_gaussian_matrix.argtypes = [_vp, _i64, _i64, _dp]
        L.orc_rng_uniform_fill.argtypes = [_vp, _i64, _dp]
        L.orc_rng_uniform_fill.restype = None
        L.orc_sample_without_replacement.argtypes = [_vp, _i64, _i64, C.POINTER(_i64)]
        L.orc_orthonormal_columns.argtypes = [_i64, _i64, _dp, _dp]
        L.orc_thin_svd.argtypes = [_i64, _i64, _dp, _dp, _dp]
        L.orc_sym_eig.argtypes = [_i64, _dp, _dp, _dp]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_ulp_spacing.restype = C.c_double
        L.orc_ulp_spacing.argtypes = [C.c_double]
        L.orc_op_dim.restype = _i64
        L.orc_op_dim.argtypes = [_vp]
        L.orc_op_free.argtypes = [_vp]
        L.orc_sketch_free.argtypes = [_vp]
        L.orc_sketch_size.restype = _i64
        L.orc_sketch_size.argtypes = [_vp]
        L.orc_sketch_get.argtypes = [_vp, _dp, _dp]
        L.orc_approx_free.argtypes = [_vp]
        L.orc_approx_info.argtypes = [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(C.c_double)]
        L.orc_approx_get.argtypes = [_vp, _dp, _dp]
        L.orc_pre_free.argtypes = [_vp]
        for name in ("orc_set_threads",):
            getattr(L, name).argtypes = [C.c_int]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _f64(a, shape=None):
    arr = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        arr = arr.reshape(shape, order="F")
    return arr


def _check(rc, report=None):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 3:
        raise SolveDivergenceError(msg, report)
    raise OracleError(msg)


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return lib().orc_get_threads()


def corename() -> str:
    return lib().orc_corename().decode()


# ---------------------------------------------------------------- random.cpp
class Rng:
    """reference npcg::Rng (random.hpp:21-38): std::mt19937_64 + Box-Muller."""

    def __init__(self, seed: int = 0, _handle=None):
        self.h = _handle if _handle is not None else lib().orc_rng_new(C.c_uint64(seed))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_rng_free(self.h)
            self.h = None

    def clone(self) -> "Rng":
        return Rng(_handle=lib().orc_rng_clone(self.h))

    def normal(self) -> float:
        return lib().orc_rng_normal(self.h)

    def uniform(self) -> float:
        return lib().orc_rng_uniform(self.h)

    def word(self) -> int:
        return lib().orc_rng_word(self.h)

    def discard(self, k: int):
        lib().orc_rng_discard(self.h, C.c_uint64(k))

    def integer(self, bound: int) -> int:
        out = C.c_uint64()
        _check(lib().orc_rng_integer(self.h, C.c_uint64(bound), C.byref(out)))
        return out.value

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        lib().orc_gaussian_matrix(self.h, rows, cols, _ptr(out))
        return out

    def gaussian_vector(self, n: int) -> np.ndarray:
        return self.gaussian_matrix(n, 1)[:, 0].copy()

    def uniform_fill(self, count: int) -> np.ndarray:
        out = np.empty(count)
        lib().orc_rng_uniform_fill(self.h, _i64(count), _ptr(out))
        return out

    def sample_without_replacement(self, n: int, k: int) -> np.ndarray:
        out = np.empty(max(k, 0), dtype=np.int64)
        _check(lib().orc_sample_without_replacement(self.h, n, k, out.ctypes.data_as(C.POINTER(_i64))))
        return out


def splitmix64(seed: int) -> int:
    """bench.cpp:180-185 synthetic_operator_seed."""
    return lib().orc_splitmix64(C.c_uint64(seed))


# ---------------------------------------------------------------- dense.cpp
def ulp_spacing(x: float) -> float:
    return lib().orc_ulp_spacing(float(x))


def orthonormal_columns(g) -> np.ndarray:
    g = _f64(g)
    q = np.empty_like(g, order="F")
    _check(lib().orc_orthonormal_columns(g.shape[0], g.shape[1], _ptr(g), _ptr(q)))
    return q


def thin_svd(b):
    b = _f64(b)
    m, n = b.shape
    u = np.empty((m, n), order="F")
    s = np.empty(n)
    _check(lib().orc_thin_svd(m, n, _ptr(b), _ptr(u), _ptr(s)))
    return u, s


def sym_eig(a):
    a = _f64(a)
    n = a.shape[0]
    vals = np.empty(n)
    vecs = np.empty((n, n), order="F")
    _check(lib().orc_sym_eig(n, _ptr(a), _ptr(vals), _ptr(vecs)))
    return vals, vecs


# ---------------------------------------------------------------- operators.cpp
class LinearOperator:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_op_free(C.c_void_p(self.h))
            self.h = None

    def dim(self) -> int:
        return lib().orc_op_dim(C.c_void_p(self.h))

    def matvec(self, v) -> np.ndarray:
        v = _f64(v).ravel(order="F")
        out = np.empty(self.dim())
        _check(lib().orc_op_apply(C.c_void_p(self.h), _i64(v.size), _i64(1), _ptr(v), _ptr(out)))
        return out

    def apply_block(self, V) -> np.ndarray:
        V = _f64(V)
        if V.ndim == 1:
            V = V.reshape(-1, 1, order="F")
        out = np.empty((self.dim(), V.shape[1]), order="F")
        _check(lib().orc_op_apply_block(C.c_void_p(self.h), _i64(V.shape[0]), _i64(V.shape[1]), _ptr(V), _ptr(out)))
        return out

    def column(self, j: int) -> np.ndarray:
        out = np.empty(self.dim())
        _check(lib().orc_op_column(C.c_void_p(self.h), _i64(j), _ptr(out)))
        return out

    def dense(self) -> np.ndarray:
        n = self.dim()
        out = np.empty((n, n), order="F")
        _check(lib().orc_op_dense_data(C.c_void_p(self.h), _ptr(out)))
        return out


def _new_op(fn, *args) -> LinearOperator:
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return LinearOperator(h.value)


def DenseOperator(a) -> LinearOperator:
    a = _f64(a)
    if a.ndim != 2:
        raise InvalidArgument("DenseOperator: matrix must be square")
    return _new_op(lib().orc_op_dense, _i64(a.shape[0]), _i64(a.shape[1]), _ptr(a))


def GramRidgeOperator(g) -> LinearOperator:
    g = _f64(g)
    if g.ndim != 2:
        g = g.reshape(g.shape[0] if g.ndim else 0, -1)
    return _new_op(lib().orc_op_gram, _i64(g.shape[0]), _i64(g.shape[1]), _ptr(g))


def KernelOperator(points, sigma: float, dense_cap: int = 20000) -> LinearOperator:
    p = _f64(points)
    return _new_op(lib().orc_op_kernel, _i64(p.shape[0]), _i64(p.shape[1]), _ptr(p),
                   C.c_double(sigma), _i64(dense_cap))


def synthesize_operator(eigenvalues, seed: int) -> LinearOperator:
    lam = _f64(eigenvalues).ravel()
    return _new_op(lib().orc_op_synth, _i64(lam.size), _ptr(lam), C.c_uint64(seed))


# ---------------------------------------------------------------- nystrom.cpp
@dataclass
class NystromApproximation:
    u: np.ndarray
    lam: np.ndarray
    shift_used: float
    h: object = field(default=None, repr=False)

    @property
    def lambda_min(self):
        return float(self.lam[-1]) if self.lam.size else 0.0

    def materialize(self):
        return (self.u * self.lam) @ self.u.T


class _Handle:
    def __init__(self, h, free):
        self.h, self._free = h, free

    def __del__(self):
        if self.h:
            self._free(C.c_void_p(self.h))
            self.h = None


def _approx_from_handle(h) -> NystromApproximation:
    n, ell, shift = _i64(), _i64(), C.c_double()
    lib().orc_approx_info(C.c_void_p(h), C.byref(n), C.byref(ell), C.byref(shift))
    u = np.empty((n.value, ell.value), order="F")
    lam = np.empty(ell.value)
    lib().orc_approx_get(C.c_void_p(h), _ptr(u), _ptr(lam))
    return NystromApproximation(u, lam, shift.value, _Handle(h, lib().orc_approx_free))


def make_approximation(u, lam, shift_used=0.0) -> NystromApproximation:
    u = _f64(u)
    lam = _f64(lam).ravel()
    if u.ndim == 1:
        u = u.reshape(-1, 0 if lam.size == 0 else 1)
    h = C.c_void_p()
    _check(lib().orc_approx_make(_i64(u.shape[0]), _i64(u.shape[1]), _ptr(u), _ptr(lam),
                                 C.c_double(shift_used), C.byref(h)))
    return _approx_from_handle(h.value)


class SketchPair:
    def __init__(self, h):
        self._h = _Handle(h, lib().orc_sketch_free)

    @property
    def h(self):
        return self._h.h

    def size(self):
        return lib().orc_sketch_size(C.c_void_p(self.h))

    def arrays(self, n):
        k = self.size()
        om = np.empty((n, k), order="F")
        y = np.empty((n, k), order="F")
        lib().orc_sketch_get(C.c_void_p(self.h), _ptr(om), _ptr(y))
        return om, y


def make_empty_sketch(n: int) -> SketchPair:
    h = C.c_void_p()
    _check(lib().orc_sketch_empty(_i64(n), C.byref(h)))
    return SketchPair(h.value)


def extend_sketch(pair: SketchPair, op: LinearOperator, extra: int, rng: Rng) -> SketchPair:
    h = C.c_void_p()
    _check(lib().orc_sketch_extend(C.c_void_p(pair.h), C.c_void_p(op.h), _i64(extra), C.c_void_p(rng.h), C.byref(h)))
    return SketchPair(h.value)


def extend_sketch_with(pair: SketchPair, op: LinearOperator, fresh) -> SketchPair:
    fresh = _f64(fresh)
    h = C.c_void_p()
    _check(lib().orc_sketch_extend_with(C.c_void_p(pair.h), C.c_void_p(op.h), _i64(fresh.shape[1]),
                                        _ptr(fresh), C.byref(h)))
    return SketchPair(h.value)


def extend_sketch_columns(pair: SketchPair, op: LinearOperator, extra: int, used: list, rng: Rng) -> SketchPair:
    """extend_sketch_columns (nystrom.cpp:60-94); `used` is extended in place."""
    u = np.ascontiguousarray(used, dtype=np.int64)
    uo = np.zeros(len(used) + max(int(extra), 0), dtype=np.int64)
    h = C.c_void_p()
    _check(lib().orc_sketch_extend_columns(C.c_void_p(pair.h), C.c_void_p(op.h), _i64(extra),
                                           u.ctypes.data_as(C.c_void_p), _i64(len(used)), C.c_void_p(rng.h),
                                           uo.ctypes.data_as(C.c_void_p), C.byref(h)))
    used[:] = [int(v) for v in uo]
    return SketchPair(h.value)


def column_sampling_nystrom(op: LinearOperator, ell_or_indices, rng: Rng | None = None) -> NystromApproximation:
    """column_sampling_nystrom (nystrom.cpp:150-184): by count with an Rng, or by caller indices."""
    h = C.c_void_p()
    if rng is not None:
        _check(lib().orc_column_sampling_nystrom_rng(C.c_void_p(op.h), _i64(ell_or_indices), C.c_void_p(rng.h),
                                                     C.byref(h)))
    else:
        idx = np.ascontiguousarray(ell_or_indices, dtype=np.int64)
        _check(lib().orc_column_sampling_nystrom(C.c_void_p(op.h), _i64(idx.size), idx.ctypes.data_as(C.c_void_p),
                                                 C.byref(h)))
    return _approx_from_handle(h.value)


def nystrom_from_sketch(pair: SketchPair) -> NystromApproximation:
    h = C.c_void_p()
    _check(lib().orc_nystrom_from_sketch(C.c_void_p(pair.h), C.byref(h)))
    return _approx_from_handle(h.value)


def randomized_nystrom(op: LinearOperator, ell: int, rng: Rng) -> NystromApproximation:
    h = C.c_void_p()
    _check(lib().orc_randomized_nystrom(C.c_void_p(op.h), _i64(ell), C.c_void_p(rng.h), C.byref(h)))
    return _approx_from_handle(h.value)


# ---------------------------------------------------------------- preconditioner.cpp
class NystromPreconditioner:
    def __init__(self, h, n, mu):
        self._h = _Handle(h, lib().orc_pre_free)
        self.n, self.mu = n, mu

    @property
    def h(self):
        return self._h.h

    def apply_inverse(self, r) -> np.ndarray:
        r = _f64(r)
        s = 1 if r.ndim == 1 else r.shape[1]
        out = np.empty(r.shape, order="F")
        _check(lib().orc_pre_apply_inverse(C.c_void_p(self.h), _i64(r.shape[0]), _i64(s), _ptr(r), _ptr(out)))
        return out

    def apply(self, v) -> np.ndarray:
        v = _f64(v)
        out = np.empty_like(v)
        _check(lib().orc_pre_apply(C.c_void_p(self.h), _i64(v.size), _ptr(v), _ptr(out)))
        return out


def build_preconditioner(approx: NystromApproximation, mu: float) -> NystromPreconditioner:
    h = C.c_void_p()
    _check(lib().orc_pre_build(C.c_void_p(approx.h.h), C.c_double(mu), C.byref(h)))
    return NystromPreconditioner(h.value, approx.u.shape[0], mu)


def woodbury_inverse_apply(approx: NystromApproximation, mu: float, b) -> np.ndarray:
    """preconditioner.cpp:104-114 on the approximation's (U, lambda)."""
    b = _f64(b).ravel()
    x = np.empty(b.size)
    _check(lib().orc_woodbury(C.c_void_p(approx.h.h), C.c_double(mu), _i64(b.size), _ptr(b), _ptr(x)))
    return x


def sketch_and_solve(op, b, mu: float, ell: int, rng: Rng) -> np.ndarray:
    """preconditioner.cpp:116-121."""
    if not mu > 0.0:
        raise InvalidArgument("sketch_and_solve: mu must be > 0")
    return woodbury_inverse_apply(randomized_nystrom(op, ell, rng), mu, b)


# ---------------------------------------------------------------- solvers.cpp
@dataclass
class SolveReport:
    x: np.ndarray
    iterations: int
    residual_history: np.ndarray
    converged: bool
    matvec_count: int
    wall_time: float
    eta_used: float
    iterates: np.ndarray | None = None


def _solve_buffers(n, max_iter, record_iterates):
    return dict(
        x=np.empty(n), it=_i64(), conv=C.c_int(), mvc=_i64(), eta=C.c_double(), wall=C.c_double(),
        hist=np.empty(max_iter + 1), hlen=_i64(),
        iters=np.empty((max_iter + 1) * n) if record_iterates else None)


def _report(b, n):
    hl = b["hlen"].value
    iters = None
    if b["iters"] is not None:
        iters = b["iters"][: hl * n].reshape(hl, n)
    return SolveReport(b["x"], b["it"].value, b["hist"][:hl].copy(), bool(b["conv"].value),
                       b["mvc"].value, b["wall"].value, b["eta"].value, iters)


def nystrom_pcg(op: LinearOperator, b, mu: float, precond: NystromPreconditioner | None,
                eta=1e-10, max_iter=500, relative=False, record_iterates=False, x0=None) -> SolveReport:
    n = op.dim()
    b = _f64(b).ravel()
    x0 = None if x0 is None else _f64(x0).ravel()
    buf = _solve_buffers(n, max_iter, record_iterates)
    rc = lib().orc_pcg(C.c_void_p(op.h), _ptr(b), _ptr(x0), C.c_double(mu),
                       None if precond is None else C.c_void_p(precond.h), C.c_double(eta),
                       _i64(max_iter), C.c_int(int(relative)), C.c_int(int(record_iterates)),
                       _ptr(buf["x"]), C.byref(buf["it"]), C.byref(buf["conv"]), C.byref(buf["mvc"]),
                       C.byref(buf["eta"]), C.byref(buf["wall"]), _ptr(buf["hist"]), C.byref(buf["hlen"]),
                       _ptr(buf["iters"]))
    rep = _report(buf, n)
    _check(rc, rep)
    return rep


class RegularizedOperator:
    """RegularizedOperator(base, mu) (operators.cpp:82-103): matvec = base.matvec(v); out += mu v."""

    def __init__(self, base, mu: float):
        if base is None:
            raise InvalidArgument("RegularizedOperator: base operator is null")
        if not mu >= 0.0:
            raise InvalidArgument("RegularizedOperator: mu must be >= 0")
        self.base, self.mu = base, float(mu)

    def dim(self) -> int:
        return self.base.dim()

    def has_column_access(self) -> bool:
        return False

    def matvec(self, v) -> np.ndarray:
        out = self.base.matvec(v)
        out += self.mu * np.asarray(v, dtype=np.float64)
        return out

    def apply_block(self, V) -> np.ndarray:
        out = self.base.apply_block(V)
        out += self.mu * np.asarray(V, dtype=np.float64)
        return out


def regularize(op, mu: float) -> RegularizedOperator:
    return RegularizedOperator(op, mu)


def cg(op, *args, eta=1e-10, max_iter=500, relative=False, x0=None) -> SolveReport:
    """cg(op_mu, b[, x0]) (solvers.cpp:111-120), or the shorthand cg(op, mu, b)."""
    if len(args) >= 1 and np.ndim(args[0]) == 0:
        mu, rest = float(args[0]), args[1:]
    else:
        mu, rest = 0.0, args
    b = rest[0]
    if len(rest) > 1:
        x0 = rest[1]
    if isinstance(op, RegularizedOperator):  # the C++ restatement's Regularized wrapper does the same arithmetic
        if mu != 0.0:
            raise InvalidArgument("cg: shift given twice")
        op, mu = op.base, op.mu
    n = op.dim()
    b = _f64(b).ravel()
    x0 = None if x0 is None else _f64(x0).ravel()
    buf = _solve_buffers(n, max_iter, False)
    rc = lib().orc_cg(C.c_void_p(op.h), C.c_double(mu), _ptr(b), _ptr(x0), C.c_double(eta),
                      _i64(max_iter), C.c_int(int(relative)), _ptr(buf["x"]), C.byref(buf["it"]),
                      C.byref(buf["conv"]), C.byref(buf["mvc"]), C.byref(buf["eta"]), C.byref(buf["wall"]),
                      _ptr(buf["hist"]), C.byref(buf["hlen"]))
    rep = _report(buf, n)
    _check(rc, rep)
    return rep


@dataclass
class BlockSolveReport:
    x: np.ndarray
    iterations: int
    converged: list
    deflated: list
    fallback_count: int
    final_residual: np.ndarray
    residual_history: list | None = None  # per column, every iteration (solvers.hpp:40-49)


def block_nystrom_pcg(op, B, mu, precond, eta=1e-10, max_iter=500, relative=False) -> BlockSolveReport:
    B = _f64(B)
    n, s = B.shape
    x = np.empty((n, s), order="F")
    it, nd, fb = _i64(), _i64(), _i64()
    conv = (C.c_int * s)()
    defl = (_i64 * s)()
    fres = np.empty(s)
    hist = np.zeros((max_iter + 1, s), order="F")
    hlen = np.zeros(s, dtype=np.int64)
    _check(lib().orc_block_pcg(C.c_void_p(op.h), _i64(s), _ptr(B), C.c_double(mu),
                               None if precond is None else C.c_void_p(precond.h), C.c_double(eta),
                               _i64(max_iter), C.c_int(int(relative)), _ptr(x), C.byref(it), conv, defl,
                               C.byref(nd), C.byref(fb), _ptr(fres), _ptr(hist), hlen.ctypes.data_as(C.c_void_p)))
    return BlockSolveReport(x, it.value, [bool(c) for c in conv], list(defl[: nd.value]), fb.value, fres,
                            [hist[: hlen[j], j].copy() for j in range(s)])


def iteration_bound(kappa: float, eps: float) -> int:
    out = _i64()
    _check(lib().orc_iteration_bound(C.c_double(kappa), C.c_double(eps), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- adaptive.cpp
def estimate_error_power(op, approx: NystromApproximation, q: int, rng: Rng) -> float:
    out = C.c_double()
    _check(lib().orc_estimate_error_power(C.c_void_p(op.h), C.c_void_p(approx.h.h), _i64(q),
                                          C.c_void_p(rng.h), C.byref(out)))
    return out.value


@dataclass
class AdaptiveOutcome:
    approximation: NystromApproximation
    error_estimate: float | None
    doublings: int
    hit_cap: bool
    posterior_condition_estimate: float
    ell_final: int


def adaptive(op, rng: Rng, *, mode="error", ell0=10, ell_max=0, mu=0.0, tau=None, q=5,
             secondary_criterion=True, sketch="gaussian") -> AdaptiveOutcome:
    modes = {"error": 0, "ratio": 1, "fixed": 2}
    h = C.c_void_p()
    has_err, err, dbl, cap, post, ellf = C.c_int(), C.c_double(), _i64(), C.c_int(), C.c_double(), _i64()
    _check(lib().orc_adaptive(C.c_void_p(op.h), C.c_int(modes[mode]), _i64(ell0), _i64(ell_max),
                              C.c_double(mu), C.c_int(tau is not None), C.c_double(tau or 0.0), _i64(q),
                              C.c_int(int(secondary_criterion)), C.c_int(0 if sketch == "gaussian" else 1),
                              C.c_void_p(rng.h), C.byref(h), C.byref(has_err), C.byref(err), C.byref(dbl),
                              C.byref(cap), C.byref(post), C.byref(ellf)))
    return AdaptiveOutcome(_approx_from_handle(h.value), err.value if has_err.value else None, dbl.value,
                           bool(cap.value), post.value, ellf.value)


def posterior_condition_estimate(lam_ell, mu, err) -> float:
    out = C.c_double()
    _check(lib().orc_posterior(C.c_double(lam_ell), C.c_double(mu), C.c_double(err), C.byref(out)))
    return out.value
