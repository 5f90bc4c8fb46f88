"""B200-native Nyström PCG — Python host mirror of the reference's C++ API.

Every call goes through the C-ABI of ``libnpcg_b200.so`` (include/npcg_capi.h),
whose compute runs in hand-written sm_100a CUDA kernels. Names, argument
meaning and error behaviour follow /root/reference/proj/core/include/npcg/:

  reference                                  here
  -----------------------------------------  -----------------------------------
  Rng (random.hpp:21-38)                     Rng
  DenseOperator / GramRidgeOperator /        DenseOperator / GramRidgeOperator /
  KernelOperator / synthesize_operator        KernelOperator / synthesize_operator
  (operators.hpp:50-168)
  make_empty_sketch / extend_sketch /        same names (nystrom.hpp:51-89)
  nystrom_from_sketch / randomized_nystrom
  build_preconditioner,                      build_preconditioner,
  NystromPreconditioner::apply(_inverse)     NystromPreconditioner.apply(_inverse)
  nystrom_pcg / cg (solvers.hpp:60-87)       nystrom_pcg / cg
  estimate_error_power / adaptive_nystrom    estimate_error_power / adaptive
  (adaptive.hpp:56-85)

Exceptions: std::invalid_argument -> InvalidArgument (ValueError),
std::runtime_error -> NpcgRuntimeError (RuntimeError), SolveDivergenceError ->
SolveDivergenceError (carries the partial report). There is no CPU fallback:
if the library or a B200 is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
from contextlib import contextmanager
import os
import threading
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["NPCG_LIB_PATH"]) if os.environ.get("NPCG_LIB_PATH") else PKG / "libnpcg_b200.so"  # override: diagnostics

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
HOST, DEVICE = 0, 1


class InvalidArgument(ValueError):
    """reference std::invalid_argument"""


class NpcgRuntimeError(RuntimeError):
    """reference std::runtime_error"""


class CudaError(RuntimeError):
    """CUDA failure / no B200 device"""


class SolveDivergenceError(RuntimeError):
    """reference npcg::SolveDivergenceError (solvers.hpp:51-57)"""

    def __init__(self, msg, report=None):
        super().__init__(msg)
        self.report = report


class _SolveOpts(C.Structure):
    _fields_ = [("eta", C.c_double), ("max_iter", _i64), ("relative", C.c_int), ("record_iterates", C.c_int)]


class _SolveReport(C.Structure):
    _fields_ = [("iterations", _i64), ("matvec_count", _i64), ("converged", C.c_int), ("status", C.c_int),
                ("eta_used", C.c_double), ("wall_time", C.c_double), ("history_len", _i64)]


class _BlockReport(C.Structure):
    _fields_ = [("iterations", _i64), ("fallback_count", _i64), ("n_deflated", _i64), ("eta_used", C.c_double),
                ("wall_time", C.c_double)]


class _AdaptiveCfg(C.Structure):
    _fields_ = [("ell0", _i64), ("ell_max", _i64), ("mu", C.c_double), ("tol_mode", C.c_int), ("has_tau", C.c_int),
                ("tau", C.c_double), ("q", _i64), ("secondary_criterion", C.c_int), ("sketch", C.c_int)]


class _AdaptiveOutcome(C.Structure):
    _fields_ = [("ell_final", _i64), ("doublings", _i64), ("hit_cap", C.c_int), ("has_error_estimate", C.c_int),
                ("error_estimate", C.c_double), ("posterior_condition", C.c_double)]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libnpcg_b200.so (built in-tree by ``build.py``). Fails loudly."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise CudaError(f"{LIB_PATH} is missing: run `python -m paper_2110_02820_b200.build`")
            L = C.CDLL(str(LIB_PATH))
            L.npcg_last_error.restype = C.c_char_p
            L.npcg_version.restype = C.c_char_p
            L.npcg_rng_normal.restype = C.c_double
            L.npcg_rng_normal.argtypes = [_vp]
            L.npcg_rng_uniform.restype = C.c_double
            L.npcg_rng_uniform.argtypes = [_vp]
            L.npcg_rng_word.restype = C.c_uint64
            L.npcg_rng_word.argtypes = [_vp]
            L.npcg_rng_discard.argtypes = [_vp, C.c_uint64]
            L.npcg_rng_discard.restype = None
            L.npcg_splitmix64.restype = C.c_uint64
            L.npcg_splitmix64.argtypes = [C.c_uint64]
            L.npcg_ulp_spacing.restype = C.c_double
            L.npcg_ulp_spacing.argtypes = [C.c_double]
            L.npcg_ctx_stream.restype = _vp
            L.npcg_ctx_launches.restype = _i64
            L.npcg_ctx_launches.argtypes = [_vp]
            L.npcg_op_kind.argtypes = [_vp]
            L.npcg_op_has_column_access.argtypes = [_vp]
            _lib = L
    return _lib


def _check(rc, report=None):
    if rc == 0:
        return
    msg = lib().npcg_last_error().decode()
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 3:
        raise SolveDivergenceError(msg, report)
    if rc == 4:
        raise CudaError(msg)
    raise NpcgRuntimeError(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ------------------------------------------------------------------ context
class Context:
    """npcg_ctx: one B200, one stream. ``Context.sharded(...)`` /
    ``Context.exchange(...)`` make a row-sharded context (one process per GPU,
    include/npcg_capi.h): every n-vector argument is then this rank's row
    block (``LinearOperator.rows()``)."""

    def __init__(self, device: int = 0, _handle=None):
        if _handle is None:
            h = _vp()
            _check(lib().npcg_ctx_create(C.c_int(device), C.byref(h)))
            _handle = h.value
        self.h = _handle
        self.device = device
        self._keep = None

    @classmethod
    def sharded(cls, device: int, rank: int, world: int, nccl_id: bytes) -> "Context":
        """NCCL data plane created inside the library (ncclCommInitRank)."""
        if len(nccl_id) != 128:
            raise InvalidArgument("Context.sharded: the NCCL unique id is 128 bytes")
        h = _vp()
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().npcg_ctx_create_sharded(C.c_int(device), C.c_int(rank), C.c_int(world), idbuf, C.byref(h)))
        return cls(device, h.value)

    @classmethod
    def exchange(cls, device: int, rank: int, world: int, exchange) -> "Context":
        """Host-callback data plane (``exchange.cfn`` an npcg_exchange_fn, e.g.
        dist.TorchExchange); the exchange object is kept alive with the context."""
        h = _vp()
        _check(lib().npcg_ctx_create_exchange(C.c_int(device), C.c_int(rank), C.c_int(world), exchange.cfn, None,
                                              C.byref(h)))
        ctx = cls(device, h.value)
        ctx._keep = exchange
        return ctx

    def layout(self, n: int) -> tuple[int, int, int, int]:
        """(rank, world, offset, count) of dimension n's row blocks."""
        r, w, off, cnt = C.c_int(), C.c_int(), _i64(), _i64()
        _check(lib().npcg_ctx_layout(_vp(self.h), _i64(n), C.byref(r), C.byref(w), C.byref(off), C.byref(cnt)))
        return r.value, w.value, off.value, cnt.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.npcg_ctx_destroy(_vp(self.h))
            self.h = None

    def sync(self):
        _check(lib().npcg_ctx_sync(_vp(self.h)))

    @property
    def launches(self) -> int:
        return lib().npcg_ctx_launches(_vp(self.h))

    def prof_enable(self, on: bool = True):
        """Per-kernel CUDA-event timing on this context's stream."""
        _check(lib().npcg_prof_enable(_vp(self.h), C.c_int(int(on))))

    def prof_report(self) -> dict:
        """{kernel name: (launches, total_ms, algorithmic flops, algorithmic bytes)}
        since prof_enable(True)."""
        cap = 1 << 20
        while True:
            buf = C.create_string_buffer(cap)
            rc = lib().npcg_prof_report(_vp(self.h), buf, _i64(cap))
            if rc == 0 or cap >= 1 << 28:
                _check(rc)
                break
            cap <<= 2  # many distinct launch labels (e.g. per-shape GEMMs of a long run)
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms, fl, by = line.split("\t")
            out[name] = (int(cnt), float(ms), float(fl), float(by))
        return out

    @property
    def stream(self) -> int:
        return lib().npcg_ctx_stream(_vp(self.h))


_default_ctx = None


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for Context.sharded (rank 0 creates, the host distributes)."""
    buf = C.create_string_buffer(128)
    _check(lib().npcg_nccl_unique_id(buf))
    return buf.raw


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("NPCG_DEVICE", "0")))
    return _default_ctx


# ------------------------------------------------------------------ random
class Rng:
    """reference npcg::Rng (random.hpp:21-38), bitwise: mt19937_64 + Box-Muller."""

    def __init__(self, seed: int = 0, _handle=None):
        if _handle is None:
            h = _vp()
            _check(lib().npcg_rng_create(C.c_uint64(seed), C.byref(h)))
            _handle = h.value
        self.h = _handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.npcg_rng_destroy(_vp(self.h))
            self.h = None

    def clone(self) -> "Rng":
        h = _vp()
        _check(lib().npcg_rng_clone(_vp(self.h), C.byref(h)))
        return Rng(_handle=h.value)

    def normal(self) -> float:
        return lib().npcg_rng_normal(_vp(self.h))

    def uniform(self) -> float:
        return lib().npcg_rng_uniform(_vp(self.h))

    def word(self) -> int:
        return lib().npcg_rng_word(_vp(self.h))

    def discard(self, k: int):
        lib().npcg_rng_discard(_vp(self.h), C.c_uint64(k))

    def integer(self, bound: int) -> int:
        out = C.c_uint64()
        _check(lib().npcg_rng_integer(_vp(self.h), C.c_uint64(bound), C.byref(out)))
        return out.value

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        _check(lib().npcg_rng_gaussian(_vp(self.h), _i64(rows), _i64(cols), _ptr(out)))
        return out

    def gaussian_vector(self, n: int) -> np.ndarray:
        return self.gaussian_matrix(n, 1)[:, 0].copy()

    def _device_buffer(self, ctx, nbytes):
        p = _vp()
        _check(lib().npcg_dev_alloc(_vp(ctx.h), _i64(nbytes), C.byref(p)))
        return p

    def words_device(self, count: int, ctx: "Context | None" = None) -> np.ndarray:
        """`count` engine words generated on the GPU (npcg_rng_words_device), copied to the host."""
        ctx = ctx or default_context()
        buf = self._device_buffer(ctx, 8 * max(count, 1))
        try:
            _check(lib().npcg_rng_words_device(_vp(ctx.h), _vp(self.h), _i64(count), buf))
            out = np.empty(count, dtype=np.uint64)
            _check(lib().npcg_memcpy(_vp(ctx.h), out.ctypes.data_as(_vp), HOST, buf, DEVICE, _i64(8 * count)))
        finally:
            lib().npcg_dev_free(_vp(ctx.h), buf)
        return out

    def gaussian_matrix_device(self, rows: int, cols: int, ctx: "Context | None" = None) -> np.ndarray:
        """gaussian_matrix drawn on the GPU (npcg_rng_gaussian_device), copied to the host."""
        ctx = ctx or default_context()
        buf = self._device_buffer(ctx, 8 * max(rows * cols, 1))
        try:
            _check(lib().npcg_rng_gaussian_device(_vp(ctx.h), _vp(self.h), _i64(rows), _i64(cols), buf,
                                                  _i64(max(rows, 1))))
            out = np.empty((rows, cols), order="F")
            _check(lib().npcg_memcpy(_vp(ctx.h), _ptr(out), HOST, buf, DEVICE, _i64(8 * rows * cols)))
        finally:
            lib().npcg_dev_free(_vp(ctx.h), buf)
        return out

    def uniform_fill(self, count: int) -> np.ndarray:
        out = np.empty(count)
        _check(lib().npcg_rng_uniform_fill(_vp(self.h), _i64(count), _ptr(out)))
        return out

    def sample_without_replacement(self, n: int, k: int) -> np.ndarray:
        out = np.empty(max(k, 0), dtype=np.int64)
        _check(lib().npcg_rng_sample(_vp(self.h), _i64(n), _i64(k), out.ctypes.data_as(C.POINTER(_i64))))
        return out


def splitmix64(seed: int) -> int:
    return lib().npcg_splitmix64(C.c_uint64(seed))


def ulp_spacing(x: float) -> float:
    return lib().npcg_ulp_spacing(float(x))


def orthonormal_columns(g, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    g = _f64(g)
    q = np.empty_like(g, order="F")
    _check(lib().npcg_orthonormal_columns(_vp(ctx.h), _i64(g.shape[0]), _i64(g.shape[1]), _ptr(g), _ptr(q), HOST))
    return q


def gemm(a, b, transa=False, transb=False, alpha=1.0, beta=0.0, c=None, ctx: Context | None = None):
    """alpha op(a) op(b) + beta c on the FP64 DMMA GEMM (npcg_gemm)."""
    ctx = ctx or default_context()
    a, b = _f64(a), _f64(b)
    m, k = (a.shape[1], a.shape[0]) if transa else a.shape
    kb, n = (b.shape[1], b.shape[0]) if transb else b.shape
    if k != kb:
        raise InvalidArgument("gemm: inner dimensions differ")
    out = np.zeros((m, n), order="F") if c is None else _f64(c).copy(order="F")
    _check(lib().npcg_gemm(_vp(ctx.h), _i64(m), _i64(n), _i64(k), C.c_double(alpha), _ptr(a),
                           _i64(max(a.shape[0], 1)), C.c_int(int(transa)), _ptr(b), _i64(max(b.shape[0], 1)),
                           C.c_int(int(not transb)), C.c_double(beta), _ptr(out), _i64(max(m, 1)), HOST))
    return out


def gemm_ozaki(a, b, transa=True, transb=False, ctx: Context | None = None):
    """op(a) @ op(b) on the INT8 tensor cores (digit-plane splitting, FP64
    accuracy; npcg_gemm_ozaki): op(a) = a.T for a (K x M) (K-major), else a
    (M x K); op(b) = b (K x N), or b.T for b (N x K) when transb."""
    ctx = ctx or default_context()
    a, b = _f64(a), _f64(b)
    k, m = a.shape if transa else a.shape[::-1]
    kb, n = b.shape[::-1] if transb else b.shape
    if k != kb:
        raise InvalidArgument("gemm_ozaki: inner dimensions differ")
    out = np.zeros((m, n), order="F")
    _check(lib().npcg_gemm_ozaki(_vp(ctx.h), _i64(m), _i64(n), _i64(k), _ptr(a), _i64(max(a.shape[0], 1)),
                                 C.c_int(int(transa)), _ptr(b), _i64(max(b.shape[0], 1)), C.c_int(int(not transb)),
                                 _ptr(out), _i64(max(m, 1)), HOST))
    return out


def gemm_i8(a8, b8, ctx: Context | None = None):
    """a8 @ b8.T (int8 in, int32 out) on the tcgen05 INT8 GEMM (diagnostics)."""
    ctx = ctx or default_context()
    a8 = np.ascontiguousarray(a8, dtype=np.int8)
    b8 = np.ascontiguousarray(b8, dtype=np.int8)
    m, kp = a8.shape
    n = b8.shape[0]
    out = np.zeros((n, m), dtype=np.int32)  # col-major m x n
    _check(lib().npcg_gemm_i8(_vp(ctx.h), _i64(m), _i64(n), _i64(kp), a8.ctypes.data_as(C.c_void_p),
                              b8.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
    return out.T


def thin_svd(b, ctx: Context | None = None):
    ctx = ctx or default_context()
    b = _f64(b)
    m, n = b.shape
    u = np.empty((m, n), order="F")
    s = np.empty(n)
    _check(lib().npcg_thin_svd(_vp(ctx.h), _i64(m), _i64(n), _ptr(b), _ptr(u), _ptr(s), HOST))
    return u, s


# ------------------------------------------------------------------ operators
class LinearOperator:
    """npcg_op handle: LinearOperator NVI (operators.hpp:25-47) on a B200."""

    def __init__(self, h, ctx: Context):
        self.h, self.ctx = h, ctx

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.npcg_op_destroy(_vp(self.h))
            self.h = None

    def dim(self) -> int:
        n = _i64()
        _check(lib().npcg_op_dim(_vp(self.h), C.byref(n)))
        return n.value

    def rows(self) -> tuple[int, int]:
        """(offset, count) of this rank's row block of every n-vector ((0, n) unsharded)."""
        off, cnt = _i64(), _i64()
        _check(lib().npcg_op_rows(_vp(self.h), C.byref(off), C.byref(cnt)))
        return off.value, cnt.value

    def local_dim(self) -> int:
        return self.rows()[1]

    @property
    def kind(self) -> int:
        return lib().npcg_op_kind(_vp(self.h))

    def has_column_access(self) -> bool:
        return bool(lib().npcg_op_has_column_access(_vp(self.h)))

    def matvec(self, v) -> np.ndarray:
        v = _f64(v).ravel(order="F")
        out = np.empty(self.local_dim())
        _check(lib().npcg_op_apply(_vp(self.h), _i64(v.size), _i64(1), _ptr(v), _i64(max(v.size, 1)), _ptr(out),
                                   _i64(max(out.size, 1)), HOST))
        return out

    def apply_block(self, V) -> np.ndarray:
        V = _f64(V)
        if V.ndim == 1:
            V = V.reshape(-1, 1, order="F")
        rows, k = V.shape
        nl = self.local_dim()
        out = np.empty((nl, k), order="F")
        _check(lib().npcg_op_apply(_vp(self.h), _i64(rows), _i64(k), _ptr(V), _i64(max(rows, 1)), _ptr(out),
                                   _i64(max(nl, 1)), HOST))
        return out

    def column(self, j: int) -> np.ndarray:
        out = np.empty(self.local_dim())
        _check(lib().npcg_op_column(_vp(self.h), _i64(j), _ptr(out), HOST))
        return out

    def dense(self) -> np.ndarray:
        return self.apply_block(np.eye(self.dim()))


def _new_op(ctx, fn, *args) -> LinearOperator:
    h = _vp()
    _check(fn(*args, C.byref(h)))
    return LinearOperator(h.value, ctx)


def DenseOperator(a, ctx: Context | None = None) -> LinearOperator:
    ctx = ctx or default_context()
    a = _f64(a)
    if a.ndim != 2:
        raise InvalidArgument("DenseOperator: matrix must be square")
    return _new_op(ctx, lib().npcg_op_dense_create, _vp(ctx.h), _i64(a.shape[0]), _i64(a.shape[1]), _ptr(a),
                   _i64(max(a.shape[0], 1)), HOST)


def GramRidgeOperator(g, ctx: Context | None = None, streamed: bool = False) -> LinearOperator:
    """operators.cpp:105-121. `streamed=True` (npcg_op_gram_create_streamed):
    the upload of X overlaps the first product (the sketch); the non-finite
    check then raises from that first product instead of the constructor.
    The operator keeps a reference to the host array, which must not be
    modified until then."""
    ctx = ctx or default_context()
    g = _f64(g)
    if g.ndim != 2:
        raise InvalidArgument("GramRidgeOperator: design matrix must be nonempty")
    if streamed:
        op = _new_op(ctx, lib().npcg_op_gram_create_streamed, _vp(ctx.h), _i64(g.shape[0]), _i64(g.shape[1]),
                     _ptr(g), _i64(max(g.shape[0], 1)))
        op._host_ref = g
        return op
    return _new_op(ctx, lib().npcg_op_gram_create, _vp(ctx.h), _i64(g.shape[0]), _i64(g.shape[1]), _ptr(g),
                   _i64(max(g.shape[0], 1)), HOST)


def KernelOperator(points, sigma: float, dense_cap: int = 20000, ctx: Context | None = None) -> LinearOperator:
    ctx = ctx or default_context()
    p = _f64(points)
    if p.ndim == 1:
        p = p.reshape(-1, 1, order="F")
    return _new_op(ctx, lib().npcg_op_kernel_create, _vp(ctx.h), _i64(p.shape[0]), _i64(p.shape[1]), _ptr(p),
                   _i64(max(p.shape[0], 1)), C.c_double(sigma), _i64(dense_cap), HOST)


def synthesize_operator(eigenvalues, seed: int, ctx: Context | None = None) -> LinearOperator:
    ctx = ctx or default_context()
    lam = _f64(eigenvalues).ravel()
    return _new_op(ctx, lib().npcg_op_synthesize, _vp(ctx.h), _i64(lam.size), _ptr(lam), C.c_uint64(seed))


def LowRankOperator(g, lam, ctx: Context | None = None) -> LinearOperator:
    """A = G diag(lam) G^T / r (BASELINE config 5 generator), built on device."""
    ctx = ctx or default_context()
    g = _f64(g)
    lam = _f64(lam).ravel()
    return _new_op(ctx, lib().npcg_op_lowrank_create, _vp(ctx.h), _i64(g.shape[0]), _i64(g.shape[1]), _ptr(g),
                   _i64(g.shape[0]), _ptr(lam), HOST)


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                       C.c_void_p)
COLUMN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class UserOperator:
    """The reference's plug-in point (operators.hpp:25-47, NVI): subclass and
    implement ``do_dim`` and ``do_matvec`` (optionally ``do_apply_block``,
    ``has_column_access`` + ``do_column``). Every solver entry point accepts
    it; the library calls back into it through npcg_op_callback_create."""

    def dim(self) -> int:
        return int(self.do_dim())

    def matvec(self, v) -> np.ndarray:  # operators.cpp:25-30
        v = np.asarray(v, dtype=np.float64)
        if v.shape != (self.dim(),):
            raise InvalidArgument(f"LinearOperator - matvec: dimension mismatch (got {v.size}, operator dim "
                                  f"{self.dim()})")
        if not np.all(np.isfinite(v)):
            raise InvalidArgument("LinearOperator - matvec: input has non-finite entries")
        return np.asarray(self.do_matvec(v), dtype=np.float64)

    def apply_block(self, V) -> np.ndarray:  # operators.cpp:32-40
        V = np.asarray(V, dtype=np.float64)
        if V.ndim != 2 or V.shape[0] != self.dim():
            raise InvalidArgument("LinearOperator - apply_block: dimension mismatch")
        if not np.all(np.isfinite(V)):
            raise InvalidArgument("LinearOperator - apply_block: input has non-finite entries")
        return np.asarray(self.do_apply_block(V), dtype=np.float64)

    def has_column_access(self) -> bool:
        return False

    def column(self, j: int) -> np.ndarray:  # operators.cpp:42-50
        if not self.has_column_access():
            raise NpcgRuntimeError("LinearOperator - column: operator has no column access")
        if not 0 <= j < self.dim():
            raise InvalidArgument("LinearOperator - column: index out of range")
        return np.asarray(self.do_column(j), dtype=np.float64)

    def do_apply_block(self, V):  # operators.cpp:52-58: one do_matvec per column
        return np.column_stack([self.do_matvec(V[:, j]) for j in range(V.shape[1])]) if V.shape[1] else \
            np.empty((self.dim(), 0))

    def do_column(self, j):
        raise NpcgRuntimeError("LinearOperator - column: operator has no column access")


class _CallbackBinding:
    """A user operator bound to the C-ABI for one library call (host buffers).
    An exception raised by the operator is kept and re-raised by _bound()."""

    def __init__(self, op, ctx=None):
        self.op, self.error = op, None
        ctx = ctx or default_context()
        self._apply = APPLY_FN(self._apply_cb)
        self._column = COLUMN_FN(self._column_cb) if op.has_column_access() else None
        h = _vp()
        _check(lib().npcg_op_callback_create(_vp(ctx.h), _i64(op.dim()), self._apply,
                                             self._column if self._column else COLUMN_FN(), None, HOST, C.byref(h)))
        self.h = h.value

    def _apply_cb(self, user, n, k, v, ldv, out, ldo, stream):
        try:
            V = np.ctypeslib.as_array(C.cast(v, C.POINTER(C.c_double)), shape=(k, ldv)).T[:n, :]
            O = np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_double)), shape=(k, ldo)).T[:n, :]
            if k == 1:
                O[:, 0] = self.op.matvec(V[:, 0].copy())
            else:
                O[:, :] = self.op.apply_block(np.asfortranarray(V))
            return 0
        except BaseException as e:  # noqa: BLE001 - carried across the C boundary
            self.error = e
            return 1

    def _column_cb(self, user, j, out, stream):
        try:
            n = self.op.dim()
            np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_double)), shape=(n,))[:] = self.op.column(int(j))
            return 0
        except BaseException as e:  # noqa: BLE001
            self.error = e
            return 1

    def close(self):
        if self.h:
            lib().npcg_op_destroy(_vp(self.h))
            self.h = None


@contextmanager
def _bound(op):
    """The device handle a library call runs on: the operator's own, or a
    callback operator around a user operator for the duration of the call."""
    if isinstance(op, LinearOperator):
        yield op.h
        return
    if not hasattr(op, "matvec") or not hasattr(op, "dim"):
        raise InvalidArgument("npcg: operator must be a LinearOperator or provide dim()/matvec()")
    b = _CallbackBinding(op)
    try:
        yield b.h
    except (NpcgRuntimeError, InvalidArgument, CudaError, SolveDivergenceError):
        if b.error is not None:
            raise b.error from None
        raise
    finally:
        b.close()


class RegularizedOperator(LinearOperator):
    """RegularizedOperator(base, mu) (operators.hpp:69-94; operators.cpp:82-103):
    A_mu v = base v; += mu v. Over a device operator this is a device operator
    (npcg_op_regularize): cg(regularize(op, mu), b) runs the same fused kernels
    as nystrom_pcg(op, b, mu, None). Over a user operator it evaluates on the
    host through the base's NVI (and is bound by callback like any user op)."""

    def __init__(self, base, mu: float):
        if base is None:
            raise InvalidArgument("RegularizedOperator: base operator is null")
        if not mu >= 0.0:
            raise InvalidArgument("RegularizedOperator: mu must be >= 0")
        self.base, self.mu = base, float(mu)
        if isinstance(base, LinearOperator):
            h = _vp()
            _check(lib().npcg_op_regularize(_vp(base.h), C.c_double(mu), C.byref(h)))
            super().__init__(h.value, base.ctx)
        else:
            self.h, self.ctx = None, None
            self._user = _RegularizedUser(base, self.mu)

    def dim(self) -> int:
        return self.base.dim()

    def local_dim(self) -> int:
        return super().local_dim() if self.h else self.base.dim()

    def has_column_access(self) -> bool:
        return False

    def matvec(self, v):
        return super().matvec(v) if self.h else self._user.matvec(v)

    def apply_block(self, V):
        return super().apply_block(V) if self.h else self._user.apply_block(V)


class _RegularizedUser(UserOperator):
    def __init__(self, base, mu):
        self.base, self.mu = base, mu

    def do_dim(self):
        return self.base.dim()

    def do_matvec(self, v):
        out = np.array(self.base.matvec(v), dtype=np.float64)
        out += self.mu * v
        return out

    def do_apply_block(self, V):
        out = np.array(self.base.apply_block(V), dtype=np.float64)
        out += self.mu * V
        return out


def regularize(op, mu: float) -> RegularizedOperator:
    """regularize(op, mu) (operators.hpp:153; operators.cpp:201-203)."""
    return RegularizedOperator(op, mu)


def _unwrap(op):
    """RegularizedOperator over a user operator binds as that user operator."""
    if isinstance(op, RegularizedOperator) and op.h is None:
        return op._user
    return op


# ------------------------------------------------------------------ Nyström
class _Nys:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.npcg_nys_destroy(_vp(self.h))
            self.h = None


class NystromApproximation:
    """reference NystromApproximation (nystrom.hpp:19-33). The factors live on
    the device (a factors-only npcg_nys handle, immutable); `lam` is mirrored
    on construction, `u` is downloaded on first access only."""

    def __init__(self, u, lam, shift_used, h=None, n=None):
        self._u, self.lam, self.shift_used, self.h = u, lam, shift_used, h
        self._n = n if n is not None else (u.shape[0] if u is not None else 0)

    @property
    def u(self) -> np.ndarray:
        if self._u is None:
            e = self.lam.size
            u = np.empty((self._n, e), order="F")
            if e:
                _check(lib().npcg_nys_get(_vp(self.h.h), None, _ptr(u), _i64(max(self._n, 1)), HOST))
            self._u = u
        return self._u

    @property
    def lambda_min(self):
        return float(self.lam[-1]) if self.lam.size else 0.0

    def dim(self):
        return self._n

    def size(self):
        return int(self.lam.size)

    def rank(self):
        return int(np.count_nonzero(self.lam > 0))

    def materialize(self):
        return (self.u * self.lam) @ self.u.T


def _clone(nys: "_Nys", factors_only: bool) -> "_Nys":
    h = _vp()
    _check(lib().npcg_nys_clone(_vp(nys.h), int(factors_only), C.byref(h)))
    return _Nys(h.value)


def _nys_rows(nys: "_Nys") -> int:
    off, cnt = _i64(), _i64()
    _check(lib().npcg_nys_rows(_vp(nys.h), C.byref(off), C.byref(cnt)))
    return cnt.value


def _approx_from(nys: _Nys) -> NystromApproximation:
    """The factored approximation of `nys` as an independent value: a
    factors-only handle (later extends / refactors of the pair leave it
    unchanged); U stays on the device until `.u` is read."""
    n, size, ell, shift = _i64(), _i64(), _i64(), C.c_double()
    _check(lib().npcg_nys_info(_vp(nys.h), C.byref(n), C.byref(size), C.byref(ell), C.byref(shift)))
    e = max(ell.value, 0)
    lam = np.empty(e)
    _check(lib().npcg_nys_get(_vp(nys.h), _ptr(lam), None, _i64(max(n.value, 1)), HOST))
    return NystromApproximation(None, lam, shift.value, _clone(nys, True), _nys_rows(nys))


class SketchPair:
    """reference SketchPair (nystrom.hpp:42-48): device-resident (omega, y)."""

    def __init__(self, nys: _Nys, op: LinearOperator):
        self._nys, self.op = nys, op

    @property
    def h(self):
        return self._nys.h

    def size(self) -> int:
        size = _i64()
        _check(lib().npcg_nys_info(_vp(self.h), None, C.byref(size), None, None))
        return size.value

    def arrays(self, n=None):
        n = _nys_rows(self._nys)  # this rank's rows (all n unsharded)
        k = self.size()
        om = np.empty((n, k), order="F")
        y = np.empty((n, k), order="F")
        _check(lib().npcg_nys_get_sketch(_vp(self.h), _ptr(om), _ptr(y), _i64(max(n, 1)), HOST))
        return om, y


def make_empty_sketch(n_or_op, op: LinearOperator | None = None) -> "SketchPair | _PendingSketch":
    """make_empty_sketch(n) (nystrom.cpp:28-34). The device sketch binds to its
    operator at the first extend_sketch call."""
    if not np.isscalar(n_or_op):  # an operator (device, regularized or user)
        op = n_or_op
    if op is not None:
        h = _vp()
        with _bound(_unwrap(op)) as oh:
            _check(lib().npcg_nys_create(_vp(oh), C.byref(h)))
        return SketchPair(_Nys(h.value), op)
    n = int(n_or_op)
    if n < 1:
        raise InvalidArgument("make_empty_sketch: dimension must be positive")
    return _PendingSketch(n)


class _PendingSketch:
    def __init__(self, n):
        self.n = n

    def size(self):
        return 0


def _fresh_pair(pair, op, what):
    """The pair a non-mutating extend writes into: an empty sketch bound to
    `op`, or an O(1) copy-on-append clone of `pair` (the input stays as it was,
    as the reference's extend_sketch returns a new SketchPair)."""
    if isinstance(pair, _PendingSketch):
        if pair.n != op.dim():
            raise InvalidArgument(f"{what}: dimension mismatch")
        return make_empty_sketch(op)
    if pair.op.dim() != op.dim():
        raise InvalidArgument(f"{what}: dimension mismatch")
    return SketchPair(_clone(pair._nys, False), op)


def extend_sketch(pair, op: LinearOperator, extra: int, rng: Rng) -> SketchPair:
    """extend_sketch (nystrom.cpp:36-58): returns a new pair; `pair` is left
    unchanged (device storage is shared copy-on-append)."""
    out = _fresh_pair(pair, op, "extend_sketch")
    with _bound(_unwrap(op)) as oh:  # the reference passes op to every extend (nystrom.cpp:36)
        _check(lib().npcg_nys_bind(_vp(out.h), _vp(oh)))
        _check(lib().npcg_nys_extend_rng(_vp(out.h), _i64(extra), _vp(rng.h)))
    return out


def extend_sketch_with(pair, op: LinearOperator, fresh) -> SketchPair:
    """extend_sketch with a caller-drawn raw Gaussian block (n x extra)."""
    out = _fresh_pair(pair, op, "extend_sketch")
    fresh = _f64(fresh)
    with _bound(_unwrap(op)) as oh:
        _check(lib().npcg_nys_bind(_vp(out.h), _vp(oh)))
        _check(lib().npcg_nys_extend(_vp(out.h), _i64(fresh.shape[1]), _ptr(fresh), _i64(fresh.shape[0]), HOST))
    return out


def extend_sketch_columns(pair, op: LinearOperator, extra: int, used: list, rng: Rng) -> SketchPair:
    """extend_sketch_columns (nystrom.cpp:60-94): appends `extra` unused columns of A
    drawn from `rng`; `used` is extended in place (the handle keeps its own copy).
    Returns a new pair; `pair` is left unchanged."""
    pair = _fresh_pair(pair, op, "extend_sketch_columns")
    with _bound(_unwrap(op)) as oh:
        _check(lib().npcg_nys_bind(_vp(pair.h), _vp(oh)))
        _check(lib().npcg_nys_extend_columns(_vp(pair.h), _i64(extra), _vp(rng.h)))
    cnt = _i64()
    _check(lib().npcg_nys_used(_vp(pair.h), None, C.byref(cnt)))
    buf = np.zeros(max(cnt.value, 1), dtype=np.int64)
    _check(lib().npcg_nys_used(_vp(pair.h), buf.ctypes.data_as(_vp), C.byref(cnt)))
    used[:] = [int(v) for v in buf[:cnt.value]]
    return pair


def column_sampling_nystrom(op: LinearOperator, ell_or_indices, rng: Rng | None = None) -> "NystromApproximation":
    """column_sampling_nystrom (nystrom.cpp:150-184): `ell` columns drawn from
    `rng`, or the caller's distinct indices."""
    h = _vp()
    with _bound(_unwrap(op)) as oh:
        if rng is not None:
            _check(lib().npcg_column_sampling_nystrom(_vp(oh), _i64(int(ell_or_indices)), None, _vp(rng.h),
                                                      C.byref(h)))
        else:
            idx = np.ascontiguousarray(ell_or_indices, dtype=np.int64)
            _check(lib().npcg_column_sampling_nystrom(_vp(oh), _i64(idx.size), idx.ctypes.data_as(_vp), None,
                                                      C.byref(h)))
    return _approx_from(_Nys(h.value))


def nystrom_from_sketch(pair: SketchPair) -> NystromApproximation:
    """nystrom_from_sketch (nystrom.cpp:96-140), factored on device."""
    _check(lib().npcg_nys_factor(_vp(pair.h)))
    return _approx_from(pair._nys)


def randomized_nystrom(op: LinearOperator, ell: int, rng: Rng) -> NystromApproximation:
    """randomized_nystrom (nystrom.cpp:142-148)."""
    n = op.dim()
    if ell < 1 or ell > n:
        raise InvalidArgument("randomized_nystrom: need 1 <= ell <= dim")
    pair = extend_sketch(make_empty_sketch(op), op, ell, rng)
    return nystrom_from_sketch(pair)


def make_approximation(u, lam, shift_used=0.0, ctx: Context | None = None, n: int | None = None) -> NystromApproximation:
    """An approximation from its factors; on a sharded context `u` is this
    rank's row block and `n` the full dimension."""
    ctx = ctx or default_context()
    u = _f64(u)
    lam = _f64(lam).ravel()
    n, ell = (u.shape[0] if n is None else int(n)), lam.size
    h = _vp()
    _check(lib().npcg_nys_from_factors(_vp(ctx.h), _i64(n), _i64(ell), _ptr(u) if ell else None, _i64(max(n, 1)),
                                       _ptr(lam) if ell else None, C.c_double(shift_used), HOST, C.byref(h)))
    return NystromApproximation(u.reshape(u.shape[0], ell), lam, shift_used, _Nys(h.value), u.shape[0])


# ------------------------------------------------------------------ preconditioner
class NystromPreconditioner:
    """npcg_pre: NystromPreconditioner (preconditioner.hpp:20-37) on device."""

    def __init__(self, h, approx: NystromApproximation, mu: float):
        self.h, self.approx, self.mu = h, approx, mu
        self.n = approx.dim()
        self.lambda_ell = approx.lambda_min

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.npcg_pre_destroy(_vp(self.h))
            self.h = None

    def _apply(self, fn, r):
        r = _f64(r)
        s = 1 if r.ndim == 1 else r.shape[1]
        out = np.empty(r.shape, order="F")
        _check(fn(_vp(self.h), _i64(s), _ptr(r), _i64(max(r.shape[0], 1)), _ptr(out), _i64(max(r.shape[0], 1)), HOST))
        return out

    def apply_inverse(self, r) -> np.ndarray:
        r = np.asarray(r)
        if r.shape[0] != self.n:
            raise InvalidArgument("NystromPreconditioner - apply_inverse: length mismatch")
        return self._apply(lib().npcg_pre_apply_inverse, r)

    def apply(self, v) -> np.ndarray:
        v = np.asarray(v)
        if v.shape[0] != self.n:
            raise InvalidArgument("NystromPreconditioner - apply: length mismatch")
        return self._apply(lib().npcg_pre_apply, v)


def build_preconditioner(approx: NystromApproximation, mu: float) -> NystromPreconditioner:
    """build_preconditioner (preconditioner.cpp:80-89)."""
    h = _vp()
    _check(lib().npcg_pre_create(_vp(approx.h.h), C.c_double(mu), C.byref(h)))
    return NystromPreconditioner(h.value, approx, mu)


def woodbury_inverse_apply(approx: NystromApproximation, mu: float, b) -> np.ndarray:
    """woodbury_inverse_apply (preconditioner.cpp:104-114) on the device factors:
    (U diag(lambda) U^T + mu I)^-1 b."""
    b = _f64(b)
    single = b.ndim == 1
    B = b.reshape(-1, 1, order="F") if single else b
    out = np.empty(B.shape, order="F")
    _check(lib().npcg_woodbury_inverse_apply(_vp(approx.h.h), C.c_double(mu), _i64(B.shape[1]), _ptr(B),
                                             _i64(max(B.shape[0], 1)), _ptr(out), _i64(max(B.shape[0], 1)), HOST))
    return out[:, 0].copy() if single else out


def sketch_and_solve(op, b, mu: float, ell: int, rng: "Rng") -> np.ndarray:
    """sketch_and_solve (preconditioner.cpp:116-121)."""
    if not mu > 0.0:
        raise InvalidArgument("sketch_and_solve: mu must be > 0")
    return woodbury_inverse_apply(randomized_nystrom(op, ell, rng), mu, b)


# ------------------------------------------------------------------ solvers
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
    status: int = 0


def _pcg(op, pre, mu, B, eta, max_iter, relative, record_iterates, x0):
    B = _f64(B)
    single = B.ndim == 1
    if single:
        B = B.reshape(-1, 1, order="F")
    n, s = B.shape
    if n != (op.local_dim() if isinstance(op, LinearOperator) else op.dim()):
        raise InvalidArgument("nystrom_pcg: right-hand side length mismatch")
    if x0 is not None:
        x0 = _f64(x0).reshape(n, s, order="F")
        if x0.shape[0] != n:
            raise InvalidArgument("nystrom_pcg: initial guess length mismatch")
    X = np.empty((n, s), order="F")
    reps = (_SolveReport * s)()
    hist = np.zeros((max(max_iter, 0) + 1, s), order="F")
    its = np.zeros(((max_iter + 1) * n * s,)) if record_iterates else None
    opts = _SolveOpts(float(eta), int(max_iter), int(bool(relative)), int(bool(record_iterates)))
    with _bound(_unwrap(op)) as oh:
        rc = lib().npcg_pcg(_vp(oh), None if pre is None else _vp(pre.h), C.c_double(mu), _i64(s), _ptr(B),
                            _i64(n), _ptr(x0), _i64(n), C.byref(opts), _ptr(X), _i64(n), reps, _ptr(hist), _ptr(its),
                            HOST)
        if rc not in (0, 3):
            _check(rc)
    out = []
    for j in range(s):
        r = reps[j]
        iters = None
        if its is not None:
            full = its.reshape(max_iter + 1, s, n)
            iters = full[: r.history_len, j, :].copy()
        out.append(SolveReport(X[:, j].copy(), r.iterations, hist[: r.history_len, j].copy(), bool(r.converged),
                               r.matvec_count, r.wall_time, r.eta_used, iters, r.status))
    if rc != 0:
        bad = next((o for o in out if o.status != 0), out[0])
        _check(rc, bad if single or rc == 3 else None)
    return out[0] if single else out


def nystrom_pcg(op: LinearOperator, b, mu: float, precond: NystromPreconditioner | None, eta=1e-10, max_iter=500,
                relative=False, record_iterates=False, x0=None):
    """nystrom_pcg (solvers.cpp:122-148). `b` may be n x s: s independent
    solves sharing each pass over A (returns a list of reports)."""
    if precond is None:  # empty preconditioner == identity
        return _pcg(op, None, mu, b, eta, max_iter, relative, record_iterates, x0)
    return _pcg(op, precond, mu, b, eta, max_iter, relative, record_iterates, x0)


def cg(op, *args, eta=1e-10, max_iter=500, relative=False, x0=None):
    """cg (solvers.cpp:111-120): ``cg(op_mu, b[, x0])`` on an spd operator --
    typically regularize(op, mu), as the reference bench calls it
    (bench.cpp:218-220) -- or the shorthand ``cg(op, mu, b)`` on op + mu I."""
    if len(args) >= 1 and np.ndim(args[0]) == 0:
        mu, rest = float(args[0]), args[1:]
    else:
        mu, rest = 0.0, args
    if not rest:
        raise InvalidArgument("cg: right-hand side missing")
    b = rest[0]
    if len(rest) > 1:
        x0 = rest[1]
    return _pcg(op, None, mu, b, eta, max_iter, relative, False, x0)


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
    """block_nystrom_pcg (solvers.cpp:150-279), 1 <= s <= 32 columns."""
    B = _f64(B)
    n, s = B.shape
    X = np.empty((n, s), order="F")
    rep = _BlockReport()
    conv = (C.c_int * s)()
    defl = (_i64 * s)()
    fres = np.empty(s)
    hist = np.zeros((max_iter + 1, s), order="F")
    hlen = np.zeros(s, dtype=np.int64)
    opts = _SolveOpts(float(eta), int(max_iter), int(bool(relative)), 0)
    with _bound(_unwrap(op)) as h:
        _check(lib().npcg_block_pcg(_vp(h), None if precond is None else _vp(precond.h), C.c_double(mu), _i64(s),
                                    _ptr(B), _i64(n), C.byref(opts), _ptr(X), _i64(n), C.byref(rep), conv, defl,
                                    _ptr(fres), _ptr(hist), hlen.ctypes.data_as(_vp), HOST))
    return BlockSolveReport(X, rep.iterations, [bool(c) for c in conv], list(defl[: rep.n_deflated]),
                            rep.fallback_count, fres, [hist[: hlen[j], j].copy() for j in range(s)])


def regularization_path(op: LinearOperator, B, mus, approx: NystromApproximation, warm_start: bool = True,
                        eta=1e-10, max_iter=500, relative=True):
    """One Nystrom approximation reused along a regularisation path
    (npcg_regularization_path): for each mu in order the
    preconditioner is rebuilt and the right-hand sides solved, warm-started
    from the previous mu's solutions. Returns [(mu, [SolveReport per column])]."""
    B = _f64(B)
    if B.ndim == 1:
        B = B.reshape(-1, 1, order="F")
    n, s = B.shape
    mus = np.ascontiguousarray(mus, dtype=np.float64)
    nmu = mus.size
    X = np.empty((n, s * nmu), order="F")
    reps = (_SolveReport * (s * nmu))()
    opts = _SolveOpts(float(eta), int(max_iter), int(bool(relative)), 0)
    with _bound(_unwrap(op)) as oh:
        _check(lib().npcg_regularization_path(_vp(oh), _vp(approx.h.h), _i64(nmu), _ptr(mus), _i64(s), _ptr(B),
                                              _i64(n), C.byref(opts), C.c_int(int(warm_start)), _ptr(X), _i64(n),
                                              reps, HOST))
    out = []
    for k in range(nmu):
        cols = []
        for j in range(s):
            r = reps[k * s + j]
            cols.append(SolveReport(X[:, k * s + j].copy(), r.iterations, np.empty(0), bool(r.converged),
                                    r.matvec_count, r.wall_time, r.eta_used, None, r.status))
        out.append((float(mus[k]), cols))
    return out


def iteration_bound(kappa: float, eps: float) -> int:
    out = _i64()
    _check(lib().npcg_iteration_bound(C.c_double(kappa), C.c_double(eps), C.byref(out)))
    return out.value


# ------------------------------------------------------------------ adaptive
def estimate_error_power(op: LinearOperator, approx: NystromApproximation, q: int, rng: Rng) -> float:
    """estimate_error_power (adaptive.cpp:83-109)."""
    out = C.c_double()
    with _bound(_unwrap(op)) as oh:
        _check(lib().npcg_power_estimate_rng(_vp(oh), _vp(approx.h.h), _i64(q), _vp(rng.h), C.byref(out)))
    return out.value


@dataclass
class AdaptiveOutcome:
    approximation: NystromApproximation
    error_estimate: float | None
    doublings: int
    hit_cap: bool
    posterior_condition_estimate: float
    ell_final: int


def adaptive(op, rng: Rng, *, mode="error", ell0=10, ell_max=0, mu=0.0, tau=None, q=5, secondary_criterion=True,
             sketch="gaussian") -> AdaptiveOutcome:
    """adaptive_nystrom (mode='error'), adaptive_nystrom_ratio ('ratio'),
    fixed_rank_nystrom ('fixed') — adaptive.cpp:50-148."""
    modes = {"error": 0, "ratio": 1, "fixed": 2}
    cfg = _AdaptiveCfg(int(ell0), int(ell_max), float(mu), modes[mode], int(tau is not None), float(tau or 0.0),
                       int(q), int(bool(secondary_criterion)), 0 if sketch == "gaussian" else 1)
    out = _AdaptiveOutcome()
    h = _vp()
    with _bound(_unwrap(op)) as oh:
        _check(lib().npcg_adaptive(_vp(oh), C.byref(cfg), _vp(rng.h), C.byref(h), C.byref(out)))
    approx = _approx_from(_Nys(h.value))
    return AdaptiveOutcome(approx, out.error_estimate if out.has_error_estimate else None, out.doublings,
                           bool(out.hit_cap), out.posterior_condition, out.ell_final)


def adaptive_nystrom(op, config: dict, rng: Rng) -> AdaptiveOutcome:
    return adaptive(op, rng, mode="error", **config)


def posterior_condition_estimate(lam_ell, mu, err) -> float:
    out = C.c_double()
    _check(lib().npcg_posterior_condition(C.c_double(lam_ell), C.c_double(mu), C.c_double(err), C.byref(out)))
    return out.value
