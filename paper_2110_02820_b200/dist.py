"""Multi-GPU plumbing for the row-sharded operators.

One process per GPU. The operator is split by rows and every vector (p, r,
x, Ω, Y, U) stays replicated, so the only communication of a solve is the
exchange that completes each operator product:

* Gram (ridge): rank g holds the row block X_g; A v = Σ_g X_gᵀ(X_g v)/m is an
  in-place all-reduce of n doubles per right-hand side.
* Dense / stored kernel: rank g holds the column block A[:, R_g] (= rows R_g,
  A symmetric); A v is an all-gather of ceil(n/G) doubles per rank.

The library enqueues the exchange through a C callback on its own stream
(``npcg_exchange_fn`` in include/npcg_capi.h); :class:`TorchExchange` binds it
to ``torch.distributed`` — NCCL over NVLink on B200s, gloo in the CPU tests.
Factorisation and preconditioner are replicated and deterministic, so every
rank holds bitwise-identical scalars and takes the same convergence branch.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

ALLREDUCE, ALLGATHER = 0, 1


def block_size(total: int, nranks: int) -> int:
    """Rows per rank: equal blocks of ceil(total / nranks), the last one short
    (the layout npcg_op_dense_shard_create assumes)."""
    return -(-total // nranks)


def shard_rows(total: int, nranks: int, rank: int) -> tuple[int, int]:
    """(offset, count) of `rank`'s contiguous row block."""
    if not 0 <= rank < nranks:
        raise ValueError("shard_rows: rank out of range")
    nb = block_size(total, nranks)
    off = min(total, rank * nb)
    return off, max(0, min(nb, total - off))


def unpack_gathered(recv: np.ndarray, n: int, nranks: int, k: int) -> np.ndarray:
    """Host restatement of the library's unpack_gather_kernel: rank-major
    blocks of nb x k (col-major) -> n x k."""
    nb = block_size(n, nranks)
    blocks = recv.reshape(nranks, k, nb)
    out = np.empty((n, k), order="F")
    for r in range(nranks):
        off, cnt = shard_rows(n, nranks, r)
        out[off:off + cnt, :] = blocks[r, :, :cnt].T
    return out


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


class TorchExchange:
    """Completes sharded operator products with torch.distributed collectives.

    ``exchange()`` works on torch tensors (CPU tensors + gloo in the tests);
    ``cfn`` is the C callback the library calls with device pointers and its
    stream: the collective is enqueued with that stream as torch's current
    stream, so it is ordered with the library's kernels and no host sync occurs.
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.errors: list[BaseException] = []
        self.calls = 0
        self.cfn = EXCHANGE_FN(self._call)

    def exchange(self, kind: int, send, recv) -> None:
        if kind == ALLREDUCE:
            self.dist.all_reduce(send, group=self.group)
        elif kind == ALLGATHER:
            count = send.numel()
            self.dist.all_gather(list(recv.view(self.world, count).unbind(0)), send, group=self.group)
        else:
            raise ValueError(f"unknown exchange kind {kind}")

    def _call(self, user, kind, send, recv, count, stream) -> int:
        try:
            import torch
            s = torch.cuda.ExternalStream(stream)
            with torch.cuda.stream(s):
                st = torch.as_tensor(_DevView(send, count), device="cuda")
                rt = st if kind == ALLREDUCE else torch.as_tensor(_DevView(recv, count * self.world), device="cuda")
                self.exchange(kind, st, rt)
            self.calls += 1
            return 0
        except BaseException as e:  # noqa: BLE001 - reported through the library's status code
            self.errors.append(e)
            return 1


def ShardedGramOperator(x_local, m_total: int, exchange: TorchExchange, ctx=None, where=None, ld=None):
    """GramRidgeOperator over this rank's row block X_g (m_local x n) of a
    design with m_total rows (npcg_op_gram_shard_create). `x_local` is a host
    array, or a device pointer with `where=DEVICE`, `ld` and shape given by
    (m_local, n) in `x_local` as a tuple (ptr, m_local, n)."""
    from . import DEVICE, HOST, _check, _f64, _i64, _ptr, _vp, default_context, lib, LinearOperator
    ctx = ctx or default_context()
    h = _vp()
    if where == DEVICE:
        ptr, m_local, n = x_local
        _check(lib().npcg_op_gram_shard_create(_vp(ctx.h), _i64(m_local), _i64(n), _vp(ptr), _i64(ld), DEVICE,
                                               _i64(m_total), exchange.cfn, None, C.byref(h)))
    else:
        x = _f64(x_local)
        _check(lib().npcg_op_gram_shard_create(_vp(ctx.h), _i64(x.shape[0]), _i64(x.shape[1]), _ptr(x),
                                               _i64(max(x.shape[0], 1)), HOST, _i64(m_total), exchange.cfn, None,
                                               C.byref(h)))
    op = LinearOperator(h.value, ctx)
    op._exchange = exchange  # keep the callback alive with the handle
    return op


def ShardedDenseOperator(a_block, n: int, exchange: TorchExchange, ctx=None):
    """DenseOperator over this rank's column block A[:, R_g] (n x nloc) of a
    symmetric n x n A (npcg_op_dense_shard_create)."""
    from . import HOST, _check, _f64, _i64, _ptr, _vp, default_context, lib, LinearOperator
    ctx = ctx or default_context()
    a = _f64(a_block)
    off, cnt = shard_rows(n, exchange.world, exchange.rank)
    if a.shape != (n, cnt):
        raise ValueError(f"ShardedDenseOperator: expected the {n} x {cnt} column block at {off}")
    h = _vp()
    _check(lib().npcg_op_dense_shard_create(_vp(ctx.h), _i64(n), _i64(exchange.world), _i64(exchange.rank),
                                            _ptr(a), _i64(max(n, 1)), HOST, exchange.cfn, None, C.byref(h)))
    op = LinearOperator(h.value, ctx)
    op._exchange = exchange
    return op


def ShardedKernelOperator(points, sigma: float, exchange: TorchExchange, ctx=None):
    """Stored Gaussian KernelOperator over this rank's column block K[:, R_g],
    built on device from all n points (npcg_op_kernel_shard_create)."""
    from . import HOST, _check, _f64, _i64, _ptr, _vp, default_context, lib, LinearOperator
    ctx = ctx or default_context()
    p = _f64(points)
    n, d = p.shape
    h = _vp()
    _check(lib().npcg_op_kernel_shard_create(_vp(ctx.h), _i64(n), _i64(d), _ptr(p), _i64(max(n, 1)),
                                             C.c_double(sigma), _i64(exchange.world), _i64(exchange.rank), HOST,
                                             exchange.cfn, None, C.byref(h)))
    op = LinearOperator(h.value, ctx)
    op._exchange = exchange
    return op


def ShardedLowRankOperator(g, lam, exchange: TorchExchange, ctx=None):
    """A = G diag(lam) G^T / r over this rank's column block (npcg_op_lowrank_shard_create)."""
    from . import HOST, _check, _f64, _i64, _ptr, _vp, default_context, lib, LinearOperator
    ctx = ctx or default_context()
    g = _f64(g)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    n, r = g.shape
    h = _vp()
    _check(lib().npcg_op_lowrank_shard_create(_vp(ctx.h), _i64(n), _i64(r), _ptr(g), _i64(max(n, 1)), _ptr(lam),
                                              _i64(exchange.world), _i64(exchange.rank), HOST, exchange.cfn, None,
                                              C.byref(h)))
    op = LinearOperator(h.value, ctx)
    op._exchange = exchange
    return op
