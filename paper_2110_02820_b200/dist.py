"""Multi-GPU plumbing: row-sharded contexts, one process per GPU.

On a sharded context (include/npcg_capi.h) every dimension n is split into
balanced contiguous row blocks R_g and every n-length object of the path --
Omega, Y, U, x, r, z, p, the right-hand sides -- lives on its owner as the local
row block. The library itself issues the exchanges from C++ on its stream:

* all-gather of p before each operator product (and of each sketch block);
* sum all-reduce of the row reductions: Omega^T Y_nu and the CholeskyQR /
  Gram-Schmidt Grams (l x l), ||Y||_F, U^T r (l), the PCG dots;
* reduce-scatter of full-length partial products (Gram ridge over a row
  block of X; the symmetric matrix-free kernel's share of block pairs).

Production: :func:`nccl_context` -- NCCL inside the library (the unique id
travels over torch.distributed once; no Python on the per-iteration path).
Tests: :func:`exchange_context` with :class:`TorchExchange` -- a host-staged
callback transport over torch.distributed (gloo): the library synchronises its
stream, the callback copies the block to the host, runs the collective on CPU
tensors and copies the result back, so ranks sharing one GPU never wait on
each other inside a kernel.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

ALLREDUCE, ALLGATHER, REDUCE_SCATTER = 0, 1, 2


def shard_rows(total: int, nranks: int, rank: int) -> tuple[int, int]:
    """(offset, count) of `rank`'s balanced contiguous row block (comm.cuh RowSplit):
    floor(total / nranks) rows, one more for the first total % nranks ranks."""
    if not 0 <= rank < nranks:
        raise ValueError("shard_rows: rank out of range")
    q, r = divmod(total, nranks)
    return rank * q + min(rank, r), q + (1 if rank < r else 0)


def nccl_context(device: int, group=None):
    """A row-sharded npcg Context over NCCL for this process's rank of the
    torch.distributed group (rank 0 creates the NCCL unique id)."""
    import torch.distributed as dist
    import paper_2110_02820_b200 as npcg
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [npcg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return npcg.Context.sharded(device, rank, world, obj[0])


def exchange_context(device: int, group=None):
    """A row-sharded npcg Context whose exchanges run through TorchExchange."""
    import paper_2110_02820_b200 as npcg
    ex = TorchExchange(group)
    return npcg.Context.exchange(device, ex.rank, ex.world, ex)


class TorchExchange:
    """npcg_exchange_fn over torch.distributed with host staging (any backend
    that handles CPU tensors, e.g. gloo): kind 0 sum all-reduce in place,
    1 all-gather rank-major, 2 reduce-scatter (all-reduce, keep this rank's
    block)."""

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
        """The collective on host tensors (send: count doubles; recv as documented)."""
        if kind == ALLREDUCE:
            self.dist.all_reduce(send, group=self.group)
        elif kind == ALLGATHER:
            count = send.numel()
            self.dist.all_gather(list(recv.view(self.world, count).unbind(0)), send, group=self.group)
        elif kind == REDUCE_SCATTER:
            count = recv.numel()
            full = send.clone()
            self.dist.all_reduce(full, group=self.group)
            recv.copy_(full[self.rank * count:(self.rank + 1) * count])
        else:
            raise ValueError(f"unknown exchange kind {kind}")

    def _call(self, user, kind, send, recv, count, stream) -> int:
        try:
            import torch
            nsend = count * (self.world if kind == REDUCE_SCATTER else 1)
            nrecv = count * (self.world if kind == ALLGATHER else 1)
            torch.cuda.ExternalStream(stream).synchronize()  # the library's producers are done
            dsend = torch.as_tensor(_DevView(send, nsend), device="cuda")
            hs = dsend.cpu()
            if kind == ALLREDUCE:
                self.exchange(kind, hs, hs)
                dsend.copy_(hs)
            else:
                hr = torch.empty(nrecv, dtype=torch.float64)
                self.exchange(kind, hs, hr)
                torch.as_tensor(_DevView(recv, nrecv), device="cuda").copy_(hr)
            torch.cuda.synchronize()  # the copies land before the library's consumers
            self.calls += 1
            return 0
        except BaseException as e:  # noqa: BLE001 - reported through the library's status code
            self.errors.append(e)
            return 1


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


def local_rows(a: np.ndarray, n: int, rank: int, world: int) -> np.ndarray:
    """Rows R_rank of an n-row array (Fortran order kept)."""
    off, cnt = shard_rows(n, world, rank)
    return np.asfortranarray(a[off:off + cnt])
