"""Row-sharded multi-GPU path.

CPU suite: world-size-2 gloo runs of the sharding host logic -- block
layout, exchange semantics of TorchExchange, and that a row-sharded operator
with replicated vectors reproduces the unsharded products and CG iterations
(Gram: all-reduce of partial X_g^T X_g v; dense: all-gather of column-block
products). GPU suite: the library's sharded operators, exchanging through the
C callback over NCCL (world 1), against the unsharded operators."""
import multiprocessing as mp
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent))
import dist_worker  # noqa: E402

from paper_2110_02820_b200 import dist as pd  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(target, args_per_rank, timeout=240):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(*a, q)) for a in args_per_rank]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            rank, val = q.get(timeout=timeout)
            res[rank] = val
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for v in res.values():
        assert not isinstance(v, str), v
    return res


@pytest.fixture(scope="module")
def gloo2():
    port = _port()
    return _spawn(dist_worker.cpu_checks, [(r, 2, port) for r in range(2)])


def test_block_layout():
    for total in (1, 7, 53, 4000):
        for world in (1, 2, 3, 8):
            if world > total:
                continue
            blocks = [pd.shard_rows(total, world, r) for r in range(world)]
            assert sum(c for _, c in blocks) == total
            assert all(blocks[r][0] == r * pd.block_size(total, world) for r in range(world) if blocks[r][1])
            assert all(blocks[r][0] + blocks[r][1] == blocks[r + 1][0] for r in range(world - 1) if blocks[r + 1][1])


def test_unpack_gathered_matches_layout():
    n, world, k = 11, 3, 2
    nb = pd.block_size(n, world)
    full = np.arange(n * k, dtype=float).reshape(n, k, order="F")
    recv = np.zeros(world * k * nb)
    for r in range(world):
        off, cnt = pd.shard_rows(n, world, r)
        blk = np.zeros((nb, k), order="F")
        blk[:cnt] = full[off:off + cnt]
        recv[r * k * nb:(r + 1) * k * nb] = blk.ravel(order="F")
    assert np.array_equal(pd.unpack_gathered(recv, n, world, k), full)


def test_gloo_exchange_semantics(gloo2):
    for rank in (0, 1):
        assert np.array_equal(gloo2[rank]["allreduce"], np.full(5, 3.0))
        assert np.array_equal(gloo2[rank]["allgather"], np.array([0, 1, 2, 10, 11, 12], dtype=float))


def test_gloo_sharded_gram_matvec(gloo2):
    for rank in (0, 1):
        got, want = gloo2[rank]["gram"]
        assert np.allclose(got, want, rtol=1e-13, atol=1e-15 * np.abs(want).max())
    assert np.array_equal(gloo2[0]["gram"][0], gloo2[1]["gram"][0])  # replicated, bitwise


def test_gloo_sharded_dense_matvec(gloo2):
    for rank in (0, 1):
        got, want = gloo2[rank]["dense"]
        assert np.allclose(got, want, rtol=1e-13, atol=1e-15 * np.abs(want).max())


@pytest.mark.parametrize("which", ["cg_gram", "cg_dense"])
def test_gloo_sharded_cg_iterations(gloo2, which):
    (xs, its), (x1, it1) = gloo2[0][which]
    assert abs(its - it1) <= 1
    assert np.linalg.norm(xs - x1) <= 1e-8 * np.linalg.norm(x1)
    (xs2, its2), _ = gloo2[1][which]
    assert its2 == its and np.array_equal(xs2, xs)  # ranks agree bitwise


@pytest.mark.gpu
def test_nccl_sharded_operators_world1():
    res = _spawn(dist_worker.gpu_checks, [(_port(),)], timeout=600)[0]
    assert not res["errors"], res["errors"]
    assert res["calls"] > 0
    xf, itf, lf, vf = res["full"]
    xs, its, ls, vs = res["shard"]
    assert np.allclose(vs, vf, rtol=1e-13, atol=1e-15 * np.abs(vf).max())
    assert abs(its - itf) <= 1
    assert np.linalg.norm(xs - xf) <= 1e-8 * np.linalg.norm(xf)
    big = lf >= 1e-6 * lf[0]
    assert np.all(np.abs(ls[big] - lf[big]) <= 1e-10 * lf[big])
    for key in ("dense", "kernel", "lowrank"):
        got, want = res[key]
        assert np.allclose(got, want, rtol=1e-12, atol=1e-13 * np.abs(want).max()), key
