"""Row-sharded multi-GPU path: one process per GPU, every
n-vector split into balanced row blocks, exchanges issued by the library.

CPU suite: world-size-2 gloo runs of the host side -- the balanced block
layout, TorchExchange's collectives (all-reduce, all-gather, reduce-scatter)
and a numpy restatement of the sharded PCG data flow against the unsharded
iteration.

GPU suite: the library's own sharded path. Two processes share the one GPU
as the ranks of a world-2 context with host-staged exchanges (the library
synchronises its stream around every collective, so no kernel waits on the
other rank); their row blocks are stitched and compared with an unsharded
context and with the CPU oracle: PCG iterations within +-1, x within 1e-8,
Nystrom eigenvalues within 1e-10, identical adaptive rank decisions, products
of every operator kind (dense, ridge Gram, stored kernel, low-rank, matrix-
free kernel for 1, 2, 5 and 12 vectors). The NCCL data plane inside the
library is exercised at world size 1 (bench.py's torchrun path)."""
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
            assert blocks[0][0] == 0
            assert all(blocks[r][0] + blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
            assert max(c for _, c in blocks) - min(c for _, c in blocks) <= 1  # balanced (comm.cuh RowSplit)


def test_gloo_exchange_semantics(gloo2):
    for rank in (0, 1):
        assert np.array_equal(gloo2[rank]["allreduce"], np.full(5, 3.0))
        assert np.array_equal(gloo2[rank]["allgather"], np.array([0, 1, 2, 10, 11, 12], dtype=float))
        # send_g = (0..3) * (g + 1); sum = 3 * (0..3); rank r keeps entries 2r, 2r+1
        assert np.array_equal(gloo2[rank]["reduce_scatter"], 3.0 * np.arange(2 * rank, 2 * rank + 2))


@pytest.mark.parametrize("which", ["cg_gram", "cg_dense"])
def test_gloo_sharded_pcg_dataflow(gloo2, which):
    for rank in (0, 1):
        (xs, its), (x1, it1) = gloo2[rank][which]
        assert abs(its - it1) <= 1
        assert np.linalg.norm(xs - x1) <= 1e-8 * np.linalg.norm(x1)
    assert gloo2[0][which][0][1] == gloo2[1][which][0][1]  # ranks take the same branch


def _stitch(parts, key):
    return np.concatenate([parts[r][key] for r in sorted(parts)], axis=0)


@pytest.fixture(scope="module")
def sharded2():
    """World-2 context on one GPU (host-staged gloo exchanges) + the unsharded reference."""
    port = _port()
    ranks = _spawn(dist_worker.gpu_exchange_rank, [(r, 2, port) for r in range(2)], timeout=900)
    ref = _spawn(dist_worker.gpu_reference, [()], timeout=900)[0]
    return ranks, ref


@pytest.mark.gpu
def test_sharded_world2_matches_unsharded_and_oracle(sharded2, orc):
    from oracle.workload_ops import build_oracle_operator
    ranks, ref = sharded2
    for r in (0, 1):
        assert not ranks[r]["errors"], ranks[r]["errors"]
        assert ranks[r]["calls"] > 0
    oprob = dist_worker._problems(orc)
    for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
        r0, r1, one = ranks[0][name], ranks[1][name], ref[name]
        assert r0["rows"][0] == 0 and r0["rows"][1] + r1["rows"][1] == one["rows"][1]
        # factorisation: identical l x l algebra on both ranks (all-reduced Grams)
        assert np.array_equal(r0["lam"], r1["lam"]) and r0["shift"] == r1["shift"]
        keep = one["lam"] >= 1e-6 * one["lam"][0]
        assert np.max(np.abs(r0["lam"][keep] - one["lam"][keep]) / one["lam"][keep]) <= 1e-10, name
        u = np.vstack([r0["u"], r1["u"]])
        sep = keep.copy()
        dots = np.abs(np.einsum("ij,ij->j", u[:, sep], one["u"][:, sep]))
        assert dots.min() >= 1 - 1e-8, name
        # oracle on the same inputs
        w = oprob[name]
        oop = build_oracle_operator(orc, w)
        ao = orc.nystrom_from_sketch(orc.extend_sketch_with(orc.make_empty_sketch(w.n), oop, w.omega))
        assert np.max(np.abs(r0["lam"][keep] - ao.lam[keep]) / ao.lam[keep]) <= 1e-10, name
        b = w.b.reshape(w.n, -1, order="F")
        for k, mu in enumerate(w.mus or [w.mu]):
            opre = orc.build_preconditioner(ao, mu)
            for j in range(b.shape[1]):
                it0, x0 = r0["solves"][k][j]
                it1, x1 = r1["solves"][k][j]
                itr, xr = one["solves"][k][j]
                assert it0 == it1  # both ranks leave the loop together
                x = np.concatenate([x0, x1])
                ro = orc.nystrom_pcg(oop, b[:, j], mu, opre, eta=w.eta, relative=True)
                assert abs(it0 - ro.iterations) <= 1 and abs(it0 - itr) <= 1, (name, it0, itr, ro.iterations)
                assert np.linalg.norm(x - ro.x) <= 1e-8 * np.linalg.norm(ro.x), name
                assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr), name
        if r0["block"] is not None:
            itb, xb, defl = r0["block"]
            xfull = np.vstack([xb, r1["block"][1]])
            ob = orc.block_nystrom_pcg(oop, b, w.mus[-1], orc.build_preconditioner(ao, w.mus[-1]), eta=w.eta,
                                       relative=True)
            assert abs(itb - ob.iterations) <= 1 and defl == ob.deflated
            assert np.linalg.norm(xfull - ob.x) <= 1e-8 * np.linalg.norm(ob.x)


@pytest.mark.gpu
def test_sharded_world2_matrix_free_kernel(sharded2):
    ranks, ref = sharded2
    r0, r1, one = ranks[0]["cfg4"], ranks[1]["cfg4"], ref["cfg4"]
    for key in ("Av1", "Av2", "Av5", "Av12"):
        got = np.concatenate([r0[key], r1[key]], axis=0)
        want = one[key]
        assert np.allclose(got, want, rtol=1e-12, atol=1e-13 * np.abs(want).max()), key
    assert r0["adaptive"][:3] == r1["adaptive"][:3] == one["adaptive"][:3]
    assert abs(r0["adaptive"][3] - one["adaptive"][3]) <= 1e-8 * abs(one["adaptive"][3])
    it0, x0 = r0["pcg"]
    itr, xr = one["pcg"]
    assert it0 == r1["pcg"][0] and abs(it0 - itr) <= 1
    x = np.concatenate([x0, r1["pcg"][1]])
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.gpu
def test_nccl_data_plane_world1():
    res = _spawn(dist_worker.gpu_nccl_world1, [(_port(),)], timeout=900)[0]
    ref = _spawn(dist_worker.gpu_reference, [()], timeout=900)[0]
    for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
        assert np.array_equal(res[name]["lam"], ref[name]["lam"]), name
        for a, b in zip(res[name]["solves"], ref[name]["solves"]):
            for (ia, xa), (ib, xb) in zip(a, b):
                assert ia == ib and np.array_equal(xa, xb), name
