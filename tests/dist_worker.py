"""Per-rank bodies of the multi-process tests (tests/test_dist_shard.py).

CPU ranks (gloo) check the host side of the row sharding: the block layout,
the exchange semantics of paper_2110_02820_b200.dist.TorchExchange and that
a row-sharded operator with replicated vectors reproduces the unsharded
products and the unsharded CG iteration. The GPU rank (NCCL, world 1) drives
the library's sharded operators through the C callback."""
import os

import numpy as np


def _init(rank, world, port, backend):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


def cg_numpy(matvec, b, mu, eta, max_iter=500):
    """solvers.cpp:40-107 with the identity preconditioner (relative eta)."""
    x = np.zeros_like(b)
    r = b.copy()
    eta_used = eta * np.linalg.norm(b)
    z = r.copy()
    p = z.copy()
    rz = r @ z
    it = 0
    while it < max_iter:
        it += 1
        v = matvec(p) + mu * p
        alpha = rz / (p @ v)
        x += alpha * p
        r -= alpha * v
        if np.linalg.norm(r) <= eta_used:
            break
        z = r.copy()
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it


def cpu_checks(rank, world, port, q):
    try:
        dist = _init(rank, world, port, "gloo")
        import torch
        from paper_2110_02820_b200 import dist as pd
        ex = pd.TorchExchange()
        out = {}
        # exchange semantics
        t = torch.full((5,), float(rank + 1), dtype=torch.float64)
        ex.exchange(pd.ALLREDUCE, t, t)
        out["allreduce"] = t.numpy().copy()
        s = torch.arange(3, dtype=torch.float64) + 10 * rank
        r = torch.empty(3 * world, dtype=torch.float64)
        ex.exchange(pd.ALLGATHER, s, r)
        out["allgather"] = r.numpy().copy()
        # Gram row shards: all-reduce of X_g^T (X_g v) / m
        rng = np.random.default_rng(7)
        m, n = 301, 37
        X = rng.standard_normal((m, n)) * (np.arange(1, n + 1) ** -0.5)
        v = rng.standard_normal(n)
        off, cnt = pd.shard_rows(m, world, rank)
        Xg = X[off:off + cnt]
        part = torch.from_numpy((Xg.T @ (Xg @ v)) / m)
        ex.exchange(pd.ALLREDUCE, part, part)
        out["gram"] = (part.numpy().copy(), X.T @ (X @ v) / m)

        def gram_mv(p):
            t = torch.from_numpy((Xg.T @ (Xg @ p)) / m)
            ex.exchange(pd.ALLREDUCE, t, t)
            return t.numpy()

        b = X.T @ rng.standard_normal(m) / m
        out["cg_gram"] = (cg_numpy(gram_mv, b, 1e-3, 1e-10), cg_numpy(lambda p: X.T @ (X @ p) / m, b, 1e-3, 1e-10))
        # dense column blocks: all-gather of A[:, R_g]^T v, padded to ceil(n/G)
        nd = 53
        Q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        A = (Q * (np.arange(1, nd + 1) ** -2.0)) @ Q.T
        A = 0.5 * (A + A.T)
        offd, cntd = pd.shard_rows(nd, world, rank)
        nb = pd.block_size(nd, world)

        def dense_mv(p):
            loc = np.zeros(nb)
            loc[:cntd] = A[:, offd:offd + cntd].T @ p
            recv = torch.empty(nb * world, dtype=torch.float64)
            ex.exchange(pd.ALLGATHER, torch.from_numpy(loc), recv)
            return pd.unpack_gathered(recv.numpy(), nd, world, 1)[:, 0]

        w = rng.standard_normal(nd)
        out["dense"] = (dense_mv(w), A @ w)
        bd = rng.standard_normal(nd)
        out["cg_dense"] = (cg_numpy(dense_mv, bd, 1e-4, 1e-10), cg_numpy(lambda p: A @ p, bd, 1e-4, 1e-10))
        q.put((rank, out))
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def gpu_checks(port, q):
    """World-1 NCCL run of the library's sharded operators (exchange through
    the C callback on the library stream) against the unsharded operators."""
    try:
        dist = _init(0, 1, port, "nccl")
        import torch
        torch.cuda.set_device(0)
        import paper_2110_02820_b200 as npcg
        from paper_2110_02820_b200 import dist as pd
        ex = pd.TorchExchange()
        rng = np.random.default_rng(11)
        m, n, ell, mu = 3000, 600, 60, 1e-3
        X = rng.standard_normal((m, n)) * (np.arange(1, n + 1) ** -0.5)
        b = X.T @ rng.standard_normal(m) / m
        omega = npcg.Rng(5).gaussian_matrix(n, ell)
        out = {}
        for name, op in (("full", npcg.GramRidgeOperator(X)), ("shard", pd.ShardedGramOperator(X, m, ex))):
            pair = npcg.extend_sketch_with(npcg.make_empty_sketch(n, op), op, omega)
            approx = npcg.nystrom_from_sketch(pair)
            pre = npcg.build_preconditioner(approx, mu)
            rep = npcg.nystrom_pcg(op, b, mu, pre, eta=1e-10, relative=True)
            out[name] = (rep.x.copy(), rep.iterations, np.asarray(approx.lam).copy(), op.matvec(b))
        A = X.T @ X / m
        dop = pd.ShardedDenseOperator(A, n, ex)
        out["dense"] = (dop.matvec(b), A @ b)
        pts = rng.standard_normal((700, 16))
        kfull, kshard = npcg.KernelOperator(pts, 3.0, dense_cap=5000), pd.ShardedKernelOperator(pts, 3.0, ex)
        W = rng.standard_normal((700, 3))
        out["kernel"] = (kshard.apply_block(W), kfull.apply_block(W))
        G = rng.standard_normal((500, 40))
        lam = np.exp(-np.arange(40) / 10.0)
        lfull, lshard = npcg.LowRankOperator(G, lam), pd.ShardedLowRankOperator(G, lam, ex)
        W2 = rng.standard_normal((500, 2))
        out["lowrank"] = (lshard.apply_block(W2), lfull.apply_block(W2))
        out["calls"] = ex.calls
        out["errors"] = [repr(e) for e in ex.errors]
        q.put((0, out))
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((0, traceback.format_exc()))
