"""Per-rank bodies of the multi-process tests (tests/test_dist_shard.py).

CPU ranks (gloo, world 2) check the host side of the row sharding: the
balanced block layout, TorchExchange's three collectives, and a numpy
restatement of the sharded PCG data flow (row-sharded x, r, z, p; all-gather
of p before the product; all-reduced dots; reduce-scatter for a Gram
operator) against the unsharded iteration.

GPU ranks drive the library itself on row-sharded contexts:
* `gpu_nccl_world1`: the NCCL data plane created inside the library
  (npcg_ctx_create_sharded) at world size 1 -- the path bench.py takes
  under torchrun -- against an unsharded context;
* `gpu_exchange_rank`: two processes sharing ONE GPU, each a rank of a
  world-2 context whose exchanges are host-staged through gloo
  (dist.TorchExchange: the library synchronises its stream before every
  collective, so no kernel of one rank waits on the other). Each rank solves
  the BASELINE-shaped problems on its row blocks and returns them."""
import os

import numpy as np


def _init(rank, world, port, backend):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


def pcg_sharded_numpy(local_mv, b_loc, mu, eta, allreduce, max_iter=500):
    """solvers.cpp:40-107 with the identity preconditioner on row-sharded
    vectors: each dot is a local partial summed by `allreduce`."""
    dot = lambda u, v: allreduce(np.array([u @ v]))[0]  # noqa: E731
    x = np.zeros_like(b_loc)
    r = b_loc.copy()
    eta_used = eta * np.sqrt(dot(b_loc, b_loc))
    z = r.copy()
    p = z.copy()
    rz = dot(r, z)
    it = 0
    while it < max_iter:
        it += 1
        v = local_mv(p) + mu * p
        alpha = rz / dot(p, v)
        x += alpha * p
        r -= alpha * v
        if np.sqrt(dot(r, r)) <= eta_used:
            break
        z = r.copy()
        rz_new = dot(r, z)
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
        t = torch.full((5,), float(rank + 1), dtype=torch.float64)
        ex.exchange(pd.ALLREDUCE, t, t)
        out["allreduce"] = t.numpy().copy()
        s = torch.arange(3, dtype=torch.float64) + 10 * rank
        r = torch.empty(3 * world, dtype=torch.float64)
        ex.exchange(pd.ALLGATHER, s, r)
        out["allgather"] = r.numpy().copy()
        s2 = torch.arange(2 * world, dtype=torch.float64) * (rank + 1)
        r2 = torch.empty(2, dtype=torch.float64)
        ex.exchange(pd.REDUCE_SCATTER, s2, r2)
        out["reduce_scatter"] = r2.numpy().copy()

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            ex.exchange(pd.ALLREDUCE, t, t)
            return t.numpy()

        def allgather_rows(loc, n):
            offs = [pd.shard_rows(n, world, g) for g in range(world)]
            nmax = max(c for _, c in offs)
            send = np.zeros(nmax)
            send[:loc.size] = loc
            recv = torch.empty(nmax * world, dtype=torch.float64)
            ex.exchange(pd.ALLGATHER, torch.from_numpy(send), recv)
            rv = recv.numpy()
            return np.concatenate([rv[g * nmax:g * nmax + c] for g, (_, c) in enumerate(offs)])

        def reduce_scatter_rows(full, n):
            offs = [pd.shard_rows(n, world, g) for g in range(world)]
            nmax = max(c for _, c in offs)
            send = np.zeros(nmax * world)
            for g, (o, c) in enumerate(offs):
                send[g * nmax:g * nmax + c] = full[o:o + c]
            recv = torch.empty(nmax, dtype=torch.float64)
            ex.exchange(pd.REDUCE_SCATTER, torch.from_numpy(send), recv)
            return recv.numpy()[:offs[rank][1]].copy()

        rng = np.random.default_rng(7)
        # dense column block A[:, R_g]: all-gather p, local rows of A p
        nd = 53
        Q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        A = (Q * (np.arange(1, nd + 1) ** -2.0)) @ Q.T
        A = 0.5 * (A + A.T)
        offd, cntd = pd.shard_rows(nd, world, rank)
        dense_mv = lambda p_loc: A[:, offd:offd + cntd].T @ allgather_rows(p_loc, nd)  # noqa: E731
        bd = rng.standard_normal(nd)
        xs, its = pcg_sharded_numpy(dense_mv, bd[offd:offd + cntd], 1e-4, 1e-10, allreduce)
        x1, it1 = pcg_sharded_numpy(lambda p: A @ p, bd, 1e-4, 1e-10, lambda a: a)
        out["cg_dense"] = ((xs, its), (x1[offd:offd + cntd], it1))
        # Gram over row blocks of X: all-gather p, partial X_g^T X_g p / m, reduce-scatter
        m, n = 301, 37
        X = rng.standard_normal((m, n)) * (np.arange(1, n + 1) ** -0.5)
        om, cm = pd.shard_rows(m, world, rank)
        Xg = X[om:om + cm]
        on, cn = pd.shard_rows(n, world, rank)
        gram_mv = lambda p_loc: reduce_scatter_rows(Xg.T @ (Xg @ allgather_rows(p_loc, n)) / m, n)  # noqa: E731
        b = X.T @ rng.standard_normal(m) / m
        xs, its = pcg_sharded_numpy(gram_mv, b[on:on + cn], 1e-3, 1e-10, allreduce)
        x1, it1 = pcg_sharded_numpy(lambda p: X.T @ (X @ p) / m, b, 1e-3, 1e-10, lambda a: a)
        out["cg_gram"] = ((xs, its), (x1[on:on + cn], it1))
        q.put((rank, out))
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


# ------------------------------------------------------------------ GPU ranks
def _problems(npcg_or_orc):
    """Small BASELINE-shaped problems, identical on every rank (reference Rng)."""
    from paper_2110_02820_b200 import workloads
    R, sm = npcg_or_orc.Rng, npcg_or_orc.splitmix64
    return {
        "cfg1": workloads.make("cfg1", R, sm, n=600, ell=60),
        "cfg2": workloads.make("cfg2", R, sm, m=2400, n=500, ell=60,
                               gemm=lambda a, b, transa=False: (a.T if transa else a) @ b),
        "cfg3": workloads.make("cfg3", R, sm, n=1500, ell=120),
        "cfg5": workloads.make("cfg5", R, sm, n=1200, r=150, ell=80, nmu=2),
    }


def solve_all(npcg, ctx, rows):
    """Sketch + factor + preconditioner + PCG on every problem through the
    library on `ctx`; vectors are this rank's row blocks (`rows(n)`)."""
    from paper_2110_02820_b200 import workloads
    out = {}
    for name, w in _problems(npcg).items():
        op = workloads.build_operator(npcg, w, ctx=ctx)
        off, cnt = rows(w.n)
        pair = npcg.extend_sketch_with(npcg.make_empty_sketch(op), op, w.omega[off:off + cnt])
        ap = npcg.nystrom_from_sketch(pair)
        b = w.b.reshape(w.n, -1, order="F")[off:off + cnt]
        res = []
        for mu in (w.mus or [w.mu]):
            pre = npcg.build_preconditioner(ap, mu)
            reps = npcg.nystrom_pcg(op, b, mu, pre, eta=w.eta, relative=True)
            reps = reps if isinstance(reps, list) else [reps]
            res.append([(r.iterations, r.x.copy()) for r in reps])
        blk = None
        if name == "cfg5":
            br = npcg.block_nystrom_pcg(op, b, w.mus[-1], npcg.build_preconditioner(ap, w.mus[-1]), eta=w.eta,
                                        relative=True)
            blk = (br.iterations, br.x.copy(), br.deflated)
        out[name] = {"lam": ap.lam.copy(), "shift": ap.shift_used, "u": ap.u.copy(), "solves": res, "block": blk,
                     "rows": (off, cnt)}
    # matrix-free kernel (cfg 4 shape): products and the adaptive loop
    w = workloads.make("cfg4", npcg.Rng, npcg.splitmix64, n=2600, ell_max=200)
    w.data["dense_cap"] = 1000
    op = workloads.build_operator(npcg, w, ctx=ctx)
    off, cnt = rows(w.n)
    V = npcg.Rng(9).gaussian_matrix(w.n, 12)
    rng = npcg.Rng(4)
    rng.gaussian_vector(w.n)
    ad = npcg.adaptive(op, rng, mode="error", ell0=w.adaptive["ell0"], ell_max=w.adaptive["ell_max"], mu=w.mu,
                       tau=w.adaptive["tau"], q=w.adaptive["q"])
    pre = npcg.build_preconditioner(ad.approximation, w.mu)
    rep = npcg.nystrom_pcg(op, w.b[off:off + cnt], w.mu, pre, eta=w.eta, relative=True)
    out["cfg4"] = {"Av1": op.matvec(V[off:off + cnt, 0]), "Av2": op.apply_block(V[off:off + cnt, :2]),
                   "Av5": op.apply_block(V[off:off + cnt, :5]), "Av12": op.apply_block(V[off:off + cnt]),
                   "adaptive": (ad.ell_final, ad.doublings, ad.hit_cap, ad.error_estimate),
                   "lam": ad.approximation.lam.copy(), "pcg": (rep.iterations, rep.x.copy()), "rows": (off, cnt)}
    return out


def gpu_exchange_rank(rank, world, port, q):
    """One rank of a world-`world` context on GPU 0, host-staged gloo exchanges."""
    try:
        dist = _init(rank, world, port, "gloo")
        import torch
        torch.cuda.set_device(0)
        import paper_2110_02820_b200 as npcg
        from paper_2110_02820_b200 import dist as pd
        from paper_2110_02820_b200 import workloads
        npcg.workloads = workloads
        ctx = pd.exchange_context(0)
        out = solve_all(npcg, ctx, lambda n: ctx.layout(n)[2:])
        out["calls"] = ctx._keep.calls
        out["errors"] = [repr(e) for e in ctx._keep.errors]
        q.put((rank, out))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


def gpu_reference(q):
    """The same problems on an unsharded context (world 1, no exchange)."""
    try:
        import paper_2110_02820_b200 as npcg
        from paper_2110_02820_b200 import workloads
        npcg.workloads = workloads
        q.put((0, solve_all(npcg, npcg.Context(0), lambda n: (0, n))))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((0, traceback.format_exc()))


def gpu_nccl_world1(port, q):
    """The NCCL data plane inside the library at world size 1 (bench.py's
    torchrun path): context creation over a torch.distributed-distributed id."""
    try:
        dist = _init(0, 1, port, "gloo")
        import torch
        torch.cuda.set_device(0)
        import paper_2110_02820_b200 as npcg
        from paper_2110_02820_b200 import dist as pd
        from paper_2110_02820_b200 import workloads
        npcg.workloads = workloads
        ctx = pd.nccl_context(0)
        q.put((0, solve_all(npcg, ctx, lambda n: ctx.layout(n)[2:])))
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((0, traceback.format_exc()))
