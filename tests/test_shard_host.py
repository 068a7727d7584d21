"""NEXT #3 (x-sharded 1D solve) on the host, no GPU: the partition arithmetic of the
sharded P_α⁻¹ step (b) and of the sharded 𝓜u, run by world-size-2/3 gloo process groups.

Each rank takes its chunk of the spatial index (paper_2401_16113_b200.shard.partition), solves its
Dirichlet-cut block of every shifted system with the oracle's Thomas (test side),
all-gathers the two end values per frequency through the product's TorchDistComm (gloo), solves the
reduced system with the product's host entry points (cnpint_shard_spike_ends_host /
cnpint_shard_reduced_host — the same C++ the device kernel runs), re-solves its block with the corrected
end rows and must reproduce the oracle's unsharded shifted solve; likewise 𝓜u from the all-gathered
boundary columns reproduces the oracle's block matvec."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _worker(rank, world, port, kind, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import aao, precond, problem
        from paper_2401_16113_b200 import problems, shard
        base = synth.C1 if kind == "logprice" else synth.C3
        w = synth.scaled(base, 61, 16, alpha=0.05)
        op = problem.build_operator(w)
        spec = problems.operator_spec(w)
        x0 = shard.partition(w.n, world)
        a, b = x0[rank], x0[rank + 1]
        red, ab = shard.spike_ends_host(w.N, w.T, w.alpha, spec, x0)
        comm = shard.TorchDistComm()
        N, K, tau = w.N, w.N // 2 + 1, w.T / w.N
        # ---- P_α⁻¹ step (b): local block solves, all-gather of the ends, reduced solve, re-solve
        v = synth.random_vectors(w, 1, 7)[0]
        g = precond.gamma(N, w.alpha)
        what = np.fft.fft(g[:, None] * v, axis=0)[:K]
        l1, l2 = precond.lambdas_fft(N, w.alpha)
        l1, l2 = l1[:K, None], l2[:K, None]
        A = -l2 * tau * op.lo[None, a:b]
        B = l1 - l2 * tau * op.di[None, a:b]
        Cc = -l2 * tau * op.up[None, a:b]
        A[:, 0] = 0.0                          # the Dirichlet cut of the block
        Cc[:, -1] = 0.0
        gl = precond.thomas(A, B, Cc, what[:, a:b])
        ends = np.stack([gl[:, 0], gl[:, -1]], axis=1)                 # [K][2]
        send = torch.from_numpy(ends.view(np.float64).reshape(-1).copy())
        recv = torch.empty(world * send.numel(), dtype=torch.float64)
        comm.allgather(send, recv)
        ends_all = recv.numpy().view(np.complex128).reshape(world, K, 2)
        nb = shard.reduced_neighbours_host(red, ab, ends_all, rank)    # (xe_{r−1}, xs_{r+1})
        rhs = what[:, a:b].copy()
        rhs[:, 0] += l2[:, 0] * ab[rank, 0] * nb[:, 0]
        rhs[:, -1] += l2[:, 0] * ab[rank, 1] * nb[:, 1]
        zl = precond.thomas(A, B, Cc, rhs)
        zfull = precond.shifted_solve(w, op, l1[:, 0], l2[:, 0], what)
        e_pinv = _rel(zl, zfull[:, a:b])
        # ---- 𝓜u: the Dirichlet-cut local matvec plus the all-gathered neighbour columns
        u = synth.random_vectors(w, 1, 9)[0]
        opl = problem.Operator1D(op.lo[a:b].copy(), op.di[a:b].copy(), op.up[a:b].copy(), op.x[a:b], op.h)
        opl.lo[0] = 0.0
        opl.up[-1] = 0.0
        yl = aao.apply_M(w, opl, u[:, a:b].copy())
        edges = torch.from_numpy(np.concatenate([u[:, a], u[:, b - 1]]))
        halo = torch.empty(world * 2 * N, dtype=torch.float64)
        comm.allgather(edges, halo)
        halo = halo.numpy().reshape(world, 2, N)
        if rank > 0:
            hl = halo[rank - 1, 1]
            yl[:, 0] -= 0.5 * ab[rank, 0] * (hl + np.concatenate([[0.0], hl[:-1]]))
        if rank < world - 1:
            hr = halo[rank + 1, 0]
            yl[:, -1] -= 0.5 * ab[rank, 1] * (hr + np.concatenate([[0.0], hr[:-1]]))
        e_mv = _rel(yl, aao.apply_M(w, op, u)[:, a:b])
        # ---- the dot-product all-reduce of the sharded GMRES
        t = torch.tensor([float(rank + 1), 2.0 * rank], dtype=torch.float64)
        comm.allreduce_(t)
        q.put((rank, e_pinv, e_mv, t.tolist(), ab[rank].tolist()))
    finally:
        dist.destroy_process_group()


def test_partition_bounds():
    from paper_2401_16113_b200 import shard
    assert shard.partition(10, 3) == [0, 4, 7, 10]
    assert shard.partition(4095, 8)[-1] == 4095
    x = shard.partition(4095, 8)
    assert max(np.diff(x)) - min(np.diff(x)) <= 1
    with pytest.raises(ValueError):
        shard.partition(5, 3)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["logprice", "price"])
def test_sharded_partition_arithmetic_gloo(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for rank, e_pinv, e_mv, red_sum, abr in res:
        assert e_pinv < 1e-12, (kind, world, rank, e_pinv)
        assert e_mv < 1e-13, (kind, world, rank, e_mv)
        assert red_sum == [world * (world + 1) / 2, float(world * (world - 1))]
        # the domain ends carry no coupling
        if rank == 0:
            assert abr[0] == 0.0
        if rank == world - 1:
            assert abr[1] == 0.0
