"""World-size-2 gloo test of bench.py's multi-rank plumbing on CPU (replicas: barrier, max-over-ranks
timing, whole-job throughput = Σ units / max time).  No GPU involved."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import bench
    r, wd, _ = bench.dist_init()
    assert (r, wd) == (rank, world)
    bench.barrier(wd)
    t = 2.0 if rank == 0 else 4.0                   # per-rank time
    units = 10.0                                    # per-rank solves
    tmax = bench.max_over_ranks(t, wd)
    val = bench.whole_job_throughput(units, t, wd)
    q.put((rank, tmax, val))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_replica_throughput_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    for rank, tmax, val in res:
        assert tmax == 4.0                           # max over ranks, not the local clock
        assert abs(val - 20.0 / 4.0) < 1e-12         # whole job: 2 x 10 units / 4 s
