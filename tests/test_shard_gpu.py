"""NEXT #3 on one GPU: the x-sharded handles (include/cnpint.h "1D x-sharded handles")
against the oracle.  The R ranks are emulated on the single GPU without any device-side waiting between
ranks: either phase by phase (every rank's begin phase, the exchange buffers moved by the test, every
rank's end phase) or as R host threads whose collectives rendezvous on the host (the kernels of a
rank never wait on another rank's kernels).  The multi-GPU NCCL path itself is unmeasured on hardware.
"""
import threading

import numpy as np
import pytest

import synth
from oracle import aao, gmres as ogmres, precond, problem
from tests.gpu_util import record, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2401_16113_b200 import problems, shard  # noqa: E402

CASES = {
    "c1_R2": (synth.C1, 2),
    "c1_R3": (synth.C1, 3),
    "price_R2": (synth.scaled(synth.C3, 255, 256, alpha=0.01), 2),
    "c2_R4": (synth.C2, 4),            # four-step time FFT, 2049 frequencies, chunks of 1024 rows
    "c3_R2": (synth.C3, 2),            # variable rows, N = 16384
}


def make_ranks(w, R, restart_max=0):
    spec = problems.operator_spec(w)
    return [shard.ShardSolver(w.N, w.T, w.alpha, spec, r, R, restart_max=restart_max) for r in range(R)]


def exchange(ranks, which):
    """All-gather of every rank's send buffer into every rank's receive buffer (the test moves them)."""
    bufs = [rk.buffers() for rk in ranks]
    i = 0 if which == "ends" else 2
    cat = torch.cat([b[i] for b in bufs])
    for b in bufs:
        b[i + 1].copy_(cat)


@pytest.mark.parametrize("name", list(CASES))
def test_sharded_pinv_and_matvec_phase_split(name):
    w, R = CASES[name]
    op = problem.build_operator(w)
    ranks = make_ranks(w, R)
    v = synth.random_vectors(w, 1, 13)[0]
    x0 = ranks[0].x0
    zs = [rk.empty() for rk in ranks]
    for r, rk in enumerate(ranks):
        rk.pinv_begin(rk.to_device(v[:, x0[r]:x0[r + 1]]))
    torch.cuda.synchronize()
    exchange(ranks, "ends")
    for rk, z in zip(ranks, zs):
        rk.pinv_end(z)
    zg = np.concatenate([rk.to_host(z) for rk, z in zip(ranks, zs)], axis=1)
    if w.N >= 4096:
        # reading R-tol: at c2/c3 sizes the fp64 oracle's own error nears 1e-12, so the forward
        # error is taken against the extended-precision oracle, bounded by max(1e-12, 4 × its own)
        zt = precond.pinv_dft(w, op, v, extended=True)
        own = rel(precond.pinv_dft(w, op, v), zt)
        fwd = rel(zg, zt)
        bar = max(1e-12, 4 * own)
    else:
        fwd, bar = rel(zg, precond.pinv_dft(w, op, v)), 1e-12
    back = rel(aao.apply_P(w, op, zg), v)
    # 𝓜u with the all-gathered boundary columns
    ys = [rk.empty() for rk in ranks]
    us = [rk.to_device(v[:, x0[r]:x0[r + 1]]) for r, rk in enumerate(ranks)]
    for rk, u in zip(ranks, us):
        rk.halo_begin(u)
    torch.cuda.synchronize()
    exchange(ranks, "halo")
    for rk, u, y in zip(ranks, us, ys):
        rk.apply_A_end(u, y)
    yg = np.concatenate([rk.to_host(y) for rk, y in zip(ranks, ys)], axis=1)
    e_mv = rel(yg, aao.apply_M(w, op, v))
    record(f"shard_{name}", pinv_forward=fwd, pinv_backward=back, matvec=e_mv)
    assert fwd <= bar and back < 1e-12 and e_mv < 1e-12, (fwd, bar, back, e_mv)
    for rk, z in zip(ranks, zs):
        assert float(z[:, rk.nx:].abs().max()) == 0.0 if rk.ld > rk.nx else True
        assert rk.device_status() == 0


class HostComm:
    """Collectives of R host threads that share one GPU: each rank synchronises its own stream, deposits
    its buffer, and after a host barrier every rank assembles the same result (fixed rank order, so
    the all-reduce is deterministic)."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world

    def rank(self, r):
        outer = self

        class _C:
            def allgather(self, send, recv):
                torch.cuda.current_stream().synchronize()
                outer.slots[r] = send.clone()
                outer.bar.wait()
                recv.copy_(torch.cat(outer.slots))
                torch.cuda.current_stream().synchronize()
                outer.bar.wait()

            def allreduce_(self, buf):
                torch.cuda.current_stream().synchronize()
                outer.slots[r] = buf.clone()
                outer.bar.wait()
                acc = outer.slots[0].clone()
                for s in outer.slots[1:]:
                    acc += s
                buf.copy_(acc)
                torch.cuda.current_stream().synchronize()
                outer.bar.wait()

        return _C()


def run_threads(w, R, fn):
    comm = HostComm(R)
    spec = problems.operator_spec(w)
    ranks = [shard.ShardSolver(w.N, w.T, w.alpha, spec, r, R, restart_max=w.restart, comm=comm.rank(r))
             for r in range(R)]
    out = [None] * R
    err = []

    def body(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(ranks[r], r)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover
            err.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not err, err
    return ranks, out


@pytest.mark.parametrize("name,R", [("c1", 1), ("c1", 2), ("c1", 3), ("price", 2)])
def test_sharded_gmres_threads(name, R):
    """cnpint_shard_gmres on R emulated ranks: the collective callback (all-gathers inside P⁻¹ and 𝓜,
    all-reduced CGS2 dots) — counts ±1 vs the oracle, final u vs sequential CN (1e-8), every rank the same
    report."""
    w = {"c1": synth.C1, "price": synth.scaled(synth.C3, 255, 256, alpha=0.01, restart=40)}[name]
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    x0 = shard.partition(w.n, R)

    def solve(rk, r):
        bl = rk.to_device(b[:, x0[r]:x0[r + 1]])
        u = rk.empty()
        rep = rk.gmres(bl, u, w.tol, w.restart)
        return rep, rk.to_host(u)

    ranks, out = run_threads(w, R, solve)
    reps = [o[0] for o in out]
    ug = np.concatenate([o[1] for o in out], axis=1)
    _, orep = ogmres.gmres_right(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x), b,
                                 w.tol, w.restart)
    e_seq = rel(ug, aao.solve_sequential(w, op, b))
    record(f"shard_gmres_{name}_R{R}", iterations=reps[0]["iterations"], oracle_iterations=orep.iterations,
           relres_true=reps[0]["relres_true"], u_vs_seqcn=e_seq)
    assert all(r["iterations"] == reps[0]["iterations"] and r["relres_true"] == reps[0]["relres_true"] for r in reps)
    assert reps[0]["converged"] and reps[0]["relres_true"] <= w.tol
    assert abs(reps[0]["iterations"] - orep.iterations) <= 1, (reps[0]["iterations"], orep.iterations)
    assert e_seq < 1e-8, e_seq
