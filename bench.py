#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for cnpint (arxiv 2401.16113 hot path on B200).

Workload (N=1): BASELINE.json configs[1] ("c2"): 1D Black–Scholes in log price, m = 4095, N = 4096
(16.8 M fp64 unknowns), α = 0.01 (the middle of the config's α set), GMRES(restart 30), tol 1e-10,
zero initial guess, manufactured-solution right-hand side b (synthetic, resident in HBM).

Step = one full right-preconditioned GMRES solve to tolerance — every row of SURVEY.md §8(a):
K1 AaO matvec, K2/K3/K4 P_α⁻¹ (Γ-scaled time FFT, batched complex tridiagonal solves, inverse FFT),
K7 CGS2 Arnoldi passes, K8 Givens/Hessenberg on device, K9 cycle end (GEMV, P⁻¹, true residual).
value = GMRES solves/s (time-to-tolerance⁻¹), whole job over all ranks.  Alongside: P_α⁻¹ applies/s,
AaO matvec GB/s and their fraction of the measured HBM peak, K0 stream-copy GB/s, the per-kernel
breakdown (CUDA events on the launch stream), the live roofline of the dominant kernel, the
end-to-end number through the host-buffer C-ABI call, and the CPU oracle on the same box.

Multi-GPU: replicas only: each rank solves its own copy; no data-path collective.
`--impl reference` times the CPU oracle (oracle/, numpy) on the same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json absent)


# ----------------------------------------------------------------------------------- distributed
def dist_init():
    """One process per GPU (torchrun env); returns (rank, world, local_rank)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    """Max of a per-rank scalar (timing contract: the job time is the slowest rank)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def whole_job_throughput(units_per_rank: float, seconds_per_rank: float, world: int) -> float:
    """value = units processed by all ranks / max-over-ranks time (replicas, weak scaling)."""
    total = sum_over_ranks(units_per_rank, world)
    tmax = max_over_ranks(seconds_per_rank, world)
    return total / tmax


# ----------------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"cnpint_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, p in zip(names, parts[2:6]):
                if p.lower() == "active":
                    reasons.add(n)
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, workload: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu --set full capture of the
    same workload (profiles/ncu_traffic.json, written from profiles/r01_ncu_full_summary.txt)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(kernel)
        if d and d.get("workload") == workload:
            return d["bytes_per_launch"], d.get("algo_bytes_this_launch"), d.get("launch")
    return None, None, None


# ----------------------------------------------------------------------------------- workload
def workload(name: str, alpha: float | None):
    import synth
    w = synth.WORKLOADS[name]
    return w.with_(alpha=alpha) if alpha is not None else w


def describe(w):
    return (f"{w.name}: {w.note}; {w.kind} Black-Scholes, N={w.N} steps x m={w.m} unknowns "
            f"({w.unknowns:,} fp64), T={w.T}, alpha={w.alpha}, GMRES({w.restart}) tol {w.tol}, x0=0")


# ----------------------------------------------------------------------------------- GPU arm
def run_gpu(args, rank, world, local):
    import numpy as np
    import torch

    from paper_2401_16113_b200 import problems
    from paper_2401_16113_b200.cnpint import stream_copy
    import synth

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = workload(args.workload, args.alpha)
    s = problems.make_solver(w, restart_max=w.restart)
    b = problems.rhs(w, s)
    u = s.empty()
    stream = torch.cuda.current_stream()
    vec_bytes = s.vec_elems * 8

    # K0: same-run stream copy (HBM reference), 2 x 1 GiB buffers, best of 10
    n = (1 << 30) // 8
    a0 = torch.empty(n, dtype=torch.float64, device=dev).fill_(1.0)
    a1 = torch.empty_like(a0)
    copy_best = 0.0
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        stream_copy(a0, a1)
        e1.record(stream)
        e1.synchronize()
        copy_best = max(copy_best, 2 * n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del a0, a1
    torch.cuda.empty_cache()

    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    # warm-up solves
    for _ in range(args.warmup):
        rep = s.gmres(b, u, w.tol, w.restart)
    torch.cuda.synchronize()
    # ---------------- timed region: K full GMRES solves
    barrier(world)
    torch.cuda.synchronize()
    l0 = s.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    e0.record(stream)
    for _ in range(args.steps):
        reps.append(s.gmres(b, u, w.tol, w.restart))
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    t_rank = e0.elapsed_time(e1) * 1e-3
    launches = s.launch_count() - l0
    clk = clocks.stop() if rank == 0 else None
    value = whole_job_throughput(args.steps, t_rank, world)
    t_max = max_over_ranks(t_rank, world)
    its = [r["iterations"] for r in reps]
    assert all(r["converged"] for r in reps), reps[-1]

    # ---------------- per-kernel breakdown: the same K solves again with the event profiler on
    s.profile_enable(True)
    p0 = time.perf_counter()
    for _ in range(args.steps):
        s.gmres(b, u, w.tol, w.restart)
    torch.cuda.synchronize()
    prof = s.profile_read()
    s.profile_enable(False)
    kernels = {}
    for name, (ms, cnt, by) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        kernels[name] = {"ms_per_step": ms / args.steps, "launches_per_step": cnt / args.steps,
                         "avg_launch_us": 1e3 * ms / cnt, "algo_GBps": (by / (ms * 1e-3) / 1e9) if by else None}
    dominant = max(prof.items(), key=lambda kv: kv[1][0] if kv[1][2] > 0 else -1)[0]
    d_ms, d_cnt, d_by = prof[dominant]
    peak, peak_src = measured_hbm_peak()
    for k in kernels.values():  # every kernel's fraction of the same HBM peak
        k["frac"] = k["algo_GBps"] / peak if k["algo_GBps"] else None
    achieved = d_by / (d_ms * 1e-3) / 1e9
    total_prof_ms = sum(v[0] for v in prof.values())
    traffic = ncu_traffic(dominant, w.name)

    # ---------------- standalone P⁻¹ applies/s and matvec GB/s on 4 seeded N(0,1) vectors (> L2)
    V = synth.random_vectors(w, 4, w.rand_seed)
    dv = [s.to_device(v) for v in V]
    out = [s.empty() for _ in range(2)]
    for i in range(3):
        s.apply_Pinv(dv[i % 4], out[0])
        s.apply_A(dv[i % 4], out[1])
    torch.cuda.synchronize()
    reps_p = max(20, args.steps)
    e0.record(stream)
    for i in range(reps_p):
        s.apply_Pinv(dv[i % 4], out[i % 2])
    e1.record(stream)
    torch.cuda.synchronize()
    pinv_s = e0.elapsed_time(e1) * 1e-3 / reps_p
    e0.record(stream)
    for i in range(reps_p):
        s.apply_A(dv[i % 4], out[i % 2])
    e1.record(stream)
    torch.cuda.synchronize()
    mv_s = e0.elapsed_time(e1) * 1e-3 / reps_p
    unknowns = w.unknowns
    mv_gbps = 16.0 * unknowns / mv_s / 1e9
    if w.dim == 1:  # K2 (8 B in, 16 B/complex out), K3 (in + out), K4: three passes
        pinv_gbps_structured = (16.0 * unknowns + 32.0 * (w.N // 2 + 1) * w.m + 16.0 * unknowns) / pinv_s / 1e9
    else:  # 2D: DST x, DST y, time pass, DST y, DST x — five real passes of 16 B per unknown
        pinv_gbps_structured = 80.0 * unknowns / pinv_s / 1e9
    del dv, out

    # ---------------- end to end through the host-buffer C-ABI call (pinned host memory)
    hshape = synth.shape_of(w)  # packed host layout: (N, m) in 1D, (N, n, n) in 2D
    bh = torch.empty(hshape, dtype=torch.float64, pin_memory=True)
    bh.copy_(b[..., : w.n].cpu())
    uh = torch.empty(hshape, dtype=torch.float64, pin_memory=True)
    bnp, unp = bh.numpy(), uh.numpy()
    s.gmres_host(bnp, w.tol, w.restart, u=unp)
    torch.cuda.synchronize()
    barrier(world)
    h0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        s.gmres_host(bnp, w.tol, w.restart, u=unp)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_t = e0.elapsed_time(e1) * 1e-3
    e2e_wall = time.perf_counter() - h0
    e2e_single = whole_job_throughput(args.steps, max(e2e_t, 1e-12), world)

    # ---------------- the same, with E handles on E CUDA streams driven by E host threads: one solve's
    # PCIe copies (H2D of b, D2H of u, ≈ 2.4 ms each way at c2) overlap another solve's GPU work.
    # Every step still copies its own input in and its result out; value = solves / wall time.
    import threading
    ne = max(1, args.e2e_streams)
    handles = [(s, stream, bnp, unp)]
    for _ in range(ne - 1):
        st_i = torch.cuda.Stream()
        with torch.cuda.stream(st_i):
            s_i = problems.make_solver(w, restart_max=w.restart)
        bh_i = torch.empty(hshape, dtype=torch.float64, pin_memory=True)
        bh_i.copy_(bh)
        uh_i = torch.empty(hshape, dtype=torch.float64, pin_memory=True)
        handles.append((s_i, st_i, bh_i.numpy(), uh_i.numpy()))
    counts = [args.steps // ne + (1 if i < args.steps % ne else 0) for i in range(ne)]
    reps_e2e = [None] * ne

    def drive(i):
        s_i, st_i, b_i, u_i = handles[i]
        with torch.cuda.stream(st_i):
            for _ in range(counts[i]):
                _, reps_e2e[i] = s_i.gmres_host(b_i, w.tol, w.restart, u=u_i)

    for i in range(ne):  # warm-up of every handle
        s_i, st_i, b_i, u_i = handles[i]
        with torch.cuda.stream(st_i):
            s_i.gmres_host(b_i, w.tol, w.restart, u=u_i)
    torch.cuda.synchronize()
    barrier(world)
    h1 = time.perf_counter()
    threads = [threading.Thread(target=drive, args=(i,)) for i in range(ne)]
    for t_ in threads:
        t_.start()
    for t_ in threads:
        t_.join()
    torch.cuda.synchronize()
    e2e_multi_wall = time.perf_counter() - h1
    assert all(r is None or r["converged"] for r in reps_e2e)
    assert all(np.array_equal(handles[i][3], unp) for i in range(1, ne))  # same solution on every handle
    e2e_value = whole_job_throughput(args.steps, max(e2e_multi_wall, 1e-12), world)
    del handles
    err_seq = None

    result = {
        "metric": METRIC,
        "value": value,
        "unit": "GMRES solves/s (time-to-tol^-1, whole job)",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (manufactured-solution rhs; seeded N(0,1) vectors, numpy default_rng)",
        "config": {"workload": describe(w), "N": w.N, "m": w.m, "alpha": w.alpha, "restart": w.restart,
                   "tol": w.tol, "parallelism": f"replicas x{world} (no data-path collective)",
                   "l2": "inputs larger than L2: one vector is %.0f MB; a solve streams ~%d vectors" %
                         (vec_bytes / 1e6, 50)},
        "gmres": {"iterations": its[-1], "relres_true": reps[-1]["relres_true"],
                  "time_to_tol_ms": 1e3 * t_max / args.steps, "history": reps[-1]["history"]},
        "pinv": {"applies_per_s": 1.0 / pinv_s, "ms": 1e3 * pinv_s,
                 "effective_GBps": 16.0 * unknowns / pinv_s / 1e9,
                 "structured_GBps": pinv_gbps_structured,
                 "structured_frac": pinv_gbps_structured / peak},
        "matvec": {"ms": 1e3 * mv_s, "GBps": mv_gbps, "frac": mv_gbps / peak},
        "stream_copy_GBps": copy_best,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic[0],
                     "traffic_launch": {"algo_bytes": traffic[1], "which": traffic[2]},
                     "algo_bytes_per_launch": d_by / d_cnt, "peak_source": peak_src,
                     "share_of_step": d_ms / total_prof_ms if total_prof_ms else None,
                     "frac_of_same_run_copy": achieved / copy_best if copy_best else None},
        "kernels": kernels,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": "GMRES solves/s (host buffers, pinned)",
                "streams": ne, "single_stream_value": e2e_single,
                "method": (f"cnpint_gmres_host on {ne} handles (own CUDA stream and workspace each) driven by "
                           f"{ne} host threads; each solve copies its b in and its u out inside the timed "
                           f"region; wall clock"),
                "h2d_bytes_per_step": int(w.unknowns * 8), "d2h_bytes_per_step": int(w.unknowns * 8),
                "wall_s": e2e_wall},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(w)
    return result


# ----------------------------------------------------------------------------------- CPU oracle
def oracle_solve(w):
    from oracle import aao, gmres, precond, problem
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    t0 = time.perf_counter()
    u, rep = gmres.gmres_right(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x), b,
                               w.tol, w.restart)
    return time.perf_counter() - t0, rep


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_baseline(w):
    dt, rep = oracle_solve(w)
    return {"value": 1.0 / dt, "unit": "GMRES solves/s", "cores": cores(), "kind": "oracle",
            "sample": f"1 full oracle GMRES({w.restart}) solve of {w.name} (numpy FFT + vectorised Thomas, MGS),"
                      f" {rep.iterations} its, {dt:.1f} s",
            "threads_note": "numpy/BLAS default threading (FFT and Thomas single-threaded)"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    w = workload(args.workload, args.alpha)
    for _ in range(min(args.warmup, 1)):
        oracle_solve(w)
    times, its = [], []
    budget = 150.0  # seconds: keep the reference arm within a few minutes (each solve ~20 s at c2)
    for _ in range(args.steps):
        dt, rep = oracle_solve(w)
        times.append(dt)
        its.append(rep.iterations)
        if sum(times) > budget:
            break
    tot = sum(times)
    args.steps = len(times)
    v = args.steps / tot
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "GMRES solves/s (time-to-tol^-1, whole job)",
            "n_gpus": world, "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": describe(w), "N": w.N, "m": w.m, "alpha": w.alpha},
            "gmres": {"iterations": its[-1]},
            "cpu_baseline": {"value": v, "unit": "GMRES solves/s", "cores": cores(), "kind": "oracle",
                             "sample": f"{args.steps} full oracle GMRES solves of {w.name}"},
            "e2e": {"value": v, "unit": "GMRES solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cnpint", choices=["cnpint", "reference"])
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--alpha", type=float, default=0.01)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-streams", type=int, default=4, help="concurrent handles for the e2e measurement")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "cnpint":
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    rank, world, local = dist_init()
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_gpu(args, rank, world, local)
    if rank == 0 and res is not None:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
