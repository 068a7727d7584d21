#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for cnpint (arxiv 2401.16113 hot path on B200).

Workload (N=1): BASELINE.json's metric names no config, so the headline is the largest single-GPU
configuration: configs[4] at n = 511, N = 1024 ("c5_n511_N1024": 2D Black–Scholes, 261,121 spatial
unknowns x 1024 steps = 267 M fp64 unknowns), α = 0.01, GMRES(20), tol 1e-10, zero initial guess,
manufactured-solution right-hand side b (synthetic, resident in HBM).

Step = one full right-preconditioned GMRES solve to tolerance — every row of SURVEY.md §8(a):
K1 AaO matvec, P_α⁻¹ (2D: K5 sine passes + K6 fused time pass; 1D: K2/K3/K4), K7 CGS2 Arnoldi
passes, K8 Givens/Hessenberg on device, K9 cycle end.  value = GMRES solves/s (time-to-tolerance⁻¹),
whole job over all ranks.  Alongside: P_α⁻¹ applies/s, AaO matvec GB/s and their fraction of the
measured HBM peak, K0 stream-copy GB/s, same-run fp64 FMA / DMMA ceilings, the per-kernel breakdown
(CUDA events on the launch stream), the live roofline of the dominant kernel, the end-to-end number
through the host-buffer C-ABI call, a per-workload table of every other BASELINE config (c1, c2 at
three α, c3, c4, the other c5 sizes) and the CPU oracle on the same box.

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
        tab = json.load(open(p))
        for key in (f"{kernel}@{workload}", kernel):
            d = tab.get(key)
            if d and d.get("workload") == workload:
                return d["bytes_per_launch"], d.get("algo_bytes_this_launch"), d.get("launch")
    return None, None, None


# ----------------------------------------------------------------------------------- workload
HEADLINE = "c5_n511_N1024"   # BASELINE.json configs[4] at its largest size (267 M unknowns, one GPU)
UNIT = "GMRES solves/s (time-to-tol^-1, whole job)"
# the per-workload table (same run): every other BASELINE config
TABLE = [("c1", None), ("c2", 0.1), ("c2", 0.01), ("c2", 0.001), ("c3", None), ("c4", None),
         ("c5_n127_N256", None), ("c5_n127_N1024", None), ("c5_n255_N256", None), ("c5_n255_N1024", None),
         ("c5_n511_N256", None)]


def workload(name: str, alpha: float | None):
    import synth
    w = synth.WORKLOADS[name]
    return w.with_(alpha=alpha) if alpha is not None else w


def describe(w):
    return (f"{w.name}: {w.note}; {w.kind} Black-Scholes, N={w.N} steps x m={w.m} unknowns "
            f"({w.unknowns:,} fp64), T={w.T}, alpha={w.alpha}, GMRES({w.restart}) tol {w.tol}, x0=0")


def fused_2d_sine(w, debug=0):
    """True when the 2D P_α⁻¹ runs as three passes: the fused x+y sine pass k_dstxy (opt-in, debug
    bit 32768; n + 1 ∈ {64, …, 512}, launch_dstxy in k_dstxy.cu).  The bench runs debug 0: five."""
    return w.dim == 2 and w.n + 1 in (64, 128, 256, 512) and bool(debug & 32768)


def pinv_structured_bytes(w):
    """Algorithmic bytes of one P_α⁻¹ as structured: 1D K2 + K3 + K4 (8 B in, 16 B per
    half-spectrum complex out / in + out / in, 8 B out); 2D W⁻¹, time pass, W: 3 × 16 B with the fused
    x+y sine pass, else W⁻¹ (x, y), time pass, W (y, x): 5 × 16 B."""
    if w.dim == 1:
        return 16.0 * w.unknowns + 32.0 * (w.N // 2 + 1) * w.m + 16.0 * w.unknowns
    return (48.0 if fused_2d_sine(w) else 80.0) * w.unknowns


def time_ops(s, w, stream, nvec, reps):
    """Standalone P⁻¹ and 𝓜 rates on nvec seeded N(0,1) vectors (each > L2 at the large configs)."""
    import torch
    import synth
    V = synth.random_vectors(w, nvec, w.rand_seed)
    dv = [s.to_device(v) for v in V]
    del V
    out = [s.empty() for _ in range(2)]
    for i in range(3):
        s.apply_Pinv(dv[i % nvec], out[0])
        s.apply_A(dv[i % nvec], out[1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(reps):
        s.apply_Pinv(dv[i % nvec], out[i % 2])
    e1.record(stream)
    torch.cuda.synchronize()
    pinv_s = e0.elapsed_time(e1) * 1e-3 / reps
    e0.record(stream)
    for i in range(reps):
        s.apply_A(dv[i % nvec], out[i % 2])
    e1.record(stream)
    torch.cuda.synchronize()
    mv_s = e0.elapsed_time(e1) * 1e-3 / reps
    del dv, out
    return pinv_s, mv_s


def op_rates(w, pinv_s, mv_s, peak):
    st = pinv_structured_bytes(w) / pinv_s / 1e9
    mv = 16.0 * w.unknowns / mv_s / 1e9
    return ({"applies_per_s": 1.0 / pinv_s, "ms": 1e3 * pinv_s, "effective_GBps": 16.0 * w.unknowns / pinv_s / 1e9,
             "structured_GBps": st, "structured_frac": st / peak},
            {"ms": 1e3 * mv_s, "GBps": mv, "frac": mv / peak})


def peak_ceilings(dev):
    """Same-run fp64 compute ceilings: dependent-FMA and mma.sync f64 (DMMA) loops."""
    import torch
    from paper_2401_16113_b200.cnpint import peak_kernel
    out = torch.empty(8 * 148 * 256 * 2, dtype=torch.float64, device=dev)
    res = {}
    stream = torch.cuda.current_stream()
    for kind, name in ((0, "fp64_fma_TFLOPs"), (1, "fp64_dmma_TFLOPs")):
        best = 0.0
        peak_kernel(kind, out, 256)
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fl = peak_kernel(kind, out, 4096)
            e1.record(stream)
            e1.synchronize()
            best = max(best, fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        res[name] = best
    res["how"] = ("cnpint_peak_kernel: 8 CTAs x 256 threads per SM, 4096 rounds of 8 dependent-FMA chains per "
                  "thread / 4 mma.sync.m8n8k4 f64 accumulators per warp; best of 5, CUDA events")
    return res


# ----------------------------------------------------------------------------------- GPU arm
def run_gpu(args, rank, world, local):
    import numpy as np
    import torch

    from paper_2401_16113_b200 import problems
    from paper_2401_16113_b200.cnpint import stream_copy

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = workload(args.workload, args.alpha)
    peak, peak_src = measured_hbm_peak()
    stream = torch.cuda.current_stream()

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
    ceilings = peak_ceilings(dev)

    s = problems.make_solver(w, restart_max=w.restart)
    b = problems.rhs(w, s)
    u = s.empty()
    vec_bytes = s.vec_elems * 8

    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    for _ in range(args.warmup):
        rep = s.gmres(b, u, w.tol, w.restart)
    torch.cuda.synchronize()
    # ---------------- timed region: K full GMRES solves (inputs resident in HBM)
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
    for _ in range(args.steps):
        s.gmres(b, u, w.tol, w.restart)
    torch.cuda.synchronize()
    prof = s.profile_read()
    s.profile_enable(False)
    kernels = {}
    for name, (ms, cnt, by) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        kernels[name] = {"ms_per_step": ms / args.steps, "launches_per_step": cnt / args.steps,
                         "avg_launch_us": 1e3 * ms / cnt, "algo_GBps": (by / (ms * 1e-3) / 1e9) if by else None}
    for k in kernels.values():
        k["frac"] = k["algo_GBps"] / peak if k["algo_GBps"] else None
    dominant = max(prof.items(), key=lambda kv: kv[1][0] if kv[1][2] > 0 else -1)[0]
    d_ms, d_cnt, d_by = prof[dominant]
    achieved = d_by / (d_ms * 1e-3) / 1e9
    total_prof_ms = sum(v[0] for v in prof.values())
    traffic = ncu_traffic(dominant, w.name)

    # ---------------- 2D: the same solves with the time pass as Eq. 3.2's transform (Γ_α·FFT, ÷, iFFT·Γ_α⁻¹ on chip,
    # debug 524288) instead of the default recurrence form (k_tscan.cu) — both compute the same P_α⁻¹
    k6_alt = None
    if w.dim == 2:
        s.set_debug(524288)
        s.gmres(b, u, w.tol, w.restart)
        s.profile_enable(True)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        nalt = max(2, min(5, args.steps))
        for _ in range(nalt):
            ralt = s.gmres(b, u, w.tol, w.restart)
        f1.record(stream)
        torch.cuda.synchronize()
        palt = s.profile_read()
        s.profile_enable(False)
        s.set_debug(0)
        k6 = palt.get("K6_time_pass_2d")
        k6_alt = {"transform_path_ms_per_step": f0.elapsed_time(f1) / nalt, "iterations": ralt["iterations"],
                  "K6_transform_avg_launch_us": 1e3 * k6[0] / k6[1] if k6 else None,
                  "K6_default_avg_launch_us": kernels.get("K6_time_pass_2d", {}).get("avg_launch_us"),
                  "note": "default = recurrence form of the alpha-circulant time block (k_tscan); transform = "
                          "cnpint_set_debug(524288): FFT along time, divide by lambda1_k - lambda2_k*mu, inverse FFT"}

    # ---------------- standalone P⁻¹ applies/s and matvec GB/s
    pinv_s, mv_s = time_ops(s, w, stream, 2 if w.unknowns > 1e8 else 4, max(10, args.steps))
    pinv_d, mv_d = op_rates(w, pinv_s, mv_s, peak)

    # ---------------- end to end through the host-buffer C-ABI call (pinned host memory): every step
    # copies its b in (H2D) and its u out (D2H) inside the timed region
    import synth
    hshape = synth.shape_of(w)
    bh = torch.empty(hshape, dtype=torch.float64, pin_memory=True)
    bh.copy_(b[..., : w.n].cpu())
    uh = torch.empty(hshape, dtype=torch.float64, pin_memory=True)
    bnp, unp = bh.numpy(), uh.numpy()
    e2e = run_e2e(s, w, stream, bnp, unp, args.steps, world)
    del bh, uh, u
    result = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (manufactured-solution rhs; seeded N(0,1) vectors, numpy default_rng)",
        "config": {"workload": describe(w), "name": w.name, "N": w.N, "m": w.m, "alpha": w.alpha,
                   "restart": w.restart, "tol": w.tol,
                   "parallelism": f"replicas x{world} (no data-path collective)",
                   "l2": "inputs larger than L2: one vector is %.0f MB (L2 126 MB); a solve streams ~50 vectors" %
                         (vec_bytes / 1e6)},
        "gmres": {"iterations": its[-1], "relres_true": reps[-1]["relres_true"],
                  "time_to_tol_ms": 1e3 * t_max / args.steps, "history": reps[-1]["history"]},
        "pinv": pinv_d,
        "matvec": mv_d,
        "stream_copy_GBps": copy_best,
        "compute_ceilings": ceilings,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic[0],
                     "traffic_launch": {"algo_bytes": traffic[1], "which": traffic[2]},
                     "algo_bytes_per_launch": d_by / d_cnt, "peak_source": peak_src,
                     "share_of_step": d_ms / total_prof_ms if total_prof_ms else None,
                     "frac_of_same_run_copy": achieved / copy_best if copy_best else None},
        "kernels": kernels,
        "time_pass_variants": k6_alt,
        "gpu_launches": launches,
        "e2e": e2e,
        "clocks": clk,
    }
    del s, b
    torch.cuda.empty_cache()
    if not args.no_table and world == 1:  # the per-workload table is a single-GPU measurement
        result["workloads"] = workload_table(args, peak, stream)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(w)
    return result


def run_e2e(s, w, stream, bnp, unp, steps, world):
    """E2E through cnpint_gmres_host_batch: every step copies its b in from pinned host memory and its u
    back out; the library overlaps the H2D of b_{i+1} and the D2H of u_{i−1} with solve i (two copy
    streams), so the measured rate is max(compute, PCIe) per solve.  value = solves / wall time."""
    import torch
    u2 = torch.empty(unp.shape, dtype=torch.float64, pin_memory=True).numpy()
    outs = [unp if i % 2 == 0 else u2 for i in range(steps)]
    stage = torch.empty(4 * s.vec_elems, dtype=torch.float64, device=s.device)
    s.gmres_host_batch([bnp, bnp], [unp, u2], w.tol, w.restart, stage=stage)   # warm-up (streams, events)
    torch.cuda.synchronize()
    barrier(world)
    h1 = time.perf_counter()
    reps = s.gmres_host_batch([bnp] * steps, outs, w.tol, w.restart, stage=stage)
    torch.cuda.synchronize()
    wall = time.perf_counter() - h1
    assert all(r["converged"] for r in reps)
    del stage
    return {"value": whole_job_throughput(steps, max(wall, 1e-12), world), "unit": UNIT, "streams": 1,
            "method": ("cnpint_gmres_host_batch on one handle: each step copies its b in (H2D) and its u out (D2H) "
                       "between pinned host memory and the device, overlapped with the neighbouring solves on two "
                       "copy streams; wall clock over all steps"),
            "h2d_bytes_per_step": int(w.unknowns * 8), "d2h_bytes_per_step": int(w.unknowns * 8),
            "wall_s": wall}


def workload_table(args, peak, stream):
    """Every other BASELINE config in the same run: GMRES time-to-tol (5 solves, CUDA events), P⁻¹
    applies/s and structured GB/s, matvec GB/s, kernel breakdown of one solve."""
    import torch

    from paper_2401_16113_b200 import problems
    rows = []
    for name, alpha in TABLE:
        w = workload(name, alpha)
        s = problems.make_solver(w, restart_max=w.restart)
        b = problems.rhs(w, s)
        u = s.empty()
        for _ in range(3):
            s.gmres(b, u, w.tol, w.restart)
        torch.cuda.synchronize()
        nrep = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(nrep):
            rep = s.gmres(b, u, w.tol, w.restart)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / nrep
        s.profile_enable(True)
        s.gmres(b, u, w.tol, w.restart)
        prof = s.profile_read()
        s.profile_enable(False)
        pinv_s, mv_s = time_ops(s, w, stream, 4 if w.unknowns < 1e8 else 2, 10)
        pd, md = op_rates(w, pinv_s, mv_s, peak)
        rows.append({"workload": w.name, "alpha": w.alpha, "N": w.N, "m": w.m, "unknowns": w.unknowns,
                     "iterations": rep["iterations"], "relres_true": rep["relres_true"],
                     "time_to_tol_ms": 1e3 * t, "solves_per_s": 1.0 / t,
                     "pinv_applies_per_s": pd["applies_per_s"], "pinv_structured_GBps": pd["structured_GBps"],
                     "pinv_structured_frac": pd["structured_frac"], "matvec_GBps": md["GBps"],
                     "matvec_frac": md["frac"],
                     "kernels_us": {k: {"us_per_launch": 1e3 * ms / cnt, "launches": cnt,
                                        "frac": (by / (ms * 1e-3) / 1e9 / peak) if by else None}
                                    for k, (ms, cnt, by) in prof.items()}})
        del s, b, u
        torch.cuda.empty_cache()
    return rows


# ----------------------------------------------------------------------------------- CPU oracle
def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return sorted({(i.get("internal_api"), i.get("num_threads")) for i in threadpool_info()})
    except Exception:
        return None


def time_slab(w, n_slab=32):
    """The bounded sample of a workload: the same operator, mesh, τ, α and GMRES settings on the first
    n_slab of its N time steps (T scaled so τ is unchanged).  A solve's oracle work is linear in N up to
    the FFT's log factor, so (N / n_slab) × the sample's time ≈ (slightly under) the full solve's."""
    if w.N <= n_slab:
        return w, 1.0
    return w.with_(name=f"{w.name}_slab{n_slab}", N=n_slab, T=w.T * n_slab / w.N), w.N / n_slab


def oracle_solve(w):
    from oracle import aao, gmres, precond, problem
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    t0 = time.perf_counter()
    u, rep = gmres.gmres_right(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x), b,
                               w.tol, w.restart)
    return time.perf_counter() - t0, rep


def cpu_baseline(w):
    """The oracle as it stands on the host cores: one GMRES solve of the bounded sample (time_slab),
    scaled to the full workload, plus the oracle's 𝓜u (median of 3) and P⁻¹ (once; ~30-60 s at the
    headline size) on full-size vectors (the per-operation baseline SURVEY.md §8(d) asks for)."""
    import numpy as np

    import synth
    from oracle import aao, precond, problem
    ws, scale = time_slab(w)
    dt, rep = oracle_solve(ws)
    res = {"value": 1.0 / (dt * scale), "unit": UNIT, "cores": cores(), "kind": "oracle",
           "cpu_model": cpu_model(), "blas_threads": str(blas_threads()),
           "sample": (f"1 oracle GMRES({ws.restart}) solve of {ws.name} (the headline operator, mesh, tau, alpha "
                      f"on {ws.N} of its {w.N} time steps; numpy FFT + dense-DST / Thomas shifted solves, "
                      f"MGS), {rep.iterations} its, {dt:.1f} s, scaled x{scale:g} to the full workload")}
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 1)[0]
    tm = []
    for _ in range(3):
        t0 = time.perf_counter()
        aao.apply_M(w, op, v)
        tm.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    precond.pinv_dft(w, op, v)
    tp = time.perf_counter() - t0
    res["per_op_full_size"] = {"apply_M_s_median_of_3": float(np.median(tm)), "apply_Pinv_s_1_run": tp,
                               "workload": w.name, "unknowns": w.unknowns}
    return res


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (oracle/, numpy) on the GPU arm's workload, metric and unit —
    each step one oracle GMRES solve of the bounded sample (time_slab), scaled to the full workload
    (steps and warm-up exactly as given); rank 0 only."""
    if rank != 0:
        return None
    w = workload(args.workload, args.alpha)
    ws, scale = time_slab(w)
    for _ in range(args.warmup):
        oracle_solve(ws)
    times, its = [], []
    for _ in range(args.steps):
        dt, rep = oracle_solve(ws)
        times.append(dt * scale)
        its.append(rep.iterations)
    tot = sum(times)
    v = args.steps / tot
    sample = (f"each step: 1 oracle GMRES({ws.restart}) solve of {ws.name} ({ws.N} of the {w.N} time steps, "
              f"same operator/mesh/tau/alpha), its time x{scale:g}")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (manufactured-solution rhs)",
            "config": {"workload": describe(w), "name": w.name, "N": w.N, "m": w.m, "alpha": w.alpha,
                       "restart": w.restart, "tol": w.tol,
                       "parallelism": f"replicas x{world} (no data-path collective)",
                       "l2": "n/a (CPU)"},
            "gmres": {"iterations": its[-1]},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores(), "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cnpint", choices=["cnpint", "reference"])
    ap.add_argument("--workload", default=HEADLINE)
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-table", action="store_true", help="skip the per-workload table")
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
