#!/usr/bin/env python
"""BASELINE.json configs[4] sweep on one B200: GMRES(20) iterations, time-to-solution, P_α⁻¹ and 𝓜
throughput against the measured HBM peak, for n ∈ {127, 255, 511} × N ∈ {256, 1024}; the CPU oracle
solve on the two smallest sizes.  Prints one JSON document (profiles/r01_c5_sweep.json)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import synth
    from paper_2401_16113_b200 import problems
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rows = []
    for n, N in synth.C5_SIZES:
        w = synth.c5(n, N)
        s = problems.make_solver(w, restart_max=w.restart)
        b = problems.rhs(w, s)
        u = s.empty()
        for _ in range(2):
            rep = s.gmres(b, u, w.tol, w.restart)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            rep = s.gmres(b, u, w.tol, w.restart)
        e1.record()
        torch.cuda.synchronize()
        t_solve = e0.elapsed_time(e1) / reps
        ue = problems.exact(w, s)
        err = float((u - ue).abs().max() / ue.abs().max())
        v = s.empty()
        v[..., : w.n] = torch.randn(v[..., : w.n].shape, dtype=torch.float64, device="cuda")
        z = s.empty()
        for _ in range(3):
            s.apply_Pinv(v, z)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            s.apply_Pinv(v, z)
        e1.record()
        torch.cuda.synchronize()
        t_p = e0.elapsed_time(e1) / 10
        e0.record()
        for _ in range(10):
            s.apply_A(v, z)
        e1.record()
        torch.cuda.synchronize()
        t_a = e0.elapsed_time(e1) / 10
        units = w.unknowns
        row = {"n": n, "N": N, "unknowns": units, "iterations": rep["iterations"], "relres_true": rep["relres_true"],
               "time_to_tol_ms": t_solve, "max_rel_err_vs_exact": err,
               "pinv_ms": t_p, "pinv_applies_per_s": 1e3 / t_p,
               "pinv_effective_GBps": 16.0 * units / (t_p * 1e-3) / 1e9,
               "pinv_structured_GBps": 80.0 * units / (t_p * 1e-3) / 1e9,
               "matvec_ms": t_a, "matvec_GBps": 16.0 * units / (t_a * 1e-3) / 1e9,
               "matvec_frac_of_peak": 16.0 * units / (t_a * 1e-3) / 1e9 / peak}
        rows.append(row)
        print(json.dumps(row), file=sys.stderr)
        del s, b, u, v, z, ue
        torch.cuda.empty_cache()
    oracle = []
    if "--no-oracle" not in sys.argv:
        from oracle import aao, gmres, precond, problem
        for n, N in synth.C5_SIZES[:2]:
            w = synth.c5(n, N)
            op = problem.build_operator(w)
            b = problem.assemble_rhs(w, op)
            t0 = time.perf_counter()
            uo, rep = gmres.gmres_right(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x), b,
                                        w.tol, w.restart)
            dt = time.perf_counter() - t0
            oracle.append({"n": n, "N": N, "iterations": rep.iterations, "seconds": dt,
                           "cores": len(os.sched_getaffinity(0))})
    print(json.dumps({"config": "BASELINE.json configs[4]", "hbm_peak_GBps": peak,
                      "pinv_structured_note": "2D P^-1 = 5 passes (DST x, DST y, time pass, DST y, DST x) = 80 B/unknown",
                      "gpu": rows, "oracle_cpu": oracle}, indent=1))


if __name__ == "__main__":
    main()
