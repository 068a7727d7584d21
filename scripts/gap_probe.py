#!/usr/bin/env python
"""Where does a headline solve's wall time go?  Event-timed GMRES solves vs the sum of the per-class
kernel times (event profiler) of the same solves, and the host-measured time (report 'seconds').
  python scripts/gap_probe.py --workload c5_n511_N1024 [--reps 3]"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5_n511_N1024")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--debug", type=int, default=0)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2401_16113_b200 import problems
    w = synth.WORKLOADS[a.workload]
    s = problems.make_solver(w, restart_max=w.restart)
    if a.debug:
        s.set_debug(a.debug)
    b = problems.rhs(w, s)
    u = s.empty()
    st = torch.cuda.current_stream()
    for _ in range(2):
        s.gmres(b, u, w.tol, w.restart)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    reps = [s.gmres(b, u, w.tol, w.restart) for _ in range(a.reps)]
    e1.record(st)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.reps * 1e3
    ev = e0.elapsed_time(e1) / a.reps
    s.profile_enable(True)
    for _ in range(a.reps):
        s.gmres(b, u, w.tol, w.restart)
    torch.cuda.synchronize()
    prof = s.profile_read()
    s.profile_enable(False)
    ksum = sum(v[0] for v in prof.values()) / a.reps
    print(json.dumps({"workload": a.workload, "pdl": os.environ.get("CNPINT_PDL", "1"), "debug": a.debug, "event_ms": ev,
                      "host_wall_ms": wall, "report_seconds_ms": 1e3 * sum(r["seconds"] for r in reps) / a.reps,
                      "kernel_sum_ms": ksum, "gap_ms": ev - ksum, "iterations": reps[-1]["iterations"],
                      "classes": {k: round(v[0] / a.reps, 3) for k, v in prof.items()}}))


if __name__ == "__main__":
    main()
