#!/usr/bin/env python
"""Short driver for ncu captures and per-op event timings: builds one workload's solver and runs a
few P_α⁻¹ / 𝓜 applies (or one GMRES solve) through the C ABI.  No oracle involved.

  python scripts/prof_ops.py --workload c2 --op pinv --reps 3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--op", default="pinv", choices=["pinv", "A", "gmres", "all"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--time", action="store_true", help="print per-kernel event timings (not under ncu)")
    ap.add_argument("--debug", type=int, default=0, help="cnpint_set_debug flags (kernel-variant selection)")
    args = ap.parse_args()
    import torch

    import synth
    from paper_2401_16113_b200 import problems

    w = synth.WORKLOADS[args.workload]
    if args.alpha is not None:
        w = w.with_(alpha=args.alpha)
    s = problems.make_solver(w, restart_max=w.restart if args.op in ("gmres", "all") else 0)
    if args.debug:
        s.set_debug(args.debug)
    rng = torch.Generator(device="cuda").manual_seed(1)
    vs = []
    for _ in range(2):
        v = s.empty()
        v[..., : w.n] = torch.randn(v[..., : w.n].shape, dtype=torch.float64, device="cuda", generator=rng)
        vs.append(v)
    out = s.empty()

    def run_once(i):
        if args.op in ("pinv", "all"):
            s.apply_Pinv(vs[i % 2], out)
        if args.op in ("A", "all"):
            s.apply_A(vs[i % 2], out)
        if args.op in ("gmres", "all"):
            s.gmres(problems.rhs(w, s), out, w.tol, w.restart)

    if args.time:
        run_once(0)  # warm-up (lazy module loading, first-touch)
        torch.cuda.synchronize()
        s.profile_enable(True)
    for i in range(args.reps):
        if args.op in ("pinv", "all"):
            s.apply_Pinv(vs[i % 2], out)
        if args.op in ("A", "all"):
            s.apply_A(vs[i % 2], out)
        if args.op in ("gmres", "all"):
            b = problems.rhs(w, s)
            s.gmres(b, out, w.tol, w.restart)
    torch.cuda.synchronize()
    if args.time:
        prof = s.profile_read()
        res = {k: {"avg_us": 1e3 * ms / n, "launches": n, "algo_GBps": by / (ms * 1e-3) / 1e9 if by else None}
               for k, (ms, n, by) in prof.items()}
        print(json.dumps({"workload": w.name, "op": args.op, "kernels": res}))
    assert s.device_status() == 0


if __name__ == "__main__":
    main()
