"""A/B of GMRES variants selected by cnpint_set_debug bits: time-to-tolerance (CUDA events), iterations,
true relative residual, and the relative difference of the solutions between the variants."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2401_16113_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="c2,c3,c4")
ap.add_argument("--debugs", default="0,128")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
for wn in args.workloads.split(","):
    w = synth.WORKLOADS[wn]
    s = problems.make_solver(w, restart_max=w.restart)
    b = problems.rhs(w, s)
    sols = {}
    for dbg in [int(x) for x in args.debugs.split(",")]:
        s.set_debug(dbg)
        u = s.empty()
        rep = s.gmres(b, u, w.tol, w.restart)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            rep = s.gmres(b, u, w.tol, w.restart)
        e1.record()
        torch.cuda.synchronize()
        sols[dbg] = u.clone()
        r = rep
        print(json.dumps({"workload": wn, "debug": dbg, "ms": e0.elapsed_time(e1) / args.reps,
                          "iterations": r["iterations"], "relres_true": r["relres_true"],
                          "history": r.get("history")}))
    ks = list(sols)
    for k in ks[1:]:
        d = (sols[k] - sols[ks[0]]).norm() / sols[ks[0]].norm()
        print(json.dumps({"workload": wn, "rel_diff_debug": [ks[0], k], "value": float(d)}))
    s.set_debug(0)
