"""NEXT #4 evidence: left-preconditioned GMRES histories on the GPU against Theorem 4.5's bound
(reading R27), and left vs right GMRES timing at c2.  One JSON line per case."""
import json
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2401_16113_b200 import problems, theory  # noqa: E402


def run(w, side, random_rhs=False):
    s = problems.make_solver(w, w.restart)
    b = s.to_device(synth.random_vectors(w, 1, 5)[0]) if random_rhs else problems.rhs(w, s)
    u = s.empty()
    s.gmres(b, u, w.tol, w.restart, side=side)  # warm
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    reps = 5
    for _ in range(reps):
        rep = s.gmres(b, u, w.tol, w.restart, side=side)
    ev[1].record()
    torch.cuda.synchronize()
    rep["ms"] = ev[0].elapsed_time(ev[1]) / reps
    return rep


for delta in (0.1, 0.25, 0.45):
    for N in (256, 1024, 4096, 16384):
        w = synth.heat(min(N - 1, 4095), N, delta).with_(tol=1e-12)
        rep = run(w, "left", random_rhs=True)
        chk = theory.rate_bound_check(rep["history"], w.alpha, N, w.T)
        print(json.dumps({"case": "theorem45", "rhs": "seeded N(0,1), seed 5", "delta": delta, "N": N, "m": w.n, "alpha": w.alpha,
                          "iterations": rep["iterations"], "history": rep["history"],
                          "relres_prec": rep["relres_prec"], "relres_true": rep["relres_true"],
                          "bound_rate": chk["bound_rate"], "printed_rate": chk["printed_rate"],
                          "worst_ratio_to_bound": chk["worst"], "holds": chk["holds"],
                          "holds_printed": chk["holds_printed"]}), flush=True)
for alpha in synth.C2_ALPHAS:
    w = synth.C2.with_(alpha=alpha)
    for side in ("right", "left"):
        rep = run(w, side)
        print(json.dumps({"case": "c2_side", "alpha": alpha, "side": side, "iterations": rep["iterations"],
                          "ms": rep["ms"], "relres_true": rep["relres_true"],
                          "relres_prec": rep.get("relres_prec"), "history": rep["history"]}), flush=True)
