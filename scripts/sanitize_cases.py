#!/usr/bin/env python
"""Small solves through the C ABI for compute-sanitizer (memcheck / racecheck / synccheck): each case
runs P_α⁻¹, 𝓜u and a GMRES solve on one shape that selects a given kernel family.  No oracle.

  compute-sanitizer --tool racecheck python scripts/sanitize_cases.py --case c1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    # 1D, cluster time FFT (N = 256), Toeplitz fast tree K3, Gram CGS2, fused post ops, PDL
    "c1": ("C1", None, None, 0),
    # 1D four-step persistent time FFT (N = 2048: spin-waits on acquire counters), generic K3 tree
    "fourstep": ("C1", 63, 2048, 0),
    # 1D variable rows (K3 MODE_VAR)
    "var": ("C3", 127, 256, 0),
    # 2D: DST passes + cluster time pass (N = 1024: thread-block clusters, DSMEM)
    "cluster2d": ("C4", 15, 1024, 0),
    # 2D: register time pass (N = 256) + register y DST (n = 255, E = 512)
    "reg2d": ("C4", 255, 8, 0),
    # 2D: the TMA bulk-copy DST ring (k_dst2, debug 256), n = 127
    "dst2": ("C4", 127, 16, 256),
    # classic CGS2 second pass (debug 128)
    "classic": ("C1", 63, 64, 128),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c1", choices=list(CASES))
    args = ap.parse_args()
    import torch

    import synth
    from paper_2401_16113_b200 import problems
    base, n, N, dbg = CASES[args.case]
    w = getattr(synth, base)
    if n is not None:
        w = synth.scaled(w, n, N, alpha=0.05, restart=10)
    w = w.with_(restart=min(w.restart, 10))
    s = problems.make_solver(w, restart_max=w.restart)
    s.set_debug(dbg)
    v = s.empty()
    v[..., : w.n] = torch.randn(v[..., : w.n].shape, dtype=torch.float64, device="cuda",
                                generator=torch.Generator(device="cuda").manual_seed(1))
    z = s.empty()
    for _ in range(2):
        s.apply_Pinv(v, z)
        s.apply_A(v, z)
    u = s.empty()
    rep = s.gmres(problems.rhs(w, s), u, 1e-10, w.restart)
    torch.cuda.synchronize()
    assert s.device_status() == 0
    print(f"case {args.case}: {w.name} its {rep['iterations']} converged {rep['converged']}")


if __name__ == "__main__":
    main()
