#!/usr/bin/env python
"""Phase timing of k_trivar from an experiment build with -DCNPINT_TRIVAR_TRACE (clock64 stamps per CTA):
per-phase cycles (median / mean), CTAs resident per SM over time.  CNPINT_LIB must point at that build.
  CNPINT_LIB=paper_2401_16113_b200/libcnpint_trace.so python scripts/trivar_trace.py --workload c3"""
import argparse, ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--debug", type=int, default=0)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2401_16113_b200 import problems
    w = synth.WORKLOADS[a.workload]
    s = problems.make_solver(w, 0)
    if a.debug:
        s.set_debug(a.debug)
    v = s.empty()
    v[..., : w.n] = torch.randn(v[..., : w.n].shape, dtype=torch.float64, device="cuda")
    z = s.empty()
    for _ in range(3):
        s.apply_Pinv(v, z)
    torch.cuda.synchronize()
    K = w.N // 2 + 1
    buf = (ctypes.c_longlong * (16384 * 10))()
    s.lib.cnpint_trivar_trace(buf, 16384 * 10)
    t = np.frombuffer(buf, dtype=np.int64).reshape(16384, 10)[:K]
    order = [0, 1, 2, 7, 3, 4, 5, 6]  # stamp 7: after the hand-over to warp 0
    ph = np.diff(t[:, order], axis=1)
    names = ["load", "sweep", "lower tree", "warp-0 tree", "lower down", "backsub", "store"]
    for i, n in enumerate(names):
        print(f"{n:9s} median {np.median(ph[:, i]):8.0f}  mean {ph[:, i].mean():8.0f} cycles")
    tot = t[:, 6] - t[:, 0]
    print(f"{'total':9s} median {np.median(tot):8.0f}  mean {tot.mean():8.0f} cycles")
    sm = t[:, 9]
    for smid in np.unique(sm)[:6]:
        sel = t[sm == smid]
        ev = sorted([(x, 1) for x in sel[:, 0]] + [(x, -1) for x in sel[:, 6]])
        cur = area = 0
        last = ev[0][0]
        for x, d in ev:
            area += cur * (x - last)
            cur += d
            last = x
        span = sel[:, 6].max() - sel[:, 0].min()
        print(f"sm {int(smid):3d}: {len(sel)} CTAs, span {span} cycles, mean resident {area / span:.2f}")


if __name__ == "__main__":
    main()
