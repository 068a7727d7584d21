#!/usr/bin/env python
"""K5 alternative: the DST-I of every line as a dense fp64
product on the tensor cores (DMMA) vs the FFT sine pass.  The dense product Y = X · S (X: all lines of
one axis, S the n×n DST-I matrix) is timed through cuBLAS DGEMM (torch.matmul, fp64: DMMA on sm_100),
an upper bound for any hand-written mma.sync kernel, next to the same-run DMMA / FMA ceilings
(cnpint_peak_kernel) and the K5 pass of the library on the same shape.  Prints one JSON line."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synth
    from paper_2401_16113_b200 import problems
    from paper_2401_16113_b200.cnpint import peak_kernel
    out = {}
    dev = torch.device("cuda")
    scratch = torch.empty(8 * 148 * 256 * 2, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    for kind, name in ((0, "fma"), (1, "dmma")):
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); fl = peak_kernel(kind, scratch, 4096); e1.record(st); e1.synchronize()
            best = max(best, fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        out[f"{name}_peak_TFLOPs"] = best
    for wname in ("c4", "c5_n127_N1024", "c5_n511_N256"):
        w = synth.WORKLOADS[wname]
        n, M = w.n, w.n + 1
        lines = w.N * w.n                    # x pass: every (t, y) row
        S = torch.tensor([[math.sqrt(2.0 / M) * math.sin(math.pi * (i + 1) * (j + 1) / M) for j in range(n)]
                          for i in range(n)], dtype=torch.float64, device=dev)
        X = torch.randn(lines, n, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        for _ in range(3):
            torch.matmul(X, S, out=Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(st)
        for _ in range(reps):
            torch.matmul(X, S, out=Y)
        e1.record(st)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / reps
        flops = 2.0 * lines * n * n
        del X, Y
        # the library's K5 x pass on the same workload (P⁻¹ applies, profiled per kernel class)
        s = problems.make_solver(w)
        v = s.empty()
        v[..., :n] = torch.randn(v[..., :n].shape, dtype=torch.float64, device=dev)
        z = s.empty()
        s.apply_Pinv(v, z)
        torch.cuda.synchronize()
        s.profile_enable(True)
        for _ in range(5):
            s.apply_Pinv(v, z)
        prof = s.profile_read()
        s.profile_enable(False)
        ms, cnt, by = prof["K5_dst_x"]
        out[wname] = {"dense_dgemm_us": 1e6 * t, "dense_TFLOPs": flops / t / 1e12,
                      "dense_frac_of_dmma_peak": flops / t / 1e12 / out["dmma_peak_TFLOPs"],
                      "fft_sine_pass_us": 1e3 * ms / cnt, "dense_over_fft": 1e6 * t / (1e3 * ms / cnt),
                      "dense_flops_per_unknown": 2 * n, "lines": lines, "n": n}
        del s, v, z
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
