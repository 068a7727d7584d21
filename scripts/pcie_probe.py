"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (two streams), 134 MB buffers."""
import json
import time

import torch

n = 4096 * 4095
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = n * 8


def run(h2d, d2h, reps=10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    return round(B * (h2d + d2h) / dt / 1e9, 1), round(dt * 1e3, 3)


run(1, 1, 2)
print(json.dumps({"h2d_GBps_ms": run(1, 0), "d2h_GBps_ms": run(0, 1), "both_GBps_ms": run(1, 1)}))
