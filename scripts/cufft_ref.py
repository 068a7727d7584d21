"""Reference point only (not product code): cuFFT (via torch.fft) on the same strided shapes."""
import torch
def t(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for N, W in [(4096, 4096), (512, 65280), (16384, 1024)]:
    x = torch.randn(N, W, dtype=torch.float64, device="cuda")
    us = t(lambda: torch.fft.rfft(x, dim=0))
    y = torch.fft.rfft(x, dim=0)
    us2 = t(lambda: torch.fft.irfft(y, n=N, dim=0))
    by = N * W * 8 + (N // 2 + 1) * W * 16
    print(f"cuFFT rfft dim0 N={N} W={W}: {us:.1f} us ({by/us/1e3:.0f} GB/s); irfft {us2:.1f} us ({by/us2/1e3:.0f} GB/s)")
    xt = x.t().contiguous()
    us3 = t(lambda: torch.fft.rfft(xt, dim=1))
    print(f"   contiguous rfft (batch {W} x {N}): {us3:.1f} us ({by/us3/1e3:.0f} GB/s)")
