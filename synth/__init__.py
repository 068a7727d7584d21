"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic.  It contains only

* the workload parameter table transcribed from BASELINE.json ``configs``
  (grid sizes, PDE coefficients, domains, alpha, GMRES settings), and
* the seeded random-vector generator (SURVEY.md §8(c) reading #23:
  ``numpy.random.default_rng(seed).standard_normal((count, N, m))``, C order,
  fp64).

Operators, right-hand sides, transforms and solvers are implemented twice,
independently: once in ``oracle/`` (plain CPU reference) and once on the
product side (``paper_2401_16113_b200``).  Neither side imports the other;
both import this module.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Tuple

import numpy as np


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json workload (notation of SURVEY.md §0: N = time steps,
    m = spatial unknowns; PAPER.md uses M for time steps and N for space)."""

    name: str
    dim: int                 # 1 or 2
    kind: str                # "logprice" (1D Toeplitz), "price" (1D variable), "bs2d"
    n: int                   # interior points per axis (1D: m = n; 2D: m = n*n)
    N: int                   # time steps (power of two)
    T: float                 # horizon
    alpha: float             # preconditioner parameter in (0, 1)
    restart: int             # GMRES restart length
    tol: float = 1e-10       # relative residual tolerance
    sigma: float = 0.0       # 1D volatility
    r: float = 0.0           # interest rate
    domain: Tuple[float, float] = (0.0, 1.0)      # 1D interval / 2D square side
    sigma2: Tuple[float, float] = (0.0, 0.0)      # 2D volatilities (sigma1, sigma2)
    rand_count: int = 4      # number of N(0,1) random vectors for P^-1 / A checks
    rand_seed: int = 1
    note: str = ""
    # time-varying operator 𝓛(t) = d(t)𝓛 with d(t) = exp(−dt_rate·t) (Eq. 5.8;
    # SURVEY.md §8(f) NEXT #1); 0 = the constant-coefficient method of BASELINE.json.
    dt_rate: float = 0.0

    @property
    def m(self) -> int:
        return self.n if self.dim == 1 else self.n * self.n

    @property
    def unknowns(self) -> int:
        return self.N * self.m

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)


LN100 = math.log(100.0)

# BASELINE.json configs[0]: 1D Black-Scholes, log-price, m=255, N=256, alpha=0.01, GMRES(50),
# 16 random vectors from seed 0.
C1 = Workload(name="c1", dim=1, kind="logprice", n=255, N=256, T=1.0, alpha=0.01, restart=50,
              sigma=0.3, r=0.05, domain=(LN100 - 3.0, LN100 + 3.0), rand_count=16, rand_seed=0,
              note="BASELINE.json configs[0]")
# configs[1]: same operator at m=4095, N=4096, alpha in {0.1, 0.01, 0.001}, GMRES(30), seed 1.
C2 = C1.with_(name="c2", n=4095, N=4096, restart=30, rand_count=4, rand_seed=1,
              note="BASELINE.json configs[1] (alpha in {0.1, 0.01, 0.001})")
C2_ALPHAS = (0.1, 0.01, 0.001)
# configs[2]: price-space S in [0,300], variable coefficients, m=1023, N=16384, T=5.
# Restart unspecified -> 40 (the paper's value, SURVEY.md §8(c) reading #16).
C3 = Workload(name="c3", dim=1, kind="price", n=1023, N=16384, T=5.0, alpha=0.01, restart=40,
              sigma=0.25, r=0.03, domain=(0.0, 300.0), rand_count=4, rand_seed=1,
              note="BASELINE.json configs[2]")
# configs[3]: 2D uncorrelated two-asset BS in log prices on [-3,3]^2, n=255, N=512.
C4 = Workload(name="c4", dim=2, kind="bs2d", n=255, N=512, T=1.0, alpha=0.01, restart=40,
              r=0.05, domain=(-3.0, 3.0), sigma2=(0.3, 0.2), rand_count=4, rand_seed=1,
              note="BASELINE.json configs[3]")


def c5(n: int, N: int) -> Workload:
    """configs[4]: mesh-independence sweep on the 2D operator, GMRES(20)."""
    assert n in (127, 255, 511) and N in (256, 1024)
    return C4.with_(name=f"c5_n{n}_N{N}", n=n, N=N, restart=20, note="BASELINE.json configs[4]")


C5_SIZES = [(n, N) for n in (127, 255, 511) for N in (256, 1024)]

# SURVEY.md §8(f) NEXT #1 (not a BASELINE config): the c1 / c2 operator with 𝓛(t) = e^{−t/2}𝓛, the
# shape of the paper's Set V variant (d(t) = e^{−rt}), strengthened so that d
# varies by 40 % over the horizon.
C1T = C1.with_(name="c1t", dt_rate=0.5, note="NEXT #1: c1 operator with d(t) = exp(-t/2)")
C2T = C2.with_(name="c2t", dt_rate=0.5, note="NEXT #1: c2 operator with d(t) = exp(-t/2)")

def heat(n: int, N: int, delta: float = 0.25, T: float = 1.0) -> Workload:
    """SURVEY.md §8(f) NEXT #4 (Theorem 4.5; SPEC.md:374's "symmetric 1D heat"):
    the c1 log-price operator with r = σ²/2, which removes the convection term so L = (σ²/2)∂xx − r is
    symmetric negative definite (the theorem's hypothesis), and Theorem 4.5's
    α = δ√(τ/T) with τ = T/N.  Parameters only."""
    tau = T / N
    return C1.with_(name=f"heat_n{n}_N{N}_d{delta}", n=n, N=N, T=T, r=0.5 * C1.sigma ** 2,
                    alpha=delta * math.sqrt(tau / T), restart=40,
                    note="NEXT #4: symmetric heat-type operator, alpha = delta*sqrt(tau/T)")


WORKLOADS = {w.name: w for w in (C1, C2, C3, C4, C1T, C2T)}
for _n, _N in C5_SIZES:
    WORKLOADS[f"c5_n{_n}_N{_N}"] = c5(_n, _N)


def shape_of(w: Workload) -> Tuple[int, ...]:
    """Logical (unpadded) shape of one space-time vector: (N, m) or (N, n, n), x fastest."""
    return (w.N, w.n) if w.dim == 1 else (w.N, w.n, w.n)


def random_vectors(w: Workload, count: int | None = None, seed: int | None = None) -> np.ndarray:
    """i.i.d. N(0,1) fp64 vectors, shape (count, *shape_of(w)), C order.

    SURVEY.md §8(c) reading #23.  The same bits serve the oracle and the GPU path."""
    count = w.rand_count if count is None else count
    seed = w.rand_seed if seed is None else seed
    rng = np.random.default_rng(seed)
    return rng.standard_normal((count,) + shape_of(w))


def scaled(w: Workload, n: int, N: int, **kw) -> Workload:
    """The same operator family at another mesh (used by small parity cases and the
    second-order study)."""
    return w.with_(name=f"{w.name}_n{n}_N{N}", n=n, N=N, **kw)
