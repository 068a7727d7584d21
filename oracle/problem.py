"""Grid, spatial operator L_h, manufactured solution and AaO right-hand side (ORACLE).

Test infrastructure only (see oracle/__init__.py).

PAPER.md:29-36 (Eq. 1.1)  ∂_t u = 𝓛u + f,  u(·,0) = u_0.
PAPER.md:40-46 (Eq. 1.2)  𝓛 = self-adjoint elliptic operator with drift and reaction.
PAPER.md:117-132 (§2.1, Eq. 2.1) CN with f sampled at t_{k+1/2}.
PAPER.md:184-203 (§2.2, Eq. 2.2) 𝓜u = ξ + τf := b,  ξ = [(I + ½Ã)u⁰; 0; …; 0],  Ã = τA.

The operators are the Black-Scholes ones of BASELINE.json:
second-order central differences, homogeneous Dirichlet boundaries, h = (b-a)/(m+1),
x_i = a + i h (i = 1..m).  Every manufactured solution vanishes on the boundary, so no
boundary source appears.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Operator1D:
    """Tridiagonal L_h: (L_h u)_i = lo[i] u_{i-1} + di[i] u_i + up[i] u_{i+1}, u_0 = u_{m+1} = 0."""
    lo: np.ndarray
    di: np.ndarray
    up: np.ndarray
    x: np.ndarray          # interior nodes
    h: float

    @property
    def m(self) -> int:
        return self.di.size

    def dense(self) -> np.ndarray:
        m = self.m
        A = np.diag(self.di)
        A[np.arange(1, m), np.arange(0, m - 1)] = self.lo[1:]
        A[np.arange(0, m - 1), np.arange(1, m)] = self.up[:-1]
        return A


@dataclass
class Operator2D:
    """L_h = I_y ⊗ L_x + L_y ⊗ I_x + shift·I with L_x = tridiag(xs, xd, xu), L_y = tridiag(ys, yd, yu)
    Toeplitz; vectors are [y][x], x fastest (SURVEY.md §8(c) reading #9)."""
    xs: float
    xd: float
    xu: float
    ys: float
    yd: float
    yu: float
    shift: float
    n: int
    x: np.ndarray
    h: float

    @property
    def m(self) -> int:
        return self.n * self.n

    def Lx(self) -> np.ndarray:
        return _toeplitz_tridiag(self.n, self.xs, self.xd, self.xu)

    def Ly(self) -> np.ndarray:
        return _toeplitz_tridiag(self.n, self.ys, self.yd, self.yu)

    def dense(self) -> np.ndarray:
        I = np.eye(self.n)
        return np.kron(I, self.Lx()) + np.kron(self.Ly(), I) + self.shift * np.eye(self.m)


def _toeplitz_tridiag(n: int, s: float, d: float, u: float) -> np.ndarray:
    return np.diag(np.full(n, d)) + np.diag(np.full(n - 1, s), -1) + np.diag(np.full(n - 1, u), 1)


def build_operator(w):
    """Central-difference Black-Scholes operator of workload ``w`` (BASELINE.json configs).

    logprice (configs[0], [1]):  L = (σ²/2)∂xx + (r − σ²/2)∂x − r
        rows lo = σ²/(2h²) − μ/(2h), di = −σ²/h² − r, up = σ²/(2h²) + μ/(2h), μ = r − σ²/2.
    price (configs[2]):          L = (σ²S²/2)∂SS + rS∂S − r,  S_i = a + i h
        rows lo_i = σ²S_i²/(2h²) − rS_i/(2h), di_i = −σ²S_i²/h² − r, up_i = σ²S_i²/(2h²) + rS_i/(2h).
    bs2d (configs[3], [4]):      L = Σ_d (σ_d²/2)∂dd + (r − σ_d²/2)∂d − r  (−r once, reading #9).
    """
    a, b = w.domain
    n = w.n
    h = (b - a) / (n + 1)
    x = a + h * np.arange(1, n + 1)
    if w.kind == "logprice":
        s2, mu = w.sigma ** 2, w.r - 0.5 * w.sigma ** 2
        lo = np.full(n, s2 / (2 * h * h) - mu / (2 * h))
        di = np.full(n, -s2 / (h * h) - w.r)
        up = np.full(n, s2 / (2 * h * h) + mu / (2 * h))
        return Operator1D(lo, di, up, x, h)
    if w.kind == "price":
        S = x
        s2 = w.sigma ** 2
        lo = s2 * S * S / (2 * h * h) - w.r * S / (2 * h)
        di = -s2 * S * S / (h * h) - w.r
        up = s2 * S * S / (2 * h * h) + w.r * S / (2 * h)
        return Operator1D(lo, di, up, x, h)
    if w.kind == "bs2d":
        (s1, s2) = w.sigma2
        t1, m1 = s1 * s1, w.r - 0.5 * s1 * s1
        t2, m2 = s2 * s2, w.r - 0.5 * s2 * s2
        return Operator2D(xs=t1 / (2 * h * h) - m1 / (2 * h), xd=-t1 / (h * h), xu=t1 / (2 * h * h) + m1 / (2 * h),
                          ys=t2 / (2 * h * h) - m2 / (2 * h), yd=-t2 / (h * h), yu=t2 / (2 * h * h) + m2 / (2 * h),
                          shift=-w.r, n=n, x=x, h=h)
    raise ValueError(w.kind)


def apply_L(op, u: np.ndarray) -> np.ndarray:
    """L_h applied along the trailing spatial axes of u (any leading batch axes)."""
    if isinstance(op, Operator1D):
        y = op.di * u
        y[..., 1:] += op.lo[1:] * u[..., :-1]
        y[..., :-1] += op.up[:-1] * u[..., 1:]
        return y
    y = (op.xd + op.yd + op.shift) * u
    y[..., :, 1:] += op.xs * u[..., :, :-1]
    y[..., :, :-1] += op.xu * u[..., :, 1:]
    y[..., 1:, :] += op.ys * u[..., :-1, :]
    y[..., :-1, :] += op.yu * u[..., 1:, :]
    return y


# ---------------------------------------------------------------------------------------------
# Manufactured solutions (BASELINE.json) and the analytic source f = ∂_t u − 𝓛u (continuous 𝓛,
# SURVEY.md §8(c) reading #8).
# ---------------------------------------------------------------------------------------------

def u_exact(w, op, t: float) -> np.ndarray:
    a, b = w.domain
    if w.kind == "logprice":
        k = math.pi / (b - a)
        return math.exp(-t) * np.sin(k * (op.x - a))
    if w.kind == "price":
        return math.exp(-t) * op.x * (b - op.x) / (b * b)   # S(300−S)/300², a = 0
    k = math.pi / (b - a)
    sx = np.sin(k * (op.x - a))
    return math.exp(-t) * np.outer(sx, sx)                  # [y][x]


def d_of(w, t: float) -> float:
    """Time factor of 𝓛(t) = d(t)𝓛: d(t) = exp(−dt_rate·t); 1 when dt_rate = 0."""
    return math.exp(-w.dt_rate * t)


def f_source(w, op, t: float) -> np.ndarray:
    """f = ∂_t u − d(t)𝓛u for the manufactured u (continuous 𝓛; d ≡ 1 unless dt_rate ≠ 0)."""
    return _minus_u(w, op, t) - d_of(w, t) * _L_exact(w, op, t)


def _minus_u(w, op, t: float) -> np.ndarray:
    return -u_exact(w, op, t)   # ∂_t u = −u for every manufactured u = e^{−t}φ(x)


def _L_exact(w, op, t: float) -> np.ndarray:
    """𝓛u of the manufactured solution (continuous operator, analytic derivatives)."""
    a, b = w.domain
    e = math.exp(-t)
    if w.kind == "logprice":
        k = math.pi / (b - a)
        s2, mu = w.sigma ** 2, w.r - 0.5 * w.sigma ** 2
        u = e * np.sin(k * (op.x - a))
        ux = e * k * np.cos(k * (op.x - a))
        uxx = -k * k * u
        return 0.5 * s2 * uxx + mu * ux - w.r * u
    if w.kind == "price":
        S = op.x
        u = e * S * (b - S) / (b * b)
        uS = e * (b - 2 * S) / (b * b)
        uSS = -2.0 * e / (b * b)
        return 0.5 * w.sigma ** 2 * S * S * uSS + w.r * S * uS - w.r * u
    k = math.pi / (b - a)
    (s1, s2) = w.sigma2
    m1, m2 = w.r - 0.5 * s1 * s1, w.r - 0.5 * s2 * s2
    sx, cx = np.sin(k * (op.x - a)), np.cos(k * (op.x - a))
    u = e * np.outer(sx, sx)                 # [y][x]
    ux = e * k * np.outer(sx, cx)            # derivative along x (fast axis)
    uy = e * k * np.outer(cx, sx)
    return 0.5 * s1 * s1 * (-k * k * u) + 0.5 * s2 * s2 * (-k * k * u) + m1 * ux + m2 * uy - w.r * u


def assemble_rhs(w, op) -> np.ndarray:
    """b = ξ + τf (Eq. 2.2; SURVEY.md §8(c) reading #7):
    b_t = τ f(·, (t+½)τ) for t = 0..N−1 and b_0 += (I + ½Ã) u⁰ with Ã = τ L_h; with 𝓛(t) = d(t)𝓛
    the ξ block is (I + ½d(t_½)Ã)u⁰ (Eq. 5.8)."""
    N, tau = w.N, w.T / w.N
    b = np.stack([tau * f_source(w, op, (t + 0.5) * tau) for t in range(N)])
    u0 = u_exact(w, op, 0.0)
    b[0] += u0 + 0.5 * d_of(w, 0.5 * tau) * tau * apply_L(op, u0)
    return b


def exact_blocks(w, op) -> np.ndarray:
    """u(·, t_k) for k = 1..N, stacked as the AaO unknown (block t holds u^{t+1})."""
    tau = w.T / w.N
    return np.stack([u_exact(w, op, (t + 1) * tau) for t in range(w.N)])
