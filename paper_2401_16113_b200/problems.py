"""Caller-side problem setup for the BASELINE.json workloads (product side).

Builds the spatial operator L_h handed to ``cnpint_create`` and the right-hand side b = ξ + τf of
Eq. 2.2 on the device with torch fp64.  Forming b is the caller's job in the
cnpint ABI; this module is the repo's own caller.  It is written independently of
``oracle/`` (which builds the same objects in numpy for the parity tests) and shares only the
parameter table in ``synth``.

Discretisation (BASELINE.json configs): second-order central differences on h = (b−a)/(n+1),
x_i = a + i h, homogeneous Dirichlet boundaries (every manufactured solution vanishes there).
"""
from __future__ import annotations

import math

import numpy as np

from .cnpint import OperatorSpec


def grid(w):
    lo_, hi_ = w.domain
    h = (hi_ - lo_) / (w.n + 1)
    return h, lo_ + h * np.arange(1, w.n + 1, dtype=np.float64)


def operator_spec(w) -> OperatorSpec:
    """L_h for workload w (not multiplied by τ)."""
    h, x = grid(w)
    if w.kind == "logprice":                       # (σ²/2)∂xx + (r − σ²/2)∂x − r, constant rows
        d2 = 0.5 * w.sigma ** 2 / h ** 2
        d1 = (w.r - 0.5 * w.sigma ** 2) / (2.0 * h)
        return OperatorSpec(dim=1, nx=w.n, toeplitz=True, xs=d2 - d1, xd=-2.0 * d2 - w.r, xu=d2 + d1)
    if w.kind == "price":                          # (σ²S²/2)∂SS + rS∂S − r, S_i = x_i
        d2 = 0.5 * w.sigma ** 2 * x * x / h ** 2
        d1 = w.r * x / (2.0 * h)
        return OperatorSpec(dim=1, nx=w.n, toeplitz=False, sub=d2 - d1, diag=-2.0 * d2 - w.r, sup=d2 + d1)
    if w.kind == "bs2d":                           # Σ_d (σ_d²/2)∂dd + (r − σ_d²/2)∂d, − r once
        s1, s2 = w.sigma2
        ax2, ax1 = 0.5 * s1 * s1 / h ** 2, (w.r - 0.5 * s1 * s1) / (2.0 * h)
        ay2, ay1 = 0.5 * s2 * s2 / h ** 2, (w.r - 0.5 * s2 * s2) / (2.0 * h)
        return OperatorSpec(dim=2, nx=w.n, ny=w.n, xs=ax2 - ax1, xd=-2.0 * ax2, xu=ax2 + ax1,
                            ys=ay2 - ay1, yd=-2.0 * ay2, yu=ay2 + ay1, shift=-w.r)
    raise ValueError(w.kind)


def d_time(w, t):
    """d(t) of a time-dependent operator 𝓛(t) = d(t)𝓛: exp(−dt_rate·t)."""
    return math.exp(-w.dt_rate * t)


def d_half(w) -> np.ndarray:
    """The N values d(t_{k+½}) handed to cnpint_set_time_dependence (D̃ of Eq. 5.8)."""
    tau = w.T / w.N
    return np.array([d_time(w, (k + 0.5) * tau) for k in range(w.N)])


def _exact_and_source(w, x, t):
    """(u(x, t), f(x, t)) of the manufactured solution, f = ∂_t u − d(t)𝓛u (analytic 𝓛)."""
    import torch
    lo_, hi_ = w.domain
    e = math.exp(-t)
    if w.kind == "logprice":
        k = math.pi / (hi_ - lo_)
        s, c = torch.sin(k * (x - lo_)), torch.cos(k * (x - lo_))
        u = e * s
        mu = w.r - 0.5 * w.sigma ** 2
        Lu = (-0.5 * w.sigma ** 2 * k * k - w.r) * u + mu * k * e * c
        return u, -u - d_time(w, t) * Lu
    if w.kind == "price":
        L = hi_
        u = e * x * (L - x) / (L * L)
        uS = e * (L - 2.0 * x) / (L * L)
        uSS = -2.0 * e / (L * L)
        Lu = 0.5 * w.sigma ** 2 * x * x * uSS + w.r * x * uS - w.r * u
        return u, -u - d_time(w, t) * Lu
    k = math.pi / (hi_ - lo_)
    s, c = torch.sin(k * (x - lo_)), torch.cos(k * (x - lo_))
    s1, s2 = w.sigma2
    u = e * s[:, None] * s[None, :]                         # [y][x]
    ux = e * s[:, None] * c[None, :] * k
    uy = e * c[:, None] * s[None, :] * k
    Lu = -(0.5 * (s1 * s1 + s2 * s2) * k * k + w.r) * u + (w.r - 0.5 * s1 * s1) * ux + (w.r - 0.5 * s2 * s2) * uy
    return u, -u - d_time(w, t) * Lu


def _apply_L_torch(spec: OperatorSpec, u):
    """L_h u for one time slice (caller-side input assembly of ξ = Q2 u⁰ only)."""
    import torch
    if spec.dim == 1:
        if spec.toeplitz:
            lo, di, up = spec.xs, spec.xd, spec.xu
            y = di * u
            y[1:] += lo * u[:-1]
            y[:-1] += up * u[1:]
            return y
        dev = u.device
        lo, di, up = (torch.as_tensor(a, device=dev) for a in (spec.sub, spec.diag, spec.sup))
        y = di * u
        y[1:] += lo[1:] * u[:-1]
        y[:-1] += up[:-1] * u[1:]
        return y
    y = (spec.xd + spec.yd + spec.shift) * u
    y[:, 1:] += spec.xs * u[:, :-1]
    y[:, :-1] += spec.xu * u[:, 1:]
    y[1:, :] += spec.ys * u[:-1, :]
    y[:-1, :] += spec.yu * u[1:, :]
    return y


def rhs(w, solver):
    """b = ξ + τf as a zero-padded device vector in the solver's layout:
    b_t = τ f(·, (t+½)τ), plus (I + ½d(t_½)τL_h) u⁰ in block 0 (d ≡ 1 unless 𝓛(t) = d(t)𝓛, Eq. 5.8).
    Every manufactured solution here is u = e^{−t}φ(x), so f(x, t) = e^{−t}(−φ − d(t)𝓛φ) and the
    time dependence is an outer product."""
    import torch
    spec = operator_spec(w)
    _, xs = grid(w)
    x = torch.as_tensor(xs, dtype=torch.float64, device=solver.device)
    tau = w.T / w.N
    phi, f0 = _exact_and_source(w.with_(dt_rate=0.0), x, 0.0)
    Lphi = -phi - f0                                          # 𝓛φ (continuous operator)
    th = (torch.arange(w.N, dtype=torch.float64, device=solver.device) + 0.5) * tau
    et = torch.exp(-th)
    dt = torch.exp(-w.dt_rate * th)
    b = solver.empty()
    shape = (w.N,) + (1,) * phi.dim()
    b[..., : w.n] = tau * et.reshape(shape) * (-phi - dt.reshape(shape) * Lphi)
    b[0, ..., : w.n] += phi + 0.5 * d_time(w, 0.5 * tau) * tau * _apply_L_torch(spec, phi.clone())
    return b


def exact(w, solver):
    """u(x, t_k), k = 1..N as a padded device vector (manufactured solution)."""
    import torch
    _, xs = grid(w)
    x = torch.as_tensor(xs, dtype=torch.float64, device=solver.device)
    tau = w.T / w.N
    phi, _ = _exact_and_source(w, x, 0.0)
    et = torch.exp(-(torch.arange(w.N, dtype=torch.float64, device=solver.device) + 1.0) * tau)
    u = solver.empty()
    u[..., : w.n] = et.reshape((w.N,) + (1,) * phi.dim()) * phi
    return u


def make_solver(w, restart_max: int = 0, alpha: float | None = None):
    from .cnpint import Solver
    s = Solver(w.N, w.T, w.alpha if alpha is None else alpha, operator_spec(w), restart_max)
    if w.dt_rate:
        s.set_time_dependence(d_half(w))
    return s
