"""Restarted right- and left-preconditioned GMRES and the Theorem 4.5 rate bound (ORACLE).

Test infrastructure only (see oracle/__init__.py).

PAPER.md:795 (§5): "the right-preconditioned GMRES solver (with restarting number being 40) ...
with a zero initial guess and a stopping tolerance tol ... based on the reduction in relative
residual norms"; right preconditioning is chosen because "its termination criterion is based on the
reliable true residuals".  Reading #15: solve 𝓜P⁻¹y = b, u = P⁻¹y, stop when the
Givens estimate |g_{j+1}|/‖b‖ ≤ tol, then confirm the true residual ‖b − 𝓜u‖/‖b‖ ≤ tol at the end
of the cycle (otherwise restart).  "Iterations" = total inner Arnoldi steps.  Orthogonalisation is
modified Gram-Schmidt with one reorthogonalisation pass (reading #17).

The algorithm is the textbook one (Saad, Iterative Methods, Alg. 6.9 / 9.5), written step by step.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class GmresReport:
    iterations: int = 0
    restarts: int = 0
    converged: bool = False
    relres_est: float = float("nan")
    relres_true: float = float("nan")
    relres_prec: float = float("nan")                # left preconditioning: ‖P⁻¹(b − 𝓜u)‖/‖P⁻¹b‖
    history: list = field(default_factory=list)     # |g_{j+1}|/‖b‖ after every inner step


def gmres_right(A, Pinv, b: np.ndarray, tol: float, restart: int, maxit: int = 1000,
                reorth: bool = True, iterates: list | None = None):
    """Right-preconditioned restarted GMRES(restart) with x0 = 0.

    A, Pinv: callables on arrays shaped like b.  Returns (u, GmresReport).  If maxit is reached
    inside a cycle, the cycle is closed (u updated) and the report says converged=False — so
    gmres_right(..., maxit=j) returns the j-th GMRES iterate for j ≤ restart.
    iterates (test mode): if a list is given, the iterate
    x_j = u0 + P⁻¹V_j y_j of every inner step j is formed (one extra P⁻¹ per step, by the same
    back substitution as the cycle end) and appended — the same vectors maxit=j would return."""
    shape = b.shape
    bv = b.reshape(-1)
    bnorm = float(np.linalg.norm(bv))
    rep = GmresReport()
    u = np.zeros_like(bv)
    if bnorm == 0.0:
        rep.converged, rep.relres_est, rep.relres_true = True, 0.0, 0.0
        return u.reshape(shape), rep
    Af = lambda x: A(x.reshape(shape)).reshape(-1)
    Pf = lambda x: Pinv(x.reshape(shape)).reshape(-1)
    r = bv.copy()                      # x0 = 0 ⇒ r0 = b

    def backsolve(H, g, k):                             # y = H[:k,:k]⁻¹ g[:k] (upper triangular)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        return y

    def combine(V, y):                                  # V_k y, basis rows kept as a list
        s = np.zeros_like(bv)
        for i in range(y.size):
            s += y[i] * V[i]
        return s

    while True:
        beta = float(np.linalg.norm(r))
        V = [None] * (restart + 1)                      # basis vectors (allocated as produced)
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        est = beta / bnorm
        for j in range(restart):
            w = Af(Pf(V[j]))
            rep.iterations += 1
            for i in range(j + 1):                       # MGS
                H[i, j] = float(V[i] @ w)
                w = w - H[i, j] * V[i]
            if reorth:                                   # one reorthogonalisation pass
                for i in range(j + 1):
                    c = float(V[i] @ w)
                    H[i, j] += c
                    w = w - c * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            breakdown = H[j + 1, j] == 0.0
            if not breakdown:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                           # apply previous Givens rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = float(np.hypot(H[j, j], H[j + 1, j]))  # new rotation zeroing H[j+1, j]
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / bnorm
            rep.history.append(est)
            j_done = j + 1
            if iterates is not None:
                iterates.append((u + Pf(combine(V, backsolve(H, g, j_done)))).reshape(shape))
            if est <= tol or breakdown or rep.iterations >= maxit:
                break
        y = backsolve(H, g, j_done)                      # back substitution H y = g
        u = u + Pf(combine(V, y))                        # u = u0 + P⁻¹ V y
        r = bv - Af(u)
        rep.relres_est = est
        rep.relres_true = float(np.linalg.norm(r)) / bnorm
        if rep.relres_true <= tol:
            rep.converged = True
            return u.reshape(shape), rep
        if rep.iterations >= maxit:
            return u.reshape(shape), rep
        rep.restarts += 1


def gmres_left(A, Pinv, b: np.ndarray, tol: float, restart: int, maxit: int = 1000,
               reorth: bool = True):
    """Left-preconditioned restarted GMRES(restart) with x0 = 0.

    PAPER.md:576-583 (§4): GMRES "exploited to the left-preconditioned system
    P_α⁻¹𝓜u^(k) = P_α⁻¹b" with residual r_k := P_α⁻¹(b − 𝓜u^(k)) and the minimal residual property
    ‖r_k‖ = min_{p ∈ ℙ_k, p(0)=1} ‖p(P_α⁻¹𝓜) r_0‖ (Eq. sss2x); Theorem 4.5 bounds
    ‖r_k‖/‖r_0‖.  Textbook algorithm (Saad, Iterative Methods, Alg. 9.4), step by step:
    r0 = P⁻¹b, β = ‖r0‖, v_1 = r0/β; w = P⁻¹𝓜v_j; Gram-Schmidt; Givens; u = u0 + V y.
    history[k−1] = |g_k|/‖r_0‖ is the Givens value of ‖r_k‖/‖r_0‖ (r_0 of the first cycle).
    Stops when that estimate ≤ tol, then confirms the true preconditioned residual
    ‖P⁻¹(b − 𝓜u)‖/‖P⁻¹b‖ ≤ tol at the cycle end (else restarts).  The report's relres_true is the
    unpreconditioned ‖b − 𝓜u‖/‖b‖; relres_prec the preconditioned one."""
    shape = b.shape
    bv = b.reshape(-1)
    rep = GmresReport()
    u = np.zeros_like(bv)
    Af = lambda x: A(x.reshape(shape)).reshape(-1)
    Pf = lambda x: Pinv(x.reshape(shape)).reshape(-1)
    bnorm = float(np.linalg.norm(bv))
    if bnorm == 0.0:
        rep.converged, rep.relres_est, rep.relres_true = True, 0.0, 0.0
        rep.relres_prec = 0.0
        return u.reshape(shape), rep
    r = Pf(bv)                         # x0 = 0 ⇒ r0 = P⁻¹b
    r0norm = float(np.linalg.norm(r))
    while True:
        beta = float(np.linalg.norm(r))
        V = np.zeros((restart + 1, bv.size))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        est = beta / r0norm
        for j in range(restart):
            w = Pf(Af(V[j]))
            rep.iterations += 1
            for i in range(j + 1):                       # MGS
                H[i, j] = float(V[i] @ w)
                w = w - H[i, j] * V[i]
            if reorth:
                for i in range(j + 1):
                    c = float(V[i] @ w)
                    H[i, j] += c
                    w = w - c * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            breakdown = H[j + 1, j] == 0.0
            if not breakdown:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / r0norm
            rep.history.append(est)
            j_done = j + 1
            if est <= tol or breakdown or rep.iterations >= maxit:
                break
        y = np.zeros(j_done)
        for i in range(j_done - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j_done] @ y[i + 1:j_done]) / H[i, i]
        u = u + V[:j_done].T @ y                         # u = u0 + V y (no P⁻¹: left preconditioning)
        res = bv - Af(u)
        r = Pf(res)
        rep.relres_est = est
        rep.relres_true = float(np.linalg.norm(res)) / bnorm
        rep.relres_prec = float(np.linalg.norm(r)) / r0norm
        if rep.relres_prec <= tol:
            rep.converged = True
            return u.reshape(shape), rep
        if rep.iterations >= maxit:
            return u.reshape(shape), rep
        rep.restarts += 1


def rate_bound(alpha: float, tau: float, T: float):
    """Theorem 4.5: with α = δ√(τ/T), δ ∈ (0, ½), the left-preconditioned GMRES
    residuals satisfy ‖r_k‖/‖r_0‖ ≤ [1 − (1 − 2α√(T/τ))²]^{k/2} ≤ [1 − (1 − 2δ)²]^{k/2}.
    Returns (δ, rate) with δ = α√(T/τ) and rate = [1 − (1 − 2δ)²]^{1/2} = 2√(δ(1 − δ)); raises
    ValueError when δ ∉ (0, ½) (the theorem's hypothesis fails).
    Reading R27: the paper's last equality prints [2√δ(1 − δ)]^k, which is not equal to
    the middle expression (1 − (1 − 2δ)² = 4δ(1 − δ)); the bound proved by Eq. 4.12 is the middle
    one, so that is the rate here.  printed_rate() gives the printed value for comparison."""
    delta = alpha * np.sqrt(T / tau)
    if not (0.0 < delta < 0.5):
        raise ValueError(f"Theorem 4.5 needs 0 < delta < 1/2, got {delta}")
    return float(delta), float(np.sqrt(1.0 - (1.0 - 2.0 * delta) ** 2))


def printed_rate(delta: float) -> float:
    """The rate as printed at the end of Theorem 4.5: 2√δ(1 − δ) (see reading R27)."""
    return float(2.0 * np.sqrt(delta) * (1.0 - delta))


def rate_bound_check(history, alpha: float, tau: float, T: float, slack: float = 1e-12):
    """SPEC.md:368-376 rate_bound_check: does every history ratio ‖r_k‖/‖r_0‖ (k = 1, 2, …) satisfy
    the Theorem 4.5 bound rate^k?  history must come from a single left-preconditioned cycle (no
    restart).  Returns dict(holds, delta, bound_rate, worst, printed_rate, holds_printed) with
    worst = max_k history_k / rate^k; the *_printed entries test the stricter printed rate (R27)."""
    delta, rate = rate_bound(alpha, tau, T)
    ratios = [float(h) / rate ** (k + 1) for k, h in enumerate(history)]
    worst = max(ratios) if ratios else 0.0
    pr = printed_rate(delta)
    holds_pr = all(float(h) <= pr ** (k + 1) * (1.0 + slack) for k, h in enumerate(history))
    return {"holds": worst <= 1.0 + slack, "delta": delta, "bound_rate": rate, "worst": worst,
            "printed_rate": pr, "holds_printed": holds_pr}
