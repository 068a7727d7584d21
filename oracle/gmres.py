"""Restarted right-preconditioned GMRES (ORACLE).

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
    history: list = field(default_factory=list)     # |g_{j+1}|/‖b‖ after every inner step


def gmres_right(A, Pinv, b: np.ndarray, tol: float, restart: int, maxit: int = 1000,
                reorth: bool = True):
    """Right-preconditioned restarted GMRES(restart) with x0 = 0.

    A, Pinv: callables on arrays shaped like b.  Returns (u, GmresReport).  If maxit is reached
    inside a cycle, the cycle is closed (u updated) and the report says converged=False — so
    gmres_right(..., maxit=j) returns the j-th GMRES iterate for j ≤ restart."""
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
            if est <= tol or breakdown or rep.iterations >= maxit:
                break
        y = np.zeros(j_done)                             # back substitution H y = g
        for i in range(j_done - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j_done] @ y[i + 1:j_done]) / H[i, i]
        u = u + Pf(V[:j_done].T @ y)                     # u = u0 + P⁻¹ V y
        r = bv - Af(u)
        rep.relres_est = est
        rep.relres_true = float(np.linalg.norm(r)) / bnorm
        if rep.relres_true <= tol:
            rep.converged = True
            return u.reshape(shape), rep
        if rep.iterations >= maxit:
            return u.reshape(shape), rep
        rep.restarts += 1
