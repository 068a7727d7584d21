"""Spectral statements of §3.2 evaluated on tiny dense matrices (ORACLE).

Test infrastructure only (see oracle/__init__.py).

PAPER.md:355-361 (Lemma 3.1)  P_α⁻¹𝓜 has (N−1)m eigenvalues equal to 1 and m equal to those of
                              (I − αJ_N)⁻¹, J_N = (Q1⁻¹Q2)^N.
PAPER.md:427-433 (Lemma 3.2)  −1 < Re λ(Q1⁻¹Q2) ≤ 1, |λ(Q1⁻¹Q2)| ≤ 1.
PAPER.md:597-602 (Eq. 4.2x)   λ(Q1⁻¹Q2) = (1 + μ/2)/(1 − μ/2), μ = λ(Ã).
PAPER.md:524-537 (Thm 3.1)    the m non-unit eigenvalues lie in Ω_α.
PAPER.md:213-220 (Thm 2.2)    σ_max(𝓜) ≤ 2 + τ‖A‖₂, σ_min(𝓜) ≥ 1/N.
"""
from __future__ import annotations

import numpy as np

from .aao import dense_M, dense_P, tau_of


def preconditioned_eigs(w, op, alpha=None) -> np.ndarray:
    """eig(P_α⁻¹𝓜) of the dense Kronecker matrices."""
    M = dense_M(w, op)
    P = dense_P(w, op, alpha)
    return np.linalg.eigvals(np.linalg.solve(P, M))


def step_eigs(w, op) -> np.ndarray:
    """eig(Q1⁻¹Q2) from the dense spatial matrix."""
    At = tau_of(w) * op.dense()
    I = np.eye(op.m)
    return np.linalg.eigvals(np.linalg.solve(I - 0.5 * At, I + 0.5 * At))


def closed_form_nonunit(w, op, alpha=None, mu=None) -> np.ndarray:
    """1/(1 − α g_j^N), g_j = (1 + μ_j/2)/(1 − μ_j/2), μ_j = eig(Ã) (Lemma 3.1 + Eq. 4.2x)."""
    alpha = w.alpha if alpha is None else alpha
    if mu is None:
        mu = np.linalg.eigvals(tau_of(w) * op.dense())
    g = (1 + 0.5 * mu) / (1 - 0.5 * mu)
    return 1.0 / (1.0 - alpha * g ** w.N)


def in_omega(z: np.ndarray, alpha: float, slack: float = 1e-10) -> np.ndarray:
    """Membership in Ω_α = {1/(1+α) ≤ |z| ≤ 1/(1−α), Re z > 0}."""
    a = np.abs(z)
    return (a >= 1.0 / (1.0 + alpha) - slack) & (a <= 1.0 / (1.0 - alpha) + slack) & (z.real > 0)


def singular_values_M(w, op) -> np.ndarray:
    return np.linalg.svd(dense_M(w, op), compute_uv=False)
