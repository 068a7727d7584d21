"""Theorem 4.5 of the paper as a host-side check on a GMRES history.

With α = δ√(τ/T), δ ∈ (0, ½), left-preconditioned GMRES (cnpint_gmres_left) satisfies
‖r_k‖/‖r_0‖ ≤ [1 − (1 − 2α√(T/τ))²]^{k/2} = [1 − (1 − 2δ)²]^{k/2} = (2√(δ(1 − δ)))^k, for a
symmetric negative semi-definite spatial matrix.  The paper prints the last form as [2√δ(1 − δ)]^k,
which does not equal the middle one; reading R27 takes the proved (middle) rate and
reports the printed one beside it.  SPEC.md:368-376 (rate_bound_check) is the interface model.
"""
from __future__ import annotations

import math
from typing import Sequence


def theorem_4_5_rate(alpha: float, N: int, T: float = 1.0) -> tuple[float, float]:
    """(δ, per-iteration rate) for α and τ = T/N: δ = α√(T/τ) = α√N, rate = 2√(δ(1 − δ)).
    Raises ValueError unless 0 < δ < ½."""
    tau = T / N
    delta = alpha * math.sqrt(T / tau)
    if not 0.0 < delta < 0.5:
        raise ValueError(f"Theorem 4.5 requires 0 < delta = alpha*sqrt(T/tau) < 1/2; got {delta:.6g}")
    return delta, 2.0 * math.sqrt(delta * (1.0 - delta))


def rate_bound_check(history: Sequence[float], alpha: float, N: int, T: float = 1.0, slack: float = 1e-12) -> dict:
    """history[k−1] = ‖r_k‖/‖r_0‖ from ONE left-preconditioned GMRES cycle.  Returns
    {holds, delta, bound_rate, worst, printed_rate, holds_printed}; worst = max_k history_k / rate^k."""
    delta, rate = theorem_4_5_rate(alpha, N, T)
    worst = 0.0
    printed = 2.0 * math.sqrt(delta) * (1.0 - delta)
    holds_printed = True
    bound_k = printed_k = 1.0
    for h in history:
        bound_k *= rate
        printed_k *= printed
        worst = max(worst, float(h) / bound_k)
        holds_printed = holds_printed and float(h) <= printed_k * (1.0 + slack)
    return {"holds": worst <= 1.0 + slack, "delta": delta, "bound_rate": rate, "worst": worst,
            "printed_rate": printed, "holds_printed": holds_printed}


def alpha_for_delta(delta: float, N: int, T: float = 1.0) -> float:
    """α = δ√(τ/T) (Theorem 4.5's choice) for τ = T/N."""
    return delta * math.sqrt((T / N) / T)
