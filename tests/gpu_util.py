"""Helpers shared by the GPU parity tests (test infrastructure)."""
import numpy as np


def rel(a, b):
    """Relative ℓ2 difference (real or complex)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
