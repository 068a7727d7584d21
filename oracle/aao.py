"""AaO matvec 𝓜u, preconditioner matvec P_α z, sequential CN, dense 𝓜 and P_α (ORACLE).

Test infrastructure only (see oracle/__init__.py).

Plain definitions written out:
  PAPER.md:331-351 (§3.2)  Q1 = I − ½Ã, Q2 = I + ½Ã;
                           𝓜 = block-bidiagonal(diag Q1, sub-diag −Q2);
                           P_α = 𝓜 with the extra top-right block −αQ2.
  PAPER.md:198-203 (Eq. 2.2) 𝓜 = B1 ⊗ I − B2 ⊗ Ã, B1 = tridiag(−1,1,0), B2 = ½ tridiag(1,1,0).
  PAPER.md:244-266 (Eq. 3.1) P_α = C1^(α) ⊗ I − C2^(α) ⊗ Ã.
  PAPER.md:125-128 (Eq. 2.1) CN step (I − τ/2 A) u^{k+1} = (I + τ/2 A) u^k + τ f^{k+½}.
  PAPER.md:1020-1036 (Eq. 5.8) time-dependent 𝓛(t) = d(t)𝓛: 𝓜 = B1 ⊗ I − (D̃B2) ⊗ Ã with
                           D̃ = diag(d(t_{k+½})), i.e. row t of the block form uses Q1, Q2 with
                           Ã → d(t_{t+½})Ã; the preconditioner replaces C2^(α) by d̄·C2^(α),
                           d̄ = mean_k d(t_{k+½}), i.e. Ã → d̄Ã.
Vectors are arrays of shape (N, m) (1D) or (N, n, n) (2D, [t][y][x]).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .problem import Operator1D, apply_L


def tau_of(w) -> float:
    return w.T / w.N


def d_half(w) -> np.ndarray:
    """D̃ = diag(d(t_{½}), …, d(t_{N−½})); all ones for constant 𝓛."""
    tau = tau_of(w)
    return np.exp(-w.dt_rate * (np.arange(w.N) + 0.5) * tau)


def tau_prec(w) -> float:
    """τ of the preconditioner's Ã: d̄τ with d̄ = (1/N) Σ_k d(t_{k+½}); τ if 𝓛 is
    constant."""
    return tau_of(w) * float(np.mean(d_half(w))) if w.dt_rate else tau_of(w)


def Q1(op, tau, z):
    """Q1 z = z − ½ τ L_h z."""
    return z - 0.5 * tau * apply_L(op, z)


def Q2(op, tau, z):
    """Q2 z = z + ½ τ L_h z."""
    return z + 0.5 * tau * apply_L(op, z)


def apply_M(w, op, u: np.ndarray) -> np.ndarray:
    """𝓜u by the block form of PAPER.md:337-343: y_0 = Q1u_0, y_t = Q1u_t − Q2u_{t−1}; with
    𝓛(t) = d(t)𝓛 row t uses Ã → d(t_{t+½})Ã (the t-th row of D̃B2)."""
    tau = tau_of(w)
    if not w.dt_rate:
        y = Q1(op, tau, u)
        y[1:] -= Q2(op, tau, u[:-1])
        return y
    d = d_half(w)
    y = np.empty_like(u)
    for t in range(w.N):
        y[t] = Q1(op, tau * d[t], u[t])
        if t:
            y[t] -= Q2(op, tau * d[t], u[t - 1])
    return y


def apply_P(w, op, z: np.ndarray, alpha: float | None = None) -> np.ndarray:
    """P_α z by the block form of PAPER.md:344-350: rows Q1z_t − Q2z_{t−1} and the corner
    (P z)_0 −= α Q2 z_{N−1}; Ã is d̄τL_h for a time-dependent 𝓛."""
    alpha = w.alpha if alpha is None else alpha
    tau = tau_prec(w)
    y = Q1(op, tau, z)
    y[1:] -= Q2(op, tau, z[:-1])
    y[0] -= alpha * Q2(op, tau, z[-1])
    return y


def spatial_sparse(op) -> sp.csr_matrix:
    if isinstance(op, Operator1D):
        m = op.m
        return sp.diags([op.lo[1:], op.di, op.up[:-1]], [-1, 0, 1], shape=(m, m), format="csr")
    n = op.n
    I = sp.identity(n, format="csr")
    Lx = sp.diags([np.full(n - 1, op.xs), np.full(n, op.xd), np.full(n - 1, op.xu)], [-1, 0, 1])
    Ly = sp.diags([np.full(n - 1, op.ys), np.full(n, op.yd), np.full(n - 1, op.yu)], [-1, 0, 1])
    return (sp.kron(I, Lx) + sp.kron(Ly, I) + op.shift * sp.identity(n * n)).tocsr()


class Q1Solver:
    """Solves Q1 x = r = (I − ½τL_h) x = r.  1D: banded LU (solve_banded); 2D: sparse LU, or for
    n ≥ dst_min the fast diagonalisation with dense DST-I matrices:
    L_h = W diag(μ) W⁻¹, W = (D_yS) ⊗ (D_xS), so x = W[(1 − ½τμ)⁻¹ ∘ (W⁻¹r)] — four dense n×n
    products per solve instead of sparse triangular solves with nested fill (pinned against the
    sparse LU in tests/test_oracle_pins.py)."""

    def __init__(self, op, tau, dst_min: int = 256):
        self.op, self.tau = op, tau
        self.dst = None
        if not isinstance(op, Operator1D) and op.n >= dst_min:
            from .precond import dst1_matrix, toeplitz_eig
            S = dst1_matrix(op.n)
            Dx, ex = toeplitz_eig(op.n, op.xs, op.xd, op.xu)
            Dy, ey = toeplitz_eig(op.n, op.ys, op.yd, op.yu)
            mu = ey[:, None] + ex[None, :] + op.shift        # eigenvalues of L_h, [y][x]
            self.dst = (S, Dx, Dy, 1.0 / (1.0 - 0.5 * tau * mu))
            return
        if isinstance(op, Operator1D):
            m = op.m
            ab = np.zeros((3, m))
            ab[0, 1:] = -0.5 * tau * op.up[:-1]
            ab[1, :] = 1.0 - 0.5 * tau * op.di
            ab[2, :-1] = -0.5 * tau * op.lo[1:]
            self.ab = ab
            self.lu = None
        else:
            Q = sp.identity(op.m) - 0.5 * tau * spatial_sparse(op)
            self.lu = spla.splu(Q.tocsc())

    def __call__(self, r: np.ndarray) -> np.ndarray:
        if self.dst is not None:
            S, Dx, Dy, inv = self.dst
            n = self.op.n
            R = r.reshape(n, n)
            Rh = S @ ((R / Dy[:, None]) / Dx[None, :]) @ S        # W⁻¹ r
            return (Dy[:, None] * (S @ (inv * Rh) @ S) * Dx[None, :]).reshape(r.shape)   # W (…)
        if self.lu is None:
            return sla.solve_banded((1, 1), self.ab, r)
        shp = r.shape
        return self.lu.solve(r.reshape(-1)).reshape(shp)


def solve_sequential(w, op, b: np.ndarray) -> np.ndarray:
    """The exact AaO solution by CN time stepping:
    Q1 u_t = b_t + Q2 u_{t−1}, u_{−1} := 0 (u⁰ enters through ξ in b_0); for 𝓛(t) = d(t)𝓛 step t
    uses d(t_{t+½})τ (Eq. 5.8)."""
    tau = tau_of(w)
    d = d_half(w)
    solve = Q1Solver(op, tau) if not w.dt_rate else None
    u = np.empty_like(b)
    prev = np.zeros_like(b[0])
    for t in range(w.N):
        tt = tau * d[t]
        s = solve if solve is not None else Q1Solver(op, tt)
        u[t] = s(b[t] + Q2(op, tt, prev))
        prev = u[t]
    return u


# ------------------------------------------------------------------------------- dense (tiny)

def B1(N):
    """B1 = tridiag(−1, 1, 0) ∈ R^{N×N}."""
    return np.eye(N) - np.eye(N, k=-1)


def B2(N):
    """B2 = ½ tridiag(1, 1, 0)."""
    return 0.5 * (np.eye(N) + np.eye(N, k=-1))


def C1(N, alpha):
    """α-circulant C1^(α): B1 with top-right entry −α."""
    C = B1(N)
    C[0, N - 1] += -alpha
    return C


def C2(N, alpha):
    """α-circulant C2^(α): B2 with top-right entry +α/2."""
    C = B2(N)
    C[0, N - 1] += 0.5 * alpha
    return C


def dense_M(w, op) -> np.ndarray:
    """𝓜 = B1 ⊗ I − (D̃B2) ⊗ Ã, Ã = τ L_h (D̃ = I for constant 𝓛, Eq. 5.8)."""
    At = tau_of(w) * op.dense()
    return np.kron(B1(w.N), np.eye(op.m)) - np.kron(np.diag(d_half(w)) @ B2(w.N), At)


def dense_P(w, op, alpha=None) -> np.ndarray:
    """P_α = C1^(α) ⊗ I − (d̄C2^(α)) ⊗ Ã (Eq. 3.1; d̄ = 1 for constant 𝓛)."""
    alpha = w.alpha if alpha is None else alpha
    At = tau_prec(w) * op.dense()
    return np.kron(C1(w.N, alpha), np.eye(op.m)) - np.kron(C2(w.N, alpha), At)
