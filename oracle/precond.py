"""The block α-circulant preconditioner inverse P_α⁻¹ (ORACLE).

Test infrastructure only (see oracle/__init__.py).

P_α⁻¹v is by definition the solution z of P_α z = v (Eq. 3.1; block form
PAPER.md:344-350).  The paper reaches it through the diagonalisation

    C_ℓ = V_α D_ℓ V_α⁻¹,  V_α = Λ_α⁻¹ 𝔽*,  D_ℓ = diag(√N 𝔽 Λ_α C_ℓ(:,1))
    step (a) z1 = (V⁻¹ ⊗ I) v
    step (b) (λ1_k I − λ2_k Ã) z2_k = z1_k                                  (Eq. 3.2)
    step (c) z  = (V ⊗ I) z2

with only the first ⌈(N+1)/2⌉ = N/2+1 systems solved and the rest obtained by conjugation
(Remark 3.1).  This module provides

  pinv_dft     the three steps literally: scale by Λ_α, 𝔽 (library FFT, or the dense DFT matrix
               built from an exact (k·t mod N) table), λ from D_ℓ = diag(√N 𝔽 Λ_α c_ℓ) evaluated
               literally, complex Thomas (1D) or dense-DST fast diagonalisation (2D,
               PAPER.md:315-316) for k ≤ N/2, conjugate fill, 𝔽*, unscale;
  pinv_full    the same without the halving (all N systems solved) — pin for Remark 3.1;
  pinv_sweep   an FFT-free solve of the block form P_α z = v by fixed-point sweeps (no DFT);
  pinv_dense   numpy.linalg.solve on the dense P_α (tiny sizes).

Reading #3: PAPER.md:282-286 prints λ1_k = 1 − α^{1/N} e^{+2(k−1)πi/N},
which is inconsistent with the printed 𝔽 (ω = e^{−2πi/N}); D_ℓ evaluated literally gives
λ1_k = 1 − a e^{−2πik/N}, λ2_k = ½(1 + a e^{−2πik/N}), a = α^{1/N}, k = 0..N−1.  We compute D_ℓ
literally, so the oracle is consistent with 𝔽 by construction.
"""
from __future__ import annotations

import math

import numpy as np

from .aao import Q1Solver, Q2, tau_prec
from .problem import Operator1D


# ------------------------------------------------------------------------------ DFT, scaling

def dft_table(N: int) -> np.ndarray:
    """ω^j = e^{−2πi j/N}, j = 0..N−1.  Indexed by (j·k mod N) so that no
    large argument is ever passed to sin/cos (SURVEY.md §8(c) reading #21)."""
    j = np.arange(N)
    return np.cos(2 * np.pi * j / N) - 1j * np.sin(2 * np.pi * j / N)


def fourier_matrix(N: int, rows=None) -> np.ndarray:
    """𝔽 = [ω^{jk}/√N]_{j,k=0}^{N−1}, optionally only the given rows."""
    rows = np.arange(N) if rows is None else np.asarray(rows)
    tbl = dft_table(N)
    idx = (rows[:, None] * np.arange(N)[None, :]) % N
    return tbl[idx] / math.sqrt(N)


def gamma(N: int, alpha: float, dtype=np.float64) -> np.ndarray:
    """Diagonal of Λ_α = diag(1, α^{1/N}, …, α^{(N−1)/N}); reading #5."""
    return np.exp(np.arange(N, dtype=dtype) * (np.log(dtype(alpha)) / dtype(N)))


def lambdas(N: int, alpha: float, kchunk: int = 512):
    """(λ1_k, λ2_k), k = 0..N−1, evaluated literally as D_ℓ = diag(√N 𝔽 Λ_α C_ℓ^(α)(:,1))
    (PAPER.md:273-276).  First columns: C1(:,1) = (1, −1, 0, …), C2(:,1) = ½(1, 1, 0, …)
    (PAPER.md:246-259).  The product with 𝔽 is taken in row chunks to bound memory."""
    L = gamma(N, alpha)
    c1 = np.zeros(N); c1[0], c1[1 % N] = 1.0, -1.0
    c2 = np.zeros(N); c2[0], c2[1 % N] = 0.5, 0.5
    if N == 1:
        c1[0], c2[0] = 1.0 - alpha, 0.5 + 0.5 * alpha
    lam1 = np.empty(N, dtype=complex)
    lam2 = np.empty(N, dtype=complex)
    for k0 in range(0, N, kchunk):
        rows = np.arange(k0, min(N, k0 + kchunk))
        F = fourier_matrix(N, rows)
        lam1[rows] = math.sqrt(N) * (F @ (L * c1))
        lam2[rows] = math.sqrt(N) * (F @ (L * c2))
    return lam1, lam2


# ---------------------------------------------------------------------------- shifted solves

def thomas(a: np.ndarray, b: np.ndarray, c: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Plain Thomas algorithm for a batch of tridiagonal systems, vectorised over the leading
    axis: a_i x_{i−1} + b_i x_i + c_i x_{i+1} = d_i (a_0, c_{m−1} unused).  No pivoting: every
    shifted system here is diagonally dominant (SURVEY.md §8(c) reading #22)."""
    m = d.shape[-1]
    cp = np.empty_like(d)
    dp = np.empty_like(d)
    cp[..., 0] = c[..., 0] / b[..., 0]
    dp[..., 0] = d[..., 0] / b[..., 0]
    for i in range(1, m):
        den = b[..., i] - a[..., i] * cp[..., i - 1]
        cp[..., i] = c[..., i] / den
        dp[..., i] = (d[..., i] - a[..., i] * dp[..., i - 1]) / den
    x = np.empty_like(d)
    x[..., m - 1] = dp[..., m - 1]
    for i in range(m - 2, -1, -1):
        x[..., i] = dp[..., i] - cp[..., i] * x[..., i + 1]
    return x


def dst1_matrix(n: int) -> np.ndarray:
    """Orthonormal DST-I: S_{ij} = √(2/(n+1)) sin(ijπ/(n+1)), i, j = 1..n; S = Sᵀ = S⁻¹."""
    i = np.arange(1, n + 1)
    return math.sqrt(2.0 / (n + 1)) * np.sin(np.outer(i, i) * np.pi / (n + 1))


def toeplitz_eig(n: int, s: float, d: float, u: float):
    """Eigen-decomposition of tridiag(s, d, u) (s·u > 0): L = (D S) diag(e) (S D⁻¹) with
    D = diag(ρ^i), ρ = √(s/u), e_j = d + 2σ cos(jπ/(n+1)), σ = sgn(s)·√(s u): the similarity
    D⁻¹ L D has off-diagonals s/ρ = uρ = σ, i.e. it is the symmetric Toeplitz tridiag(σ, d, σ),
    diagonalised by DST-I.  For s, u < 0 the sign matters: without it mode j
    would carry the eigenvalue of mode n+1−j."""
    assert s * u > 0
    rho = math.sqrt(s / u)
    sigma = math.copysign(math.sqrt(s * u), s)
    Dg = rho ** np.arange(1, n + 1)
    e = d + 2.0 * sigma * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))
    return Dg, e


def shifted_solve(w, op, lam1: np.ndarray, lam2: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Step (b): (λ1_k I − λ2_k Ã) z_k = rhs_k for each k, Ã = τL_h.
    1D: complex Thomas vectorised across k.  2D: fast diagonalisation with dense DST-I matrices
    (PAPER.md:315-316)."""
    rdt = np.longdouble if lam1.dtype == np.clongdouble else np.float64
    tau = rdt(w.T) / rdt(w.N) if not w.dt_rate else rdt(tau_prec(w))   # d̄τ for 𝓛(t) = d(t)𝓛
    K = lam1.size
    if isinstance(op, Operator1D):
        l1, l2 = lam1[:, None], lam2[:, None]
        a = -l2 * tau * op.lo[None, :].astype(rdt)
        b = l1 - l2 * tau * op.di[None, :].astype(rdt)
        c = -l2 * tau * op.up[None, :].astype(rdt)
        return thomas(np.broadcast_to(a, rhs.shape), np.broadcast_to(b, rhs.shape),
                      np.broadcast_to(c, rhs.shape), rhs)
    n = op.n
    S = dst1_matrix(n)
    Dx, ex = toeplitz_eig(n, op.xs, op.xd, op.xu)
    Dy, ey = toeplitz_eig(n, op.ys, op.yd, op.yu)
    mu = ey[:, None] + ex[None, :] + op.shift          # eigenvalues of L_h, [y][x]
    out = np.empty_like(rhs)
    for k in range(K):
        R = rhs[k]                                     # [y][x]
        Rh = S @ ((R / Dy[:, None]) / Dx[None, :]) @ S       # W⁻¹ R = S D_y⁻¹ R D_x⁻¹ S
        Zh = Rh / (lam1[k] - lam2[k] * tau * mu)
        out[k] = Dy[:, None] * (S @ Zh @ S) * Dx[None, :]    # W Z = D_y S Z S D_x
    return out


# ------------------------------------------------------------------------------- P_α⁻¹ routes

def _flat(v):
    return v.reshape(v.shape[0], -1)


def lambdas_fft(N: int, alpha: float, dtype=np.float64):
    """Same D_ℓ = diag(√N 𝔽 Λ_α c_ℓ) with the product √N𝔽x taken by the library FFT
    (numpy.fft.fft computes Σ_j e^{−2πijk/N} x_j = √N(𝔽x)_k; pinned against the DFT matrix)."""
    L = gamma(N, alpha, dtype)
    c1 = np.zeros(N, dtype=dtype); c1[0], c1[1] = 1, -1
    c2 = np.zeros(N, dtype=dtype); c2[0], c2[1] = dtype(0.5), dtype(0.5)
    return np.fft.fft(L * c1), np.fft.fft(L * c2)


def pinv_dft(w, op, v: np.ndarray, alpha: float | None = None, *, halving: bool = True,
             return_imag: bool = False, dft: str = "fft",
             extended: bool = False, kchunk: int = 512):
    """P_α⁻¹v by Eq. 3.2 with unitary 𝔽 (SPEC.md:84 normalisation; any consistent
    choice gives the same z, reading #4) and, if ``halving``, Remark 3.1 (k = 0..N/2 only,
    conjugate fill z_{N−k} = conj(z_k)).

    dft="fft"    step (a) 𝔽Λ_αv = fft(Λ_αv)/√N and step (c) Λ_α⁻¹𝔽*z = Λ_α⁻¹·ifft(z)·√N with the
                 library FFT (a permitted primitive; O(log N) round-off growth);
    dft="matrix" the dense DFT matrix from the exact (k·t mod N) table (O(N²m), small N only).
    extended     evaluate everything in x87 extended precision (numpy longdouble, 64-bit
                 mantissa) — used where the fp64 oracle's own round-off, amplified by
                 κ(Λ_α) ≈ 1/α, would approach the 1e-12 parity bar (1D only).
    The imaginary residue ‖Im z‖/‖Re z‖ of step (c) is returned on request."""
    alpha = w.alpha if alpha is None else alpha
    N = w.N
    shp = v.shape
    rdt = np.longdouble if extended else np.float64
    g = gamma(N, alpha, rdt)
    K = N // 2 + 1 if halving else N
    x = g[:, None] * _flat(v).astype(rdt)                      # Λ_α v
    if dft == "fft":
        lam1, lam2 = lambdas_fft(N, alpha, rdt)
        z1 = np.fft.fft(x, axis=0)[:K] / np.sqrt(rdt(N))       # step (a)
    else:
        assert not extended
        lam1, lam2 = lambdas(N, alpha)
        z1 = np.empty((K, x.shape[1]), dtype=complex)
        for k0 in range(0, K, kchunk):
            rows = np.arange(k0, min(K, k0 + kchunk))
            z1[rows] = fourier_matrix(N, rows) @ x
    z2 = shifted_solve(w, op, lam1[:K], lam2[:K], z1.reshape((K,) + shp[1:]))   # step (b)
    z2 = z2.reshape(K, -1)
    if halving:                                                # Remark 3.1: conjugate fill
        full = np.empty((N, z2.shape[1]), dtype=z2.dtype)
        full[:K] = z2
        full[K:] = np.conj(z2[1:N - K + 1][::-1])              # z_{N−k} = conj(z_k)
    else:
        full = z2
    if dft == "fft":                                           # step (c): Λ_α⁻¹ 𝔽* z2
        z = np.fft.ifft(full, axis=0) * np.sqrt(rdt(N))
    else:
        z = np.empty((N, full.shape[1]), dtype=complex)
        for t0 in range(0, N, kchunk):
            rows = np.arange(t0, min(N, t0 + kchunk))
            z[rows] = np.conj(fourier_matrix(N, rows)) @ full  # 𝔽 symmetric ⇒ (𝔽*)_{t,k} = conj(𝔽_{t,k})
    z /= g[:, None]
    imag = float(np.linalg.norm(z.imag) / max(np.linalg.norm(z.real), 1e-300))
    zr = z.real.astype(np.float64).reshape(shp)
    return (zr, imag) if return_imag else zr


def pinv_full(w, op, v, alpha=None):
    """Eq. 3.2 solving all N shifted systems (no Remark 3.1 halving)."""
    return pinv_dft(w, op, v, alpha, halving=False)


def pinv_sweep(w, op, v: np.ndarray, alpha: float | None = None, max_sweeps: int = 60):
    """FFT-free solve of the block form P_α z = v:
        Q1 z_0 = v_0 + α Q2 z_{N−1},   Q1 z_t = v_t + Q2 z_{t−1}  (t ≥ 1).
    Fixed-point iteration on ζ ≈ z_{N−1}: one sweep runs the recursion with z_{−1} := αζ; the
    error in ζ is multiplied by α J_N per sweep, J_N = (Q1⁻¹Q2)^N with spectral radius ≤ 1
    (Lemma 3.2), so it contracts at least by α.  Stops when the update of ζ
    is below 1e-15‖ζ‖ or stops shrinking (rounding level).  Returns (z, sweeps)."""
    alpha = w.alpha if alpha is None else alpha
    tau = tau_prec(w)
    solve = Q1Solver(op, tau)
    zeta = np.zeros_like(v[0])
    z = np.empty_like(v)
    last = np.inf
    for s in range(1, max_sweeps + 1):
        prev = alpha * zeta
        for t in range(w.N):
            z[t] = solve(v[t] + Q2(op, tau, prev))
            prev = z[t]
        dz = float(np.linalg.norm(z[-1] - zeta))
        zeta = z[-1].copy()
        if dz <= 1e-15 * max(float(np.linalg.norm(zeta)), 1e-300) or (s > 2 and dz > 0.5 * last):
            return z, s
        last = dz
    return z, max_sweeps


def pinv_dense(w, op, v, alpha=None):
    """numpy.linalg.solve(P_α, v) on the dense Kronecker matrix; tiny sizes."""
    from .aao import dense_P
    P = dense_P(w, op, alpha)
    return np.linalg.solve(P, v.reshape(-1)).reshape(v.shape)
