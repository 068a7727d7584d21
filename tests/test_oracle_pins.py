"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against what the paper and
mathematics fix — printed worked examples (tests/golden/), closed forms, invariants, special cases
and brute force on tiny inputs — never against itself.  See DESIGN.md "Oracle pins"."""
import json
import math
import os

import numpy as np
import pytest

import synth
from oracle import aao, gmres, precond, problem, spectrum

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def small1d(n=15, N=8, alpha=0.1, kind="logprice"):
    base = synth.C1 if kind == "logprice" else synth.C3
    return synth.scaled(base, n, N, alpha=alpha)


def small2d(n=7, N=8, alpha=0.1):
    return synth.scaled(synth.C4, n, N, alpha=alpha)


def same_set(a, b, tol):
    """Multiset equality of complex numbers up to tol (greedy nearest matching)."""
    b = list(np.asarray(b))
    for x in np.asarray(a):
        d = np.abs(np.array(b) - x)
        i = int(np.argmin(d))
        if d[i] > tol:
            return False
        b.pop(i)
    return not b


def heat_op(m, h=None):
    h = 1.0 / (m + 1) if h is None else h
    return problem.Operator1D(np.full(m, 1 / h**2), np.full(m, -2 / h**2), np.full(m, 1 / h**2),
                              np.arange(1, m + 1) * h, h)


def scalar_op(Atilde, tau):
    """1x1 spatial 'matrix' with Ã = τ·di = Atilde."""
    return problem.Operator1D(np.zeros(1), np.array([Atilde / tau]), np.zeros(1), np.zeros(1), 1.0)


# ------------------------------------------------------------------------------------- DFT

def test_dft_golden_examples():
    for key in ("dft_delta_M4", "dft_ones_M4"):
        g = GOLD[key]
        F = precond.fourier_matrix(4)
        np.testing.assert_allclose(F @ np.array(g["x"], float), np.array(g["y"], float), atol=1e-15)


def test_dft_unitary_and_matches_numpy_fft():
    rng = np.random.default_rng(3)
    for N in (2, 8, 64, 256):
        F = precond.fourier_matrix(N)
        assert np.abs(F.conj().T @ F - np.eye(N)).max() < 1e-13
        x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        # numpy.fft.fft uses the same kernel e^{-2πi jk/N}; 𝔽 is its unitary scaling.
        assert rel(F @ x, np.fft.fft(x) / math.sqrt(N)) < 1e-13


# ----------------------------------------------------------------------------------- lambdas

def test_lambda_golden_M2():
    g = GOLD["lambda_M2_alpha0.01"]
    l1, l2 = precond.lambdas(g["N"], g["alpha"])
    np.testing.assert_allclose(l1, g["lam1"], atol=1e-15)
    np.testing.assert_allclose(l2, g["lam2"], atol=1e-15)


@pytest.mark.parametrize("N,alpha", [(3, 0.1), (8, 0.01), (64, 0.001), (4096, 0.01)])
def test_lambda_closed_form_and_set(N, alpha):
    l1, l2 = precond.lambdas(N, alpha)
    a = alpha ** (1.0 / N)
    k = np.arange(N)
    # FFT-consistent ordering (reading #3): 1 − a e^{−2πik/N}
    np.testing.assert_allclose(l1, 1 - a * np.exp(-2j * np.pi * k / N), atol=1e-13)
    np.testing.assert_allclose(l2, 0.5 + 0.5 * a * np.exp(-2j * np.pi * k / N), atol=1e-13)
    # Same SET as the printed Eq. eigCx, conjugated order.
    printed = 1 - a * np.exp(2j * np.pi * k / N)
    assert same_set(l1, printed, 1e-13)
    assert (l1.real > 0).all() and (l2.real > 0).all()
    np.testing.assert_allclose(l1[1:], np.conj(l1[1:][::-1]), atol=1e-13)   # conjugate pairs


@pytest.mark.parametrize("N,alpha", [(5, 0.3), (16, 0.01), (64, 1.0)])
def test_alpha_circulant_time_block_is_a_first_order_recurrence(N, alpha):
    """The identity the CUDA path's 2D time pass uses (k_tscan.cu): for a spatial mode μ the time block
    C1^(α) − μC2^(α) (dense) is (1 − μ/2)I − (1 + μ/2)S_α, so its inverse is the recurrence
    z_t = ρ z_{t−1} + c v_t with z_{−1} = α z_{N−1}, whose closure is z_{N−1} = G/(1 − αρ^N) — here written
    as a plain loop and held against the dense solve and against the oracle's transform steps (a)-(c)."""
    rng = np.random.default_rng(N)
    for mu in (-1e-3, -0.37, -5.0, -400.0):
        T = aao.C1(N, alpha) - mu * aao.C2(N, alpha)
        S = np.eye(N, k=-1)
        S[0, N - 1] = alpha
        assert np.abs(T - ((1 - mu / 2) * np.eye(N) - (1 + mu / 2) * S)).max() < 1e-15 * (1 + abs(mu))
        v = rng.standard_normal(N)
        rho, c = (1 + mu / 2) / (1 - mu / 2), 1 / (1 - mu / 2)
        s = np.zeros(N)
        acc = 0.0
        for t in range(N):                      # scan from a zero state
            acc = rho * acc + c * v[t]
            s[t] = acc
        zl = s[N - 1] / (1 - alpha * rho**N)     # cyclic closure
        z = s + rho ** np.arange(1, N + 1) * alpha * zl
        assert rel(z, np.linalg.solve(T, v)) < 1e-12
        # the oracle's diagonalisation of the same block: Γ_α, DFT, ÷ (λ1_k − λ2_k μ), inverse, Γ_α⁻¹
        l1, l2 = precond.lambdas(N, alpha)
        g = precond.gamma(N, alpha)
        F = precond.fourier_matrix(N)
        zt = (F.conj().T @ ((F @ (g * v)) / (l1 - l2 * mu))) / g
        assert np.abs(zt.imag).max() < 1e-12 * np.abs(zt).max()
        assert rel(z, zt.real) < 1e-12


@pytest.mark.parametrize("N,alpha", [(5, 0.3), (8, 0.1)])
def test_lambda_diagonalises_alpha_circulant(N, alpha):
    """C_ℓ = V_α D_ℓ V_α⁻¹ with V_α = Λ_α⁻¹𝔽* (PAPER.md:270-276), checked against the dense
    α-circulants written from PAPER.md:246-259; the printed ordering fails it for N ≥ 3."""
    F = precond.fourier_matrix(N)
    L = np.diag(precond.gamma(N, alpha))
    V = np.linalg.inv(L) @ F.conj().T
    Vi = F @ L
    l1, l2 = precond.lambdas(N, alpha)
    assert np.abs(V @ np.diag(l1) @ Vi - aao.C1(N, alpha)).max() < 1e-13
    assert np.abs(V @ np.diag(l2) @ Vi - aao.C2(N, alpha)).max() < 1e-13
    a = alpha ** (1.0 / N)
    printed = 1 - a * np.exp(2j * np.pi * np.arange(N) / N)
    assert np.abs(V @ np.diag(printed) @ Vi - aao.C1(N, alpha)).max() > 1e-2   # negative control
    # eigenvalues of the dense C1 (LAPACK, no DFT involved) are the λ1 set
    assert same_set(np.linalg.eigvals(aao.C1(N, alpha)), l1, 1e-12)


def test_gamma():
    g = precond.gamma(8, 0.01)
    assert g[0] == 1.0
    np.testing.assert_allclose(g, 0.01 ** (np.arange(8) / 8), rtol=1e-15)


# ---------------------------------------------------------------------------------- operator

@pytest.mark.parametrize("kind", ["logprice", "price", "bs2d"])
def test_operator_second_order_consistency(kind):
    """‖L_h u − 𝓛u‖_∞ on the manufactured solution drops ~4x per h halving (central differences);
    𝓛u is taken from the analytic f: 𝓛u = u_t − f = −u − f."""
    errs = []
    for n in (31, 63, 127):
        w = synth.scaled({"logprice": synth.C1, "price": synth.C3, "bs2d": synth.C4}[kind], n, 8)
        op = problem.build_operator(w)
        t = 0.3
        u = problem.u_exact(w, op, t)
        Lu = -u - problem.f_source(w, op, t)
        errs.append(np.abs(problem.apply_L(op, u) - Lu).max())
    if kind == "price":            # u quadratic in S: central differences are exact (reading #24)
        assert max(errs) < 1e-9
    else:
        assert 3.5 < errs[0] / errs[1] < 4.5 and 3.5 < errs[1] / errs[2] < 4.5


def test_operator_dense_matches_stencil():
    rng = np.random.default_rng(0)
    for w in (small1d(9), small1d(9, kind="price"), small2d(5)):
        op = problem.build_operator(w)
        u = rng.standard_normal(op.m)
        shp = (op.m,) if w.dim == 1 else (op.n, op.n)
        np.testing.assert_allclose(op.dense() @ u, problem.apply_L(op, u.reshape(shp)).reshape(-1), rtol=1e-13,
                                   atol=1e-10)


def test_operator_row_values_logprice():
    """Hand stencil: central differences of (σ²/2)u_xx + (r−σ²/2)u_x − ru (BASELINE.json configs[0])."""
    w = synth.C1
    op = problem.build_operator(w)
    h = 6.0 / 256
    s2, mu = 0.09, 0.05 - 0.045
    assert abs(op.h - h) < 1e-15
    assert abs(op.lo[3] - (s2 / (2 * h * h) - mu / (2 * h))) < 1e-9
    assert abs(op.di[3] - (-s2 / (h * h) - 0.05)) < 1e-9
    assert abs(op.up[3] - (s2 / (2 * h * h) + mu / (2 * h))) < 1e-9


def test_assumption_3_1_negative_semidefinite():
    """All BASELINE operators are NSD (reading #11): symmetric part has eigenvalues ≤ 0 and
    eig(L_h) is real negative."""
    for w in (small1d(31), small1d(31, kind="price"), small2d(7)):
        A = problem.build_operator(w).dense()
        assert np.linalg.eigvalsh(0.5 * (A + A.T)).max() <= 1e-9
        ev = np.linalg.eigvals(A)
        assert np.abs(ev.imag).max() < 1e-8 * np.abs(ev).max() and ev.real.max() < 0


# ---------------------------------------------------------------------------------- AaO / CN

def test_M_golden_M3_N1():
    tau = 0.25
    w = synth.scaled(synth.C1, 1, 3, T=3 * tau)
    op = scalar_op(-tau, tau)            # Ã = [−τ]
    M = aao.dense_M(w, op)
    expect = np.array([[1 + tau / 2, 0, 0], [-(1 - tau / 2), 1 + tau / 2, 0], [0, -(1 - tau / 2), 1 + tau / 2]])
    np.testing.assert_allclose(M, expect, atol=1e-15)
    u = np.array([[1.0], [2.0], [5.0]])
    np.testing.assert_allclose(aao.apply_M(w, op, u).ravel(), expect @ u.ravel(), atol=1e-15)


def test_M_A0_is_time_difference():
    w = small1d(9, 6)
    op = problem.Operator1D(np.zeros(9), np.zeros(9), np.zeros(9), np.zeros(9), 1.0)
    u = np.random.default_rng(1).standard_normal((6, 9))
    y = aao.apply_M(w, op, u)
    np.testing.assert_allclose(y[0], u[0])
    np.testing.assert_allclose(y[1:], u[1:] - u[:-1])


@pytest.mark.parametrize("mk", [lambda: small1d(11, 6), lambda: small1d(11, 6, kind="price"), lambda: small2d(5, 6)])
def test_block_matvecs_equal_kronecker(mk):
    w = mk()
    op = problem.build_operator(w)
    u = np.random.default_rng(2).standard_normal(synth.shape_of(w))
    np.testing.assert_allclose(aao.apply_M(w, op, u).ravel(), aao.dense_M(w, op) @ u.ravel(), rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(aao.apply_P(w, op, u).ravel(), aao.dense_P(w, op) @ u.ravel(), rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("mk", [lambda: small1d(31, 16), lambda: small1d(31, 16, kind="price"), lambda: small2d(7, 8)])
def test_sequential_cn_solves_aao(mk):
    """AaO solution = sequential CN: 𝓜 u_seq = b to round-off, and equals the
    dense solve of 𝓜u = b."""
    w = mk()
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    u = aao.solve_sequential(w, op, b)
    assert rel(aao.apply_M(w, op, u), b) < 1e-13
    ud = np.linalg.solve(aao.dense_M(w, op), b.ravel())
    assert rel(u.ravel(), ud) < 1e-11


def test_second_order_space_time():
    """Manufactured-solution error ‖u − u_exact‖_∞ over all steps falls ~16x per 4x refinement of
    (m, N) and ~4x per 2x (second order in τ and h)."""
    errs = []
    for n in (63, 127, 255):
        w = synth.scaled(synth.C1, n, n + 1)
        op = problem.build_operator(w)
        u = aao.solve_sequential(w, op, problem.assemble_rhs(w, op))
        errs.append(np.abs(u - problem.exact_blocks(w, op)).max())
    assert 3.6 < errs[0] / errs[1] < 4.4 and 3.6 < errs[1] / errs[2] < 4.4


def test_second_order_time_price_space():
    errs = []
    for N in (16, 32, 64):
        w = synth.scaled(synth.C3, 63, N)
        op = problem.build_operator(w)
        u = aao.solve_sequential(w, op, problem.assemble_rhs(w, op))
        errs.append(np.abs(u - problem.exact_blocks(w, op)).max())
    assert 3.6 < errs[0] / errs[1] < 4.4 and 3.6 < errs[1] / errs[2] < 4.4


def test_second_order_2d():
    errs = []
    for n in (15, 31):
        w = synth.scaled(synth.C4, n, n + 1)
        op = problem.build_operator(w)
        u = aao.solve_sequential(w, op, problem.assemble_rhs(w, op))
        errs.append(np.abs(u - problem.exact_blocks(w, op)).max())
    assert 3.5 < errs[0] / errs[1] < 4.5


def test_cn_stability_theorem_2_1():
    """‖Q1⁻¹Q2‖₂ ≤ 1 for symmetric NSD A; for the nonsymmetric BS operator after
    the diagonal symmetrising similarity."""
    w = small1d(15, 8)
    tau = w.T / w.N
    A = heat_op(15).dense()
    I = np.eye(15)
    R = np.linalg.solve(I - 0.5 * tau * A, I + 0.5 * tau * A)
    assert np.linalg.norm(R, 2) <= 1 + 1e-12


def test_theorem_2_2_bounds_and_golden_cond():
    g = GOLD["cond_M_A0_M2"]
    w = synth.scaled(synth.C1, 1, 2, T=2.0)
    op = scalar_op(0.0, 1.0)
    s = spectrum.singular_values_M(w, op)
    assert abs(s[0] / s[-1] - g["cond"]) < 1e-12 and s[0] / s[-1] <= g["bound"]
    for w in (small1d(7, 8), small1d(7, 8, kind="price"), small2d(3, 6)):
        op = problem.build_operator(w)
        s = spectrum.singular_values_M(w, op)
        tau = w.T / w.N
        nA = np.linalg.norm(op.dense(), 2)
        assert s.min() >= 1.0 / w.N - 1e-12
        assert s.max() <= 2 + tau * nA + 1e-9
        assert s.max() / s.min() <= 2 * w.N + w.T * nA + 1e-9


# ------------------------------------------------------------------------------------- P_α⁻¹

CASES = [lambda a: small1d(15, 8, a), lambda a: small1d(13, 16, a, kind="price"), lambda a: small2d(5, 8, a)]


@pytest.mark.parametrize("alpha", [0.5, 0.1, 1e-3])
@pytest.mark.parametrize("mk", CASES)
def test_pinv_equals_dense_solve(mk, alpha):
    w = mk(alpha)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 2, 7)
    for vi in v:
        z = precond.pinv_dft(w, op, vi)
        assert rel(z, precond.pinv_dense(w, op, vi)) < 1e-10
        assert rel(aao.apply_P(w, op, z), vi) < 1e-12


@pytest.mark.parametrize("mk", CASES)
def test_pinv_halving_equals_full_and_real(mk):
    w = mk(0.01)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 11)[0]
    zh, imag_h = precond.pinv_dft(w, op, v, return_imag=True)
    zf, imag_f = precond.pinv_dft(w, op, v, halving=False, return_imag=True)
    zm, imag_m = precond.pinv_dft(w, op, v, dft="matrix", return_imag=True)
    assert rel(zh, zf) < 1e-14 and rel(zm, zf) < 1e-13       # matrix DFT: O(N) round-off growth
    assert imag_h < 1e-15 and imag_f < 1e-12 and imag_m < 1e-15


def test_pinv_extended_precision_agrees():
    w = small1d(15, 16, 1e-3)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 3)[0]
    ze = precond.pinv_dft(w, op, v, extended=True)
    assert rel(precond.pinv_dft(w, op, v), ze) < 1e-13
    assert rel(aao.apply_P(w, op, ze), v) < 1e-14


@pytest.mark.parametrize("mk", CASES)
def test_pinv_equals_fft_free_sweep(mk):
    w = mk(0.01)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 5)[0]
    zs, sweeps = precond.pinv_sweep(w, op, v)
    assert sweeps <= 12
    assert rel(precond.pinv_dft(w, op, v), zs) < 1e-13


def test_pinv_A0_golden():
    """Ã = 0 ⇒ P_α = C1 ⊗ I and P_α⁻¹(e₁-block) = (1/(1−α))·𝟙."""
    for alpha in (0.5, 0.1, 0.01):
        w = synth.scaled(synth.C1, 3, 8, alpha=alpha)
        op = problem.Operator1D(np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3), 1.0)
        v = np.zeros((8, 3)); v[0] = 1.0
        z = precond.pinv_dft(w, op, v)
        np.testing.assert_allclose(z * (1 - alpha), GOLD["pinv_A0_e1"]["value_times_one_minus_alpha"], atol=1e-13)


def test_pinv_printed_ordering_negative_control():
    """Using the printed Eq. eigCx ordering with the printed 𝔽 must break P(P⁻¹v) = v (reading #3)."""
    w = small1d(7, 8, 0.1)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 1)[0]
    orig = precond.lambdas
    try:
        def printed(N, alpha, kchunk=512):
            a = alpha ** (1.0 / N)
            e = np.exp(2j * np.pi * np.arange(N) / N)
            return 1 - a * e, 0.5 + 0.5 * a * e
        precond.lambdas = printed
        zbad = precond.pinv_dft(w, op, v, halving=False, dft="matrix")
    finally:
        precond.lambdas = orig
    assert rel(aao.apply_P(w, op, zbad), v) > 1e-2


def test_2d_fast_diagonalisation_vs_dense_shifted_solve():
    w = small2d(6, 4, 0.01)
    op = problem.build_operator(w)
    tau = w.T / w.N
    l1, l2 = precond.lambdas(w.N, w.alpha)
    rng = np.random.default_rng(4)
    R = rng.standard_normal((3, 6, 6)) + 1j * rng.standard_normal((3, 6, 6))
    Z = precond.shifted_solve(w, op, l1[:3], l2[:3], R)
    A = tau * op.dense()
    for k in range(3):
        zd = np.linalg.solve(l1[k] * np.eye(36) - l2[k] * A, R[k].ravel())
        assert rel(Z[k].ravel(), zd) < 1e-12


def test_toeplitz_eig_closed_form():
    # the last two triples have negative off-diagonals (s·u > 0 still): the symmetrised off-diagonal
    # is sgn(s)·√(su), so mode j's eigenvalue must not be that of mode n+1−j
    for (s, d, u) in ((1.0, -2.0, 1.0), (35.77, -72.8, 37.05), (0.3, -1.0, 0.6), (-1.0, -4.0, -1.0),
                      (-0.3, 1.0, -0.6)):
        n = 9
        D, e = precond.toeplitz_eig(n, s, d, u)
        S = precond.dst1_matrix(n)
        L = np.diag(np.full(n, d)) + np.diag(np.full(n - 1, s), -1) + np.diag(np.full(n - 1, u), 1)
        assert np.abs(S @ S - np.eye(n)).max() < 1e-13
        assert np.abs((D[:, None] * S) @ np.diag(e) @ (S / D[None, :]) - L).max() < 1e-12
        np.testing.assert_allclose(np.sort(np.linalg.eigvals(L).real), np.sort(e), atol=1e-12)


def test_2d_shifted_solve_negative_offdiagonals_vs_dense():
    """2D fast diagonalisation with L_x = tridiag(−1, −4, −1), L_y = tridiag(−0.5, −3, −0.7)
    (negative-definite, negative off-diagonals): each shifted system against a dense solve, and P_α⁻¹
    against numpy.linalg.solve on the dense P_α."""
    w = small2d(5, 8, 0.1)
    op = problem.Operator2D(xs=-1.0, xd=-4.0, xu=-1.0, ys=-0.5, yd=-3.0, yu=-0.7, shift=-0.2, n=5,
                            x=np.arange(1, 6) / 6.0, h=1.0 / 6.0)
    tau = w.T / w.N
    l1, l2 = precond.lambdas(w.N, w.alpha)
    rng = np.random.default_rng(7)
    R = rng.standard_normal((3, 5, 5)) + 1j * rng.standard_normal((3, 5, 5))
    Z = precond.shifted_solve(w, op, l1[:3], l2[:3], R)
    A = tau * op.dense()
    for k in range(3):
        assert rel(Z[k].ravel(), np.linalg.solve(l1[k] * np.eye(25) - l2[k] * A, R[k].ravel())) < 1e-12
    v = rng.standard_normal((w.N, 5, 5))
    assert rel(precond.pinv_dft(w, op, v), precond.pinv_dense(w, op, v)) < 1e-12


@pytest.mark.parametrize("kind", ["logprice", "price", "bs2d"])
def test_operator_rows_exact_on_quadratics(kind):
    """Central differences are exact on polynomials of degree ≤ 2, so at interior rows (both
    neighbours inside the domain) L_h applied to 1, x, x² (and y, y², xy in 2D) must equal the
    continuous 𝓛 (BASELINE.json configs: σ²/2·∂xx + drift·∂x − r) evaluated by hand:
      𝓛1 = −r,  𝓛x = b(x) − r x,  𝓛x² = σ²(x)·… — three equations per row pin lo, di, up (a dropped
    term, a wrong sign or swapped lo/up fails one of them), independently of build_operator's formulas."""
    w = {"logprice": synth.scaled(synth.C1, 31, 8), "price": synth.scaled(synth.C3, 31, 8),
         "bs2d": synth.scaled(synth.C4, 15, 8)}[kind]
    op = problem.build_operator(w)
    r = w.r
    if kind in ("logprice", "price"):
        x = op.x
        inner = slice(1, op.m - 1)
        if kind == "logprice":        # 𝓛 = (σ²/2)∂xx + (r − σ²/2)∂x − r
            a2 = 0.5 * w.sigma ** 2 * np.ones_like(x)
            a1 = (r - 0.5 * w.sigma ** 2) * np.ones_like(x)
        else:                         # 𝓛 = (σ²S²/2)∂SS + rS∂S − r
            a2 = 0.5 * w.sigma ** 2 * x * x
            a1 = r * x
        for u, Lu in ((np.ones_like(x), -r * np.ones_like(x)),
                      (x.copy(), a1 - r * x),
                      (x * x, 2 * a2 + 2 * a1 * x - r * x * x)):
            got = problem.apply_L(op, u)
            assert np.abs(got[inner] - Lu[inner]).max() <= 1e-9 * max(1.0, np.abs(Lu[inner]).max())
        return
    X, Y = np.meshgrid(op.x, op.x)     # [y][x]
    s1, s2 = w.sigma2
    b1, b2 = r - 0.5 * s1 * s1, r - 0.5 * s2 * s2
    inner = (slice(1, op.n - 1), slice(1, op.n - 1))
    one = np.ones_like(X)
    cases = ((one, -r * one), (X, b1 - r * X), (Y, b2 - r * Y), (X * X, s1 * s1 + 2 * b1 * X - r * X * X),
             (Y * Y, s2 * s2 + 2 * b2 * Y - r * Y * Y), (X * Y, b1 * Y + b2 * X - r * X * Y))
    for u, Lu in cases:
        got = problem.apply_L(op, u)
        assert np.abs(got[inner] - Lu[inner]).max() <= 1e-9 * max(1.0, np.abs(Lu[inner]).max())


def test_pinv_dft_matrix_route_at_N4096():
    """The dense-DFT-matrix route of Eq. 3.2 (exact (k·t mod N) table, λ from D_ℓ = diag(√N𝔽Λ_αc_ℓ)
    by a dense product) against the library-FFT route at N = 4096 (c2's time length) on one column
    block (m = 15), and both against the FFT-free fixed-point sweep of the block form."""
    w = synth.scaled(synth.C1, 15, 4096, alpha=0.01)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 3)[0]
    zf = precond.pinv_dft(w, op, v)
    zm = precond.pinv_dft(w, op, v, dft="matrix")
    zs, _ = precond.pinv_sweep(w, op, v)
    assert rel(zm, zf) < 1e-12 and rel(zs, zf) < 1e-12 and rel(zs, zm) < 1e-12
    assert rel(aao.apply_P(w, op, zm), v) < 1e-12


def test_gmres_iterates_equal_maxit_reruns():
    """gmres_right(iterates=[…]) records x_j after every inner step; each equals the result of a
    separate run stopped at maxit = j (the definition of the j-th iterate)."""
    w = synth.scaled(synth.C1, 31, 32, alpha=0.3)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    A = lambda x: aao.apply_M(w, op, x)
    P = lambda x: precond.pinv_dft(w, op, x)
    its = []
    u, rep = gmres.gmres_right(A, P, b, 1e-10, 3, iterates=its)   # restart 3: crosses cycles
    assert len(its) == rep.iterations >= 4 and rep.restarts >= 1
    for j in (1, 2, 3):
        uj, _ = gmres.gmres_right(A, P, b, 1e-10, 3, maxit=j)
        assert rel(its[j - 1], uj) < 1e-14
    assert rel(its[-1], u) < 1e-14


@pytest.mark.parametrize("n", [15, 31])
def test_q1_solver_dst_equals_sparse_lu(n):
    """The dense-DST Q1 solve (used for n ≥ 256) against scipy's sparse LU of Q1 = I − ½τL_h."""
    w = small2d(n, 8)
    op = problem.build_operator(w)
    tau = w.T / w.N
    r = np.random.default_rng(n).standard_normal((n, n))
    x1 = aao.Q1Solver(op, tau, dst_min=1)(r)
    x2 = aao.Q1Solver(op, tau, dst_min=10 ** 9)(r)
    assert aao.Q1Solver(op, tau, dst_min=1).dst is not None and aao.Q1Solver(op, tau, dst_min=10 ** 9).dst is None
    assert rel(x1, x2) < 1e-13
    assert rel(aao.Q1(op, tau, x1), r) < 1e-13


@pytest.mark.parametrize("mk", [lambda: synth.C1])
def test_pinv_roundtrip_c1_all_vectors(mk):
    """North-star oracle check: P_α(P_α⁻¹v) = v to 1e-12 on the 16 c1 vectors (BASELINE configs[0])."""
    w = mk()
    op = problem.build_operator(w)
    V = synth.random_vectors(w)
    assert V.shape == (16, 256, 255)
    for v in V:
        assert rel(aao.apply_P(w, op, precond.pinv_dft(w, op, v)), v) < 1e-12


# ---------------------------------------------------------------------------------- spectrum

def test_spectrum_golden_heat():
    g = GOLD["heat_M8_N15_alpha0.1"]
    w = synth.scaled(synth.C1, g["space"], g["time_steps"], alpha=g["alpha"])
    op = heat_op(g["space"])
    ev = spectrum.preconditioned_eigs(w, op)
    unit = np.abs(ev - 1) <= 1e-8
    assert unit.sum() >= g["n_unit"]
    nonunit = np.sort(np.real(ev))[np.argsort(np.abs(np.sort(np.real(ev)) - 1))][::-1]
    assert spectrum.in_omega(ev, w.alpha).all()
    cf = spectrum.closed_form_nonunit(w, op)
    # match the m eigenvalues farthest from 1 with the closed form (sorted)
    far = ev[np.argsort(-np.abs(ev - 1))][: g["space"]]
    np.testing.assert_allclose(np.sort(far.real), np.sort(cf.real), atol=1e-8)
    assert np.abs(ev.imag).max() < 1e-10
    assert (ev.real >= 1 / 1.1 - 1e-10).all() and (ev.real <= 1 / 0.9 + 1e-10).all()


@pytest.mark.parametrize("mk", [lambda: small1d(7, 8, 0.1), lambda: small1d(7, 8, 0.1, kind="price"),
                                lambda: small2d(3, 8, 0.1)])
def test_spectrum_theorem_3_1_bs(mk):
    w = mk()
    op = problem.build_operator(w)
    ev = spectrum.preconditioned_eigs(w, op)
    assert (np.abs(ev - 1) <= 1e-8).sum() >= (w.N - 1) * op.m
    assert spectrum.in_omega(ev, w.alpha).all()
    cf = spectrum.closed_form_nonunit(w, op)
    far = ev[np.argsort(-np.abs(ev - 1))][: op.m]
    np.testing.assert_allclose(np.sort(far.real), np.sort(cf.real), atol=1e-7)
    # Reading #12: real, and in [1, 1/(1−α)) for even N.  In 2D the spatial spectrum has
    # near-coincident pairs μ_ij ≈ μ_i'j'; LAPACK splits such a near-double eigenvalue of the
    # nonnormal P⁻¹𝓜 into a complex pair of size ~√(eps·cond), so the 2D bound is looser.
    assert np.abs(ev.imag).max() < (1e-8 if w.dim == 1 else 1e-3)
    assert ev.real.min() >= 1 - 1e-10 and ev.real.max() < 1 / (1 - w.alpha)


def test_spectrum_scalar_special_cases():
    for alpha in GOLD["scalar_A0_nonunit"]["alphas"]:
        w = synth.scaled(synth.C1, 1, 6, alpha=alpha)
        ev = spectrum.preconditioned_eigs(w, scalar_op(0.0, w.T / w.N))
        assert np.isclose(ev, 1 / (1 - alpha), atol=1e-12).sum() == 1
        assert np.isclose(ev, 1.0, atol=1e-12).sum() == 5
    w = synth.scaled(synth.C1, 1, 6, alpha=0.3)
    ev = spectrum.preconditioned_eigs(w, scalar_op(-2.0, w.T / w.N))
    np.testing.assert_allclose(ev, 1.0, atol=1e-12)


def test_lemma_3_2_step_eigs():
    for w in (small1d(9, 8), small1d(9, 8, kind="price"), small2d(3, 4)):
        ev = spectrum.step_eigs(w, problem.build_operator(w))
        assert (ev.real > -1).all() and (ev.real <= 1 + 1e-12).all() and (np.abs(ev) <= 1 + 1e-12).all()


def test_MinvR_norm():
    """‖𝓜⁻¹𝓡‖₂ ≤ √N for symmetric NSD A, = √N at Ã = 0."""
    for op, w in ((scalar_op(0.0, 1.0 / 6), synth.scaled(synth.C1, 1, 6)), (heat_op(5), synth.scaled(synth.C1, 5, 6))):
        M = aao.dense_M(w, op)
        P = aao.dense_P(w, op, 1.0)
        R = M - P                                        # P_1 = 𝓜 − 𝓡 (α = 1)
        nrm = np.linalg.norm(np.linalg.solve(M, R), 2)
        assert nrm <= math.sqrt(w.N) + 1e-10
    w = synth.scaled(synth.C1, 1, 6)
    M = aao.dense_M(w, scalar_op(0.0, 1 / 6))
    R = M - aao.dense_P(w, scalar_op(0.0, 1 / 6), 1.0)
    assert abs(np.linalg.norm(np.linalg.solve(M, R), 2) - math.sqrt(6)) < 1e-12


# ------------------------------------------------------------------------------------- GMRES

def test_gmres_identity_one_iteration():
    b = np.random.default_rng(0).standard_normal((4, 5))
    u, rep = gmres.gmres_right(lambda x: x, lambda x: x, b, 1e-12, 10)
    assert rep.iterations == 1 and rep.converged and rel(u, b) < 1e-14


def test_gmres_exact_preconditioner_one_iteration():
    w = small1d(15, 16)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    u, rep = gmres.gmres_right(lambda x: aao.apply_M(w, op, x), lambda x: aao.solve_sequential(w, op, x),
                               b, 1e-12, 10)
    assert rep.iterations == 1 and rep.converged


def test_gmres_minimal_residual_property_brute_force():
    """The j-th right-preconditioned GMRES iterate minimises ‖b − 𝓜P⁻¹y‖ over y ∈ K_j(𝓜P⁻¹, b)
    — checked against numpy lstsq on an explicitly built (QR-orthonormalised) Krylov basis."""
    w = small1d(9, 8, 0.3)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    A = lambda x: aao.apply_M(w, op, x)
    P = lambda x: precond.pinv_dft(w, op, x)
    AP = lambda x: A(P(x.reshape(b.shape))).reshape(-1)
    for j in (1, 2, 3):
        u, rep = gmres.gmres_right(A, P, b, 1e-15, 20, maxit=j)
        K = [b.reshape(-1)]
        for _ in range(j - 1):
            K.append(AP(K[-1]))
        Q, _ = np.linalg.qr(np.array(K).T)
        B = np.array([AP(Q[:, i]) for i in range(j)]).T
        y, *_ = np.linalg.lstsq(B, b.reshape(-1), rcond=None)
        u_ls = P((Q @ y).reshape(b.shape))
        assert rel(u, u_ls) < 1e-8
        assert abs(np.linalg.norm(b - A(u)) / np.linalg.norm(b) - rep.relres_true) < 1e-12


def test_gmres_c1_converges_to_sequential_cn():
    """North star: final u within 1e-8 of sequential CN; mesh-small iteration count (scratch: 3)."""
    w = synth.C1
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    u, rep = gmres.gmres_right(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x),
                               b, w.tol, w.restart)
    useq = aao.solve_sequential(w, op, b)
    assert rep.converged and rep.relres_true <= w.tol
    assert 2 <= rep.iterations <= 5
    assert rel(u, useq) < 1e-8
    assert all(h2 <= h1 for h1, h2 in zip(rep.history, rep.history[1:]))     # monotone within a cycle


# ------------------------------------------------------------------------------ NEXT #1: 𝓛(t) = d(t)𝓛
# PAPER.md:1020-1036 (Eq. 5.8): 𝓜 = B1⊗I − (D̃B2)⊗Ã, ξ₀ = (I + ½d(t_½)Ã)u⁰; the preconditioner uses d̄C2.

def _tv(n=15, N=8, rate=0.5, alpha=0.1):
    return synth.C1T.with_(name="tv", n=n, N=N, dt_rate=rate, alpha=alpha)


def test_tv_block_matvec_equals_dense_kronecker():
    w = _tv()
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 5)[0]
    Md = aao.dense_M(w, op)
    assert rel(aao.apply_M(w, op, v).reshape(-1), Md @ v.reshape(-1)) < 1e-14
    # the d-weighting sits on the rows (D̃B2, not B2D̃): row t uses d(t_{t+½}) for both u_t and u_{t−1}
    d = aao.d_half(w)
    tau = aao.tau_of(w)
    At = tau * op.dense()
    B2D = np.kron(np.diag(d) @ aao.B2(w.N), At)
    assert rel(np.kron(aao.B1(w.N), np.eye(op.m)) - B2D, Md) == 0.0
    assert rel(np.kron(aao.B2(w.N) @ np.diag(d), At), B2D) > 1e-3   # the other placement differs


def test_tv_dbar_closed_form():
    """d̄ = (1/N) Σ_k e^{−ρτ(k+½)} = e^{−ρτ/2}(1 − e^{−ρT}) / (N(1 − e^{−ρτ})) (geometric sum)."""
    w = _tv(N=64)
    rho, tau = w.dt_rate, w.T / w.N
    closed = math.exp(-rho * tau / 2) * (1 - math.exp(-rho * w.T)) / (w.N * (1 - math.exp(-rho * tau)))
    assert abs(aao.tau_prec(w) / tau - closed) < 1e-15
    assert aao.tau_prec(w.with_(dt_rate=0.0)) == tau


def test_tv_sequential_cn_solves_aao():
    w = _tv(n=31, N=32)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    u = aao.solve_sequential(w, op, b)
    assert rel(aao.apply_M(w, op, u), b) < 1e-13


def test_tv_second_order_convergence():
    """The time-dependent CN solution converges at second order to u = e^{−t}sin(…) (pins f = ∂_tu −
    d(t)𝓛u, the midpoint sampling of D̃ and the ξ block)."""
    errs = []
    for n in (63, 127, 255):
        w = synth.C1T.with_(name="tvc", n=n, N=n + 1)
        op = problem.build_operator(w)
        u = aao.solve_sequential(w, op, problem.assemble_rhs(w, op))
        errs.append(float(np.abs(u - problem.exact_blocks(w, op)).max()))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.5 < r1 < 4.5 and 3.5 < r2 < 4.5, errs


def test_tv_pinv_roundtrip_and_dense():
    w = _tv(n=15, N=16)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 7)[0]
    z = precond.pinv_dft(w, op, v)
    assert rel(aao.apply_P(w, op, z), v) < 1e-12
    zd = np.linalg.solve(aao.dense_P(w, op), v.reshape(-1)).reshape(v.shape)
    assert rel(z, zd) < 1e-12
    zs, _ = precond.pinv_sweep(w, op, v)
    assert rel(z, zs) < 1e-12


def test_tv_gmres_converges_to_sequential_cn():
    w = _tv(n=63, N=64, alpha=0.01).with_(restart=40, tol=1e-10)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    u, rep = gmres.gmres_right(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x), b,
                               w.tol, w.restart)
    assert rep.converged and rel(u, aao.solve_sequential(w, op, b)) < 1e-8
    assert 3 <= rep.iterations <= 12, rep.iterations   # d̄ approximation: a few more than constant 𝓛


# ------------------------------------------------------------------------------ NEXT #2: P₁ (α = 1)
# PAPER.md:324-328 (Remark 3.2): P₁ = C1^(1)⊗I − C2^(1)⊗Ã is the block circulant preconditioner; it is
# singular exactly when Ã is, because λ1,1 = 0 (here k = 0) leaves −λ2,1Ã = −Ã.

def test_P1_inverse_equals_dense_solve_and_roundtrip():
    w = synth.scaled(synth.C1, 15, 16, alpha=1.0)
    op = problem.build_operator(w)
    v = synth.random_vectors(w, 1, 3)[0]
    z = precond.pinv_dft(w, op, v)
    assert rel(aao.apply_P(w, op, z), v) < 1e-12
    zd = np.linalg.solve(aao.dense_P(w, op), v.reshape(-1)).reshape(v.shape)
    assert rel(z, zd) < 1e-12
    # the λ pair at k = N/2 degenerates to (2, 0): that shifted system is 2 z = w (no spatial coupling)
    l1, l2 = precond.lambdas(w.N, 1.0)
    assert abs(l1[w.N // 2] - 2.0) < 1e-14 and abs(l2[w.N // 2]) < 1e-14 and abs(l1[0]) < 1e-14


def test_P1_singular_iff_A_singular():
    """Remark 3.2: with a singular Ã (zero row sums: reflecting ends), P₁ is singular while P_α (α < 1)
    is not; with the Dirichlet operators of the workloads P₁ is invertible."""
    m, N = 7, 4
    lo = np.ones(m); up = np.ones(m); di = -2.0 * np.ones(m)
    di[0] = di[-1] = -1.0                                   # reflecting ends: L·1 = 0
    op = problem.Operator1D(lo=lo, di=di, up=up, x=np.arange(1, m + 1) * 0.1, h=0.1)
    w = synth.scaled(synth.C1, m, N, alpha=1.0)
    s1 = np.linalg.svd(aao.dense_P(w, op), compute_uv=False)
    sa = np.linalg.svd(aao.dense_P(w.with_(alpha=0.5), op), compute_uv=False)
    assert s1[-1] < 1e-12 * s1[0]
    assert sa[-1] > 1e-3 * sa[0]
    wd = synth.scaled(synth.C1, 15, 8, alpha=1.0)
    sd = np.linalg.svd(aao.dense_P(wd, problem.build_operator(wd)), compute_uv=False)
    assert sd[-1] > 1e-6 * sd[0]


def test_P1_needs_more_gmres_iterations():
    """The paper's comparison (Tables 1-4: P₁ 21-131 iterations vs P_α 4-6): on the c1 family the
    oracle's right-preconditioned GMRES needs more iterations with P₁ than with P_0.01."""
    w = synth.scaled(synth.C1, 63, 64, restart=50)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    its = {}
    for a in (1.0, 0.01):
        wa = w.with_(alpha=a)
        u, rep = gmres.gmres_right(lambda x: aao.apply_M(wa, op, x), lambda x: precond.pinv_dft(wa, op, x), b,
                                   1e-10, 50)
        assert rep.converged and rel(u, aao.solve_sequential(wa, op, b)) < 1e-8
        its[a] = rep.iterations
    assert its[1.0] > its[0.01] + 2, its


# ------------------------------------------------------------------ NEXT #4: left GMRES + Theorem 4.5
# PAPER.md:576-590 (§4, Eq. sss2x) left-preconditioned GMRES, residual r_k = P⁻¹(b − 𝓜u^(k));
# PAPER.md:663-718 (Eqs. 4.9, 4.11, 4.12) field-of-values bound; Theorem 4.5.

def heat_workload(n, N, delta=0.25):
    """Symmetric negative definite 1D operator (the hypothesis of Theorem 4.5), with
    α = δ√(τ/T) = δ/√N: synth.heat (c1 operator with r = σ²/2)."""
    return synth.heat(n, N, delta)


def test_heat_workload_is_symmetric_nsd():
    w = heat_workload(15, 16)
    L = problem.build_operator(w).dense()
    assert np.array_equal(L, L.T)
    assert np.linalg.eigvalsh(L).max() < 0


def test_gmres_left_identity_and_exact_preconditioner_one_iteration():
    b = np.random.default_rng(0).standard_normal((4, 5))
    u, rep = gmres.gmres_left(lambda x: x, lambda x: x, b, 1e-12, 10)
    assert rep.iterations == 1 and rep.converged and rel(u, b) < 1e-14
    w = small1d(15, 16)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    u, rep = gmres.gmres_left(lambda x: aao.apply_M(w, op, x), lambda x: aao.solve_sequential(w, op, x),
                              b, 1e-12, 10)
    assert rep.iterations == 1 and rep.converged
    assert rel(u, aao.solve_sequential(w, op, b)) < 1e-12


def test_gmres_left_minimal_residual_property_brute_force():
    """Eq. sss2x: ‖r_k‖ = min_{x ∈ K_k(B, r0)} ‖r0 − Bx‖, B = P⁻¹𝓜, r0 = P⁻¹b — the Givens history
    and the k-th iterate against numpy lstsq on an explicit Krylov basis (built from (B − I)^i r0,
    which spans the same space and stays well conditioned when B ≈ I)."""
    w = small1d(9, 8, 0.3)
    op = problem.build_operator(w)
    b = problem.assemble_rhs(w, op)
    A = lambda x: aao.apply_M(w, op, x)
    P = lambda x: precond.pinv_dft(w, op, x)
    Bf = lambda x: P(A(x.reshape(b.shape))).reshape(-1)
    r0 = P(b).reshape(-1)
    for k in (1, 2, 3):
        u, rep = gmres.gmres_left(A, P, b, 1e-15, 20, maxit=k)
        K = [r0]
        for _ in range(k - 1):
            K.append(Bf(K[-1]) - K[-1])
        Q, _ = np.linalg.qr(np.array(K).T)
        BQ = np.array([Bf(Q[:, i]) for i in range(k)]).T
        y, *_ = np.linalg.lstsq(BQ, r0, rcond=None)
        rmin = np.linalg.norm(r0 - BQ @ y) / np.linalg.norm(r0)
        assert abs(rep.history[k - 1] - rmin) <= 1e-9 * max(rmin, 1e-6)
        assert rel(u, (Q @ y).reshape(b.shape)) < 1e-8
        assert abs(rep.relres_prec - rmin) <= 1e-9 * max(rmin, 1e-6)


def test_gmres_left_and_right_agree_with_dense_solve():
    for w in (small1d(15, 16, 0.05), small1d(15, 16, 0.05, kind="price"), small2d(7, 8, 0.05)):
        op = problem.build_operator(w)
        b = problem.assemble_rhs(w, op)
        A = lambda x: aao.apply_M(w, op, x)
        P = lambda x: precond.pinv_dft(w, op, x)
        ud = np.linalg.solve(aao.dense_M(w, op), b.reshape(-1)).reshape(b.shape)
        ul, repl = gmres.gmres_left(A, P, b, 1e-11, 30)
        ur, repr_ = gmres.gmres_right(A, P, b, 1e-11, 30)
        assert repl.converged and repr_.converged
        assert rel(ul, ud) < 1e-8 and rel(ur, ud) < 1e-8
        assert abs(repl.iterations - repr_.iterations) <= 1
        # relres_true is the unpreconditioned residual of the returned iterate
        assert abs(repl.relres_true - np.linalg.norm(b - A(ul)) / np.linalg.norm(b)) < 1e-14


def test_rate_bound_values():
    """Theorem 4.5's rate [1 − (1 − 2δ)²]^{1/2} = 2√(δ(1 − δ)) (reading R27: the printed 2√δ(1 − δ)
    is the algebra slip; SPEC.md:372's "δ = ¼ → 0.75" is that printed value): δ = ¼ → √3/2,
    δ → 0 → 0, δ ≥ ½ violates the hypothesis."""
    N, T = 64, 1.0
    tau = T / N
    d, rate = gmres.rate_bound(0.25 * math.sqrt(tau / T), tau, T)
    assert abs(d - 0.25) < 1e-15 and abs(rate - math.sqrt(3) / 2) < 1e-15
    assert abs(gmres.printed_rate(0.25) - 0.75) < 1e-15
    for delta in (1e-8, 0.01, 0.1, 0.3, 0.49):
        d, rate = gmres.rate_bound(delta / math.sqrt(N), tau, T)
        exact = 2 * math.sqrt(delta * (1 - delta))
        assert abs(rate - exact) <= 1e-15 / delta * exact     # 1 − (1 − 2δ)² cancels at small δ
        assert gmres.printed_rate(delta) < rate                 # the printed value is stricter
    assert gmres.rate_bound(1e-8 / 8, tau, T)[1] < 3e-4
    for bad in (0.5, 0.7, 1.0 * math.sqrt(N)):
        with pytest.raises(ValueError):
            gmres.rate_bound(bad / math.sqrt(N), tau, T)
    r = math.sqrt(3) / 2
    chk = gmres.rate_bound_check([0.8, 0.7, 0.6], 0.25 / 8, tau, T)
    assert chk["holds"] and abs(chk["worst"] - 0.7 / r ** 2) < 1e-14 and not chk["holds_printed"]
    assert not gmres.rate_bound_check([0.8, 0.76], 0.25 / 8, tau, T)["holds"]   # 0.76 > 0.75


def test_theorem_4_5_bound_chain_dense():
    """SPEC.md:374 example: symmetric 1D heat, N = m = 32, α = ¼√(τ/T), full GMRES → the bound holds.
    Checked link by link against dense matrices: ‖𝓜⁻¹𝓡‖ ≤ √N, Eq. 4.11
    (‖P⁻¹𝓜 − I‖ ≤ α‖𝓜⁻¹𝓡‖/(1 − α‖𝓜⁻¹𝓡‖) and λ_min(H(P⁻¹𝓜)) > 0), the field-of-values bound Eq. 4.9
    / 4.12 per step, and Theorem 4.5's [2√δ(1−δ)]^k on the GMRES history."""
    w = heat_workload(31, 32)
    op = problem.build_operator(w)
    M = aao.dense_M(w, op)
    P = aao.dense_P(w, op)
    R = (M - P) / w.alpha                                  # P_α = 𝓜 − α𝓡
    mr = np.linalg.norm(np.linalg.solve(M, R), 2)
    assert mr <= math.sqrt(w.N) * (1 + 1e-12)
    B = np.linalg.solve(P, M)
    E = np.linalg.norm(B - np.eye(B.shape[0]), 2)
    assert E <= w.alpha * mr / (1 - w.alpha * mr) * (1 + 1e-9)
    Hs = 0.5 * (B + B.T)
    nu = np.linalg.eigvalsh(Hs).min()
    assert nu >= 1 - E - 1e-12 and nu > 0
    fov_rate = math.sqrt(1 - (nu / np.linalg.norm(B, 2)) ** 2)           # Eq. 4.9
    eq412 = math.sqrt(1 - (1 - 2 * w.alpha * mr) ** 2)                     # Eq. 4.12
    assert fov_rate <= eq412 * (1 + 1e-9)
    b = problem.assemble_rhs(w, op)
    u, rep = gmres.gmres_left(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x), b,
                              1e-13, 60)
    assert rep.converged and rep.restarts == 0
    for k, h in enumerate(rep.history, start=1):
        assert h <= fov_rate ** k * (1 + 1e-9)
    chk = gmres.rate_bound_check(rep.history, w.alpha, 1.0 / w.N, 1.0)
    assert chk["holds"] and abs(chk["delta"] - 0.25) < 1e-14 and abs(chk["bound_rate"] - math.sqrt(3) / 2) < 1e-14


def test_theorem_4_5_mesh_independent_counts():
    """'mesh-independent linear convergence rate': with α = δ√(τ/T) the left GMRES
    iteration count to 1e-10 does not grow under simultaneous refinement of space and time."""
    its = []
    for n, N in ((15, 16), (63, 64), (255, 256)):
        w = heat_workload(n, N)
        op = problem.build_operator(w)
        b = synth.random_vectors(w, 1, 5)[0]     # every spatial mode excited (the manufactured rhs is
        #                                          close to one eigenmode and converges in 2 steps)
        u, rep = gmres.gmres_left(lambda x: aao.apply_M(w, op, x), lambda x: precond.pinv_dft(w, op, x), b,
                                  1e-10, 40)
        assert rep.converged and rep.restarts == 0
        assert gmres.rate_bound_check(rep.history, w.alpha, 1.0 / N, 1.0)["holds"]
        its.append(rep.iterations)
    assert its == sorted(its, reverse=True) and max(its) <= 8, its     # refinement never adds iterations
