// Device bodies of the small GMRES steps (k_gmres.cu's single-thread kernels and the post-fold hook
// of the reducing kernels).  scal[0] = ||r_0||, scal[1] = estimate, scal[2] = ||w||² (reduced),
// scal[3] = non-finite flag, scal[4] = ||r||/||r_0||, scal[5] = happy breakdown.
#pragma once
#include "common.cuh"
#include "internal.h"

CNP_DEV void cycle_start_dev(double* scl, double* g, double* scal, int first, int rmax, double* G = nullptr) {
  const double beta = sqrt(scal[2]);
  if (G) G[0] = scal[2];  // Gram CGS2: G̃_00 = ‖Ṽ_0‖²
  if (!first) scal[12] = scl[0];  // the ending cycle's s_0 (cnpint_krylov_basis test hook)
  if (first) scal[0] = beta;
  scal[4] = beta / scal[0];
  scl[0] = beta > 0.0 ? 1.0 / beta : 0.0;
  for (int i = 0; i <= rmax; ++i) g[i] = 0.0;
  g[0] = beta;
  if (!isfinite(beta)) scal[3] = 1.0;
}

CNP_DEV void arnoldi_finalize_dev(int j, int ldh, const double* c1, const double* c2, double* scl, double* H,
                                  double* cs, double* sn, double* g, double* scal) {
  double* h = H + (size_t)j * ldh;
  for (int i = 0; i <= j; ++i) h[i] = scl[i] * (c1[i] + c2[i]);
  const double beta = sqrt(scal[2]);
  h[j + 1] = beta;
  scl[j + 1] = beta > 0.0 ? 1.0 / beta : 0.0;
  for (int i = 0; i < j; ++i) {  // previous rotations
    const double t = cs[i] * h[i] + sn[i] * h[i + 1];
    h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
    h[i] = t;
  }
  const double den = hypot(h[j], h[j + 1]);
  const double c = den > 0.0 ? h[j] / den : 1.0;
  const double s = den > 0.0 ? h[j + 1] / den : 0.0;
  cs[j] = c;
  sn[j] = s;
  h[j] = den;
  h[j + 1] = 0.0;
  g[j + 1] = -s * g[j];
  g[j] = c * g[j];
  const double est = fabs(g[j + 1]) / scal[0];
  scal[1] = est;
  if (!isfinite(est) || !isfinite(den)) scal[3] = 1.0;
  if (beta == 0.0) scal[5] = 1.0;  // happy breakdown
}

// Gram CGS2 (north_star (5): classical Gram-Schmidt with reorthogonalisation).  G̃ = ṼᵀṼ of the
// cycle's (unnormalised) basis, symmetric, stored at ldh; its row j+1 is reduced by the update that
// writes Ṽ_{j+1} (op 4) and G̃_00 by the cycle start, so at step j every entry i, k ≤ j is known.
//   c2 = Ṽᵀ(w − Ṽ S² c1) = c1 − G̃ S² c1,  S = diag(s_i)  (formed by the update kernel's blocks and
//   again by its folding block for the H column, op 4)
// — the coefficients classic CGS2's second pass reads back; the algebra is exact and the rounding
// differs by O(ε‖c1‖), the size of the classic pass's own rounding.
CNP_DEV void gram_c2_dev(int j, int ldh, const double* G, const double* scl, const double* c1, double* c2) {
  for (int i = 0; i <= j; ++i) {
    double acc = c1[i];
    for (int k = 0; k <= j; ++k) acc -= G[(size_t)i * ldh + k] * (scl[k] * scl[k] * c1[k]);
    c2[i] = acc;
  }
}
//   op 4 (after the update folded cg = [‖Ṽ_{j+1}‖², Ṽ_iᵀṼ_{j+1} (i ≤ j)]): c2 as above, store row/column
//   j+1 of G̃, scal[2] = ‖Ṽ_{j+1}‖², then the Arnoldi finalize of column j (op 1).
CNP_DEV void gram_store_dev(int j, int ldh, const double* cg, double* G, double* scal) {
  const int r = j + 1;
  for (int i = 0; i <= j; ++i) {
    G[(size_t)r * ldh + i] = cg[1 + i];
    G[(size_t)i * ldh + r] = cg[1 + i];
  }
  G[(size_t)r * ldh + r] = cg[0];
  scal[2] = cg[0];
}

//   op 5 (derived-norm probe of a step expected to be the last; run by the fused-dots matvec that also
//   folded ww = wᵀw into c1[j+1]): with a = S²(c1 + c2) the new vector would be w − Ṽa, whose norm follows
//   from the Gram matrix without a pass over the vectors, β² = ww − 2aᵀc1 + aᵀG̃a.  The difference cancels
//   to β²/ww, so it is trusted only when β² ≥ 1e-8·ww (relative error of β² ≤ ~1e-7); then column j is
//   finalized with it (g[j] saved in scal[13] so the host can take the step back) and scal[6] = 1.
CNP_DEV void gram_probe_dev(const PostOp& p) {
  const int j = p.j, ldh = p.ldh;
  gram_c2_dev(j, ldh, p.G, p.scl, p.c1, p.c2w);
  const double ww = p.c1[j + 1];
  double lin = 0.0, quad = 0.0;
  for (int i = 0; i <= j; ++i) {
    const double ai = p.scl[i] * p.scl[i] * (p.c1[i] + p.c2w[i]);
    lin += ai * p.c1[i];
    double row = 0.0;
    for (int k = 0; k <= j; ++k) row += p.G[(size_t)i * ldh + k] * (p.scl[k] * p.scl[k] * (p.c1[k] + p.c2w[k]));
    quad += ai * row;
  }
  const double b2 = ww - 2.0 * lin + quad;
  const bool safe = isfinite(b2) && isfinite(ww) && ww > 0.0 && b2 >= 1e-8 * ww;
  p.scal[14] = b2;
  p.scal[15] = ww;
  p.scal[6] = safe ? 1.0 : 0.0;
  if (safe) {
    p.scal[13] = p.g[j];
    p.scal[2] = b2;
    arnoldi_finalize_dev(j, ldh, p.c1, p.c2, p.scl, p.H, p.cs, p.sn, p.g, p.scal);
  }
}

// Called by the whole last block after grid_fold returned true (its thread 0 wrote scal[2]).
CNP_DEV void run_post(const PostOp& p) {
  if (p.op == 0) return;
  __syncthreads();  // the fold's outputs (written by threads < ncols) are visible to thread 0
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    if (p.op == 1) arnoldi_finalize_dev(p.j, p.ldh, p.c1, p.c2, p.scl, p.H, p.cs, p.sn, p.g, p.scal);
    else if (p.op == 3) gram_c2_dev(p.j, p.ldh, p.G, p.scl, p.c1, p.c2w);
    else if (p.op == 4) {
      gram_c2_dev(p.j, p.ldh, p.G, p.scl, p.c1, p.c2w);  // the c2 the update used, for the H column
      if (p.j + 1 < p.ldh) gram_store_dev(p.j, p.ldh, p.cg, p.G, p.scal);
      else p.scal[2] = p.cg[0];
      arnoldi_finalize_dev(p.j, p.ldh, p.c1, p.c2, p.scl, p.H, p.cs, p.sn, p.g, p.scal);
    } else if (p.op == 5) gram_probe_dev(p);
    else cycle_start_dev(p.scl, p.g, p.scal, p.first, p.rmax, p.G);
    if (p.hmap && p.op != 3) {
      for (int i = 0; i < 8; ++i) p.hmap[i] = p.scal[i];
      p.hmap[8] = (double)*p.status;
    }
  }
}
