// K3: step (b) of Eq. 3.2 for a tridiagonal L_h — the N/2+1 complex
// shifted systems (λ1_k I − λ2_k Ã) ẑ_k = ŵ_k, k = 0..N/2 (Remark 3.1 halving), one CTA per k.
//
// Each system is divided by λ2_k (Re λ2_k > 0) so that the off-diagonals stay
// real: rows  a_i x_{i−1} + b_i x_i + c_i x_{i+1} = d_i  with  a_i = −τ lo_i, c_i = −τ up_i (real),
// b_i = s_k − τ di_i, s_k = λ1_k/λ2_k, d_i = ŵ_i/λ2_k.  Diagonal dominance holds for every k
// (Re s_k > 0 and −di ≥ lo + up), so no pivoting is needed; a zero or non-finite pivot
// still sets the device status word (SPEC.md:298 SingularPreconditioner).
//
// Algorithm (partition method = per-thread Thomas + PCR-style reduced system):
//  level 1  thread p owns rows [i0, i1) (≈ m/P rows, in registers).  A modified Thomas sweep
//           (forward elimination relative to x_{i0}, backward relative to x_{i1−1}) leaves two
//           "interface" rows per chunk coupling (x_{i0−1}, x_{i0}, x_{i1−1}) and (x_{i0}, x_{i1−1},
//           x_{i1}); interior unknowns are x_i = δ'_i − α'_i x_{i0} − γ'_i x_{i1−1}.
//           Toeplitz operators: α, γ, 1/pivot depend only on the position inside the chunk, so
//           they are computed once per CTA into shared tables and each thread only sweeps δ.
//  levels   the 2P interface rows form a tridiagonal system, reduced again by 8-row chunks
//           (2P → P/2 → …) until ≤ 16 rows remain, solved by one thread (Thomas), then
//           back-substituted level by level.
// The row data is staged in shared memory with a padded index (bank-conflict free chunk reads).
#include "common.cuh"
#include "internal.h"

struct Row4 {
  double2 a, b, c, d;
};

// Generic 8-row chunk forward/backward (general complex coefficients).  In: rows r[0..7].
// Out: interface rows f, l; interior coefficients (α', γ', δ') for rows 1..6 stored back into
// r[j].a, r[j].c, r[j].d.
CNP_DEV bool chunk8(Row4* r, Row4& f, Row4& l) {
  double2 al[8], ga[8], de[8];
  bool ok = true;
  {
    const double2 inv = crecip(r[1].b);
    ok &= cfinite(inv);
    al[1] = cmul(r[1].a, inv);
    ga[1] = cmul(r[1].c, inv);
    de[1] = cmul(r[1].d, inv);
  }
#pragma unroll
  for (int j = 2; j < 8; ++j) {
    const double2 piv = cfms(r[j].b, r[j].a, ga[j - 1]);
    const double2 inv = crecip(piv);
    ok &= cfinite(inv);
    const double2 ai = cmul(r[j].a, inv);
    al[j] = make_double2(-(ai.x * al[j - 1].x - ai.y * al[j - 1].y), -(ai.x * al[j - 1].y + ai.y * al[j - 1].x));
    ga[j] = cmul(r[j].c, inv);
    de[j] = cmul(cfms(r[j].d, r[j].a, de[j - 1]), inv);
  }
  l.a = al[7]; l.b = make_double2(1.0, 0.0); l.c = ga[7]; l.d = de[7];
  double2 ap = make_double2(0.0, 0.0), gp = make_double2(-1.0, 0.0), dp = make_double2(0.0, 0.0);
#pragma unroll
  for (int j = 6; j >= 1; --j) {
    const double2 na = cfms(al[j], ga[j], ap);
    const double2 ng = make_double2(-(ga[j].x * gp.x - ga[j].y * gp.y), -(ga[j].x * gp.y + ga[j].y * gp.x));
    const double2 nd = cfms(de[j], ga[j], dp);
    ap = na; gp = ng; dp = nd;
    r[j].a = ap; r[j].c = gp; r[j].d = dp;
  }
  f.a = r[0].a;
  f.b = cfms(r[0].b, r[0].c, ap);
  f.c = make_double2(-(r[0].c.x * gp.x - r[0].c.y * gp.y), -(r[0].c.x * gp.y + r[0].c.y * gp.x));
  f.d = cfms(r[0].d, r[0].c, dp);
  return ok;
}

// Solve the reduced system stored as Row4 array `lv0` of size n0 (power of two, >= 2) in shared
// memory.  Scratch for deeper levels follows lv0.  Result x_i written into lv0[i].d.
CNP_DEV void solve_reduced(Row4* lv0, int n0, int tid, int* status) {
  // level sizes: n0, n0/4, ... until <= 16
  Row4* lv[8];
  int nn[8];
  int L = 0;
  lv[0] = lv0;
  nn[0] = n0;
  while (nn[L] > 16) {
    lv[L + 1] = lv[L] + nn[L];
    nn[L + 1] = nn[L] / 4;
    ++L;
  }
  // downward: reduce level l into level l+1
  for (int l = 0; l < L; ++l) {
    const int nt = nn[l] / 8;
    if (tid < nt) {
      Row4 r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = lv[l][8 * tid + j];
      Row4 f, g;
      bool ok = chunk8(r, f, g);
      if (!ok) atomicOr(status, 1);
#pragma unroll
      for (int j = 1; j < 7; ++j) lv[l][8 * tid + j] = r[j];
      lv[l + 1][2 * tid] = f;
      lv[l + 1][2 * tid + 1] = g;
    }
    __syncthreads();
  }
  // bottom: Thomas by one thread
  if (tid == 0) {
    Row4* r = lv[L];
    const int n = nn[L];
    double2 cp[16], dp[16];
    double2 inv = crecip(r[0].b);
    bool ok = cfinite(inv);
    cp[0] = cmul(r[0].c, inv);
    dp[0] = cmul(r[0].d, inv);
    for (int i = 1; i < n; ++i) {
      inv = crecip(cfms(r[i].b, r[i].a, cp[i - 1]));
      ok &= cfinite(inv);
      cp[i] = cmul(r[i].c, inv);
      dp[i] = cmul(cfms(r[i].d, r[i].a, dp[i - 1]), inv);
    }
    double2 x = dp[n - 1];
    r[n - 1].d = x;
    for (int i = n - 2; i >= 0; --i) {
      x = cfms(dp[i], cp[i], x);
      r[i].d = x;
    }
    if (!ok) atomicOr(status, 1);
  }
  __syncthreads();
  // upward back-substitution
  for (int l = L - 1; l >= 0; --l) {
    const int nt = nn[l] / 8;
    if (tid < nt) {
      const double2 x0 = lv[l + 1][2 * tid].d;
      const double2 x7 = lv[l + 1][2 * tid + 1].d;
      Row4* r = lv[l] + 8 * tid;
#pragma unroll
      for (int j = 1; j < 7; ++j) r[j].d = cfms(cfms(r[j].d, r[j].a, x0), r[j].c, x7);
      r[0].d = x0;
      r[7].d = x7;
    }
    __syncthreads();
  }
}

// Main kernel.  TOEP: constant rows (lo, di, up taken from index 1).  LMAX: max rows per thread.
template <bool TOEP, int LMAX>
__global__ void __launch_bounds__(256) k_tridiag(const double2* __restrict__ what, double2* __restrict__ zhat,
                                                 const double* __restrict__ lo, const double* __restrict__ di,
                                                 const double* __restrict__ up, const double2* __restrict__ sk,
                                                 const double2* __restrict__ il2, int m, int64_t W, double tau,
                                                 int* __restrict__ status) {
  extern __shared__ double2 smem[];
  double2* D = smem;  // padded data [padi(m)]
  __shared__ double2 tal[LMAX], tga[LMAX], tiv[LMAX];      // Toeplitz forward tables (pos 1..LMAX-1)
  __shared__ double2 tba[2][LMAX], tbg[2][LMAX];           // Toeplitz backward tables (two lengths)
  const int k = blockIdx.x;
  const int tid = threadIdx.x, P = blockDim.x;
  const double2 s = sk[k];
  const double2 il = il2[k];
  const double2* src = what + (int64_t)k * W;
  // ---- coalesced load of row k, scaled by 1/λ2_k
  for (int i = tid; i < m; i += P) D[padi(i)] = cmul(ldg_cs2(src + i), il);
  const int i0 = (int)(((int64_t)tid * m) / P);
  const int i1 = (int)(((int64_t)(tid + 1) * m) / P);
  const int len = i1 - i0;
  const int lmin = m / P;
  if (TOEP) {
    if (tid == 0) {
      const double a = -tau * lo[1], c = -tau * up[1];
      const double2 b = make_double2(s.x - tau * di[1], s.y);
      double2 g = make_double2(0.0, 0.0), al = make_double2(0.0, 0.0);
      for (int j = 1; j < LMAX; ++j) {
        const double2 piv = (j == 1) ? b : crfms(b, a, g);
        const double2 inv = crecip(piv);
        if (!cfinite(inv)) atomicOr(status, 1);
        al = (j == 1) ? cscale(inv, a) : cscale(cmul(al, inv), -a);
        g = cscale(inv, c);
        tal[j] = al; tga[j] = g; tiv[j] = inv;
      }
      for (int which = 0; which < 2; ++which) {
        const int L = lmin + which;
        double2 ap = make_double2(0.0, 0.0), gp = make_double2(-1.0, 0.0);
        if (L - 1 < LMAX) { tba[which][L - 1] = ap; tbg[which][L - 1] = gp; }
        for (int j = L - 2; j >= 1; --j) {
          const double2 na = cfms(tal[j], tga[j], ap);
          const double2 ng = make_double2(-(tga[j].x * gp.x - tga[j].y * gp.y), -(tga[j].x * gp.y + tga[j].y * gp.x));
          ap = na; gp = ng;
          tba[which][j] = ap; tbg[which][j] = gp;
        }
      }
    }
  }
  __syncthreads();
  // ---- level 1: per-thread modified Thomas on rows [i0, i1)
  double2 dl[LMAX];
  double2 alr[TOEP ? 1 : LMAX], gar[TOEP ? 1 : LMAX];
#pragma unroll
  for (int j = 0; j < LMAX; ++j) dl[j] = (j < len) ? D[padi(i0 + j)] : make_double2(0.0, 0.0);
  bool ok = true;
  Row4 f, l;
  if (TOEP) {
    const double a = -tau * lo[1], c = -tau * up[1];
    const double2 b = make_double2(s.x - tau * di[1], s.y);
    // forward δ (positions 1..len-1)
    double2 dprev = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j < LMAX; ++j) {
      if (j < len) {
        const double2 num = (j == 1) ? dl[1] : crfms(dl[j], a, dprev);
        dprev = cmul(num, tiv[j]);
        dl[j] = dprev;
      }
    }
    const int which = len - lmin;
    l.a = tal[len - 1]; l.b = make_double2(1.0, 0.0); l.c = tga[len - 1]; l.d = dl[len - 1];
    if (i1 == m) l.c = make_double2(0.0, 0.0);
    // backward δ' (positions len-2..1)
    double2 dp = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = LMAX - 2; j >= 1; --j) {
      if (j <= len - 2) {
        dp = cfms(dl[j], tga[j], dp);
        dl[j] = dp;
      }
    }
    const double2 ap1 = (len >= 3) ? tba[which][1] : make_double2(0.0, 0.0);
    const double2 gp1 = (len >= 3) ? tbg[which][1] : make_double2(-1.0, 0.0);
    const double2 dp1 = (len >= 3) ? dl[1] : make_double2(0.0, 0.0);
    f.a = make_double2(i0 == 0 ? 0.0 : a, 0.0);
    f.b = cfms(b, make_double2(c, 0.0), ap1);
    f.c = cscale(gp1, -c);
    f.d = crfms(dl[0], c, dp1);
  } else {
    // general rows: coefficients per row
    double2 dprev = make_double2(0.0, 0.0), gprev = make_double2(0.0, 0.0), aprev = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j < LMAX; ++j) {
      if (j < len) {
        const int i = i0 + j;
        const double a = -tau * lo[i], c = -tau * up[i];
        const double2 b = make_double2(s.x - tau * di[i], s.y);
        const double2 piv = (j == 1) ? b : crfms(b, a, gprev);
        const double2 inv = crecip(piv);
        ok &= cfinite(inv);
        aprev = (j == 1) ? cscale(inv, a) : cscale(cmul(aprev, inv), -a);
        gprev = cscale(inv, c);
        dprev = (j == 1) ? cmul(dl[1], inv) : cmul(crfms(dl[j], a, dprev), inv);
        alr[j] = aprev; gar[j] = gprev; dl[j] = dprev;
      }
    }
    l.a = aprev; l.b = make_double2(1.0, 0.0); l.c = gprev; l.d = dprev;
    double2 ap = make_double2(0.0, 0.0), gp = make_double2(-1.0, 0.0), dp = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = LMAX - 2; j >= 1; --j) {
      if (j <= len - 2) {
        const double2 na = cfms(alr[j], gar[j], ap);
        const double2 ng = make_double2(-(gar[j].x * gp.x - gar[j].y * gp.y), -(gar[j].x * gp.y + gar[j].y * gp.x));
        dp = cfms(dl[j], gar[j], dp);
        ap = na; gp = ng;
        alr[j] = ap; gar[j] = gp; dl[j] = dp;
      }
    }
    const double a0 = -tau * lo[i0], c0 = -tau * up[i0];
    const double2 b0 = make_double2(s.x - tau * di[i0], s.y);
    const double2 ap1 = (len >= 3) ? alr[1] : make_double2(0.0, 0.0);
    const double2 gp1 = (len >= 3) ? gar[1] : make_double2(-1.0, 0.0);
    const double2 dp1 = (len >= 3) ? dl[1] : make_double2(0.0, 0.0);
    f.a = make_double2(a0, 0.0);
    f.b = cfms(b0, make_double2(c0, 0.0), ap1);
    f.c = cscale(gp1, -c0);
    f.d = crfms(dl[0], c0, dp1);
    if (!ok) atomicOr(status, 1);
  }
  __syncthreads();  // D is now free: reuse it for the reduced system
  Row4* R = reinterpret_cast<Row4*>(smem);
  R[2 * tid] = f;
  R[2 * tid + 1] = l;
  __syncthreads();
  solve_reduced(R, 2 * P, tid, status);
  const double2 x0 = R[2 * tid].d, xl = R[2 * tid + 1].d;
  __syncthreads();
  // ---- back-substitute interior rows, stage into D, coalesced store
  D[padi(i0)] = x0;
  D[padi(i1 - 1)] = xl;
  if (TOEP) {
    const int which = len - lmin;
#pragma unroll
    for (int j = 1; j < LMAX - 1; ++j)
      if (j <= len - 2) D[padi(i0 + j)] = cfms(cfms(dl[j], tba[which][j], x0), tbg[which][j], xl);
  } else {
#pragma unroll
    for (int j = 1; j < LMAX - 1; ++j)
      if (j <= len - 2) D[padi(i0 + j)] = cfms(cfms(dl[j], alr[j], x0), gar[j], xl);
  }
  __syncthreads();
  double2* dst = zhat + (int64_t)k * W;
  for (int i = tid; i < m; i += P) stg_cs2(dst + i, D[padi(i)]);
}

// Small-m path (m < 64): one thread per frequency, plain Thomas on the scaled system.
__global__ void k_tridiag_small(const double2* __restrict__ what, double2* __restrict__ zhat,
                                const double* __restrict__ lo, const double* __restrict__ di,
                                const double* __restrict__ up, const double2* __restrict__ sk,
                                const double2* __restrict__ il2, int m, int64_t W, double tau, int K,
                                int* __restrict__ status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double2 s = sk[k], il = il2[k];
  double2 cp[64], dp[64];
  const double2* src = what + (int64_t)k * W;
  bool ok = true;
  for (int i = 0; i < m; ++i) {
    const double a = -tau * lo[i], c = -tau * up[i];
    const double2 b = make_double2(s.x - tau * di[i], s.y);
    const double2 d = cmul(src[i], il);
    const double2 piv = (i == 0) ? b : crfms(b, a, cp[i - 1]);
    const double2 inv = crecip(piv);
    ok &= cfinite(inv);
    cp[i] = cscale(inv, c);
    dp[i] = (i == 0) ? cmul(d, inv) : cmul(crfms(d, a, dp[i - 1]), inv);
  }
  double2* dst = zhat + (int64_t)k * W;
  double2 x = dp[m - 1];
  dst[m - 1] = x;
  for (int i = m - 2; i >= 0; --i) {
    x = cfms(dp[i], cp[i], x);
    dst[i] = x;
  }
  if (!ok) atomicOr(status, 1);
}

static int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

cudaError_t launch_shifted_solve(cnpint_ctx* c, const double2* what, double2* zhat) {
  const int m = c->nx;
  const int K = c->H + 1;
  const int64_t W = c->ld;
  cnp_prof_begin(c, KID_TRIDIAG);
  const double bytes = 32.0 * cnp_spec_units(c);
  if (m < 64) {
    k_tridiag_small<<<(K + 127) / 128, 128, 0, c->stream>>>(what, zhat, c->d_lo, c->d_di, c->d_up, c->d_sk, c->d_il2,
                                                            m, W, c->tau, K, c->d_status);
    cnp_prof_end(c, KID_TRIDIAG, bytes);
    return cudaGetLastError();
  }
  const int LM = c->toeplitz ? 16 : 8;
  int P = pow2_at_least((m + LM - 1) / LM);
  if (P < 32) P = 32;
  while (P > 32 && m / P < 2) P >>= 1;
  if (P > 256) return cudaErrorInvalidValue;
  // shared memory: padded data, or the reduced system (2P rows + deeper levels), whichever is larger
  size_t data = (size_t)(padi_host(m) + 1) * sizeof(double2);
  size_t red = (size_t)(2 * P + P) * sizeof(Row4);
  size_t smem = data > red ? data : red;
  cudaError_t e;
  if (c->toeplitz) {
    static bool attr = false;
    if (!attr) {
      e = cudaFuncSetAttribute(k_tridiag<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    k_tridiag<true, 16><<<K, P, smem, c->stream>>>(what, zhat, c->d_lo, c->d_di, c->d_up, c->d_sk, c->d_il2, m, W,
                                                    c->tau, c->d_status);
  } else {
    static bool attr = false;
    if (!attr) {
      e = cudaFuncSetAttribute(k_tridiag<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    k_tridiag<false, 8><<<K, P, smem, c->stream>>>(what, zhat, c->d_lo, c->d_di, c->d_up, c->d_sk, c->d_il2, m, W,
                                                    c->tau, c->d_status);
  }
  cnp_prof_end(c, KID_TRIDIAG, bytes);
  return cudaGetLastError();
}
