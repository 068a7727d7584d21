// K5: the spatial fast diagonalisation of the 2D operator ("if 𝓛 = κΔ, the fast
// discrete sine transform (DST) is used in step-(b)"), generalised to the Black–Scholes Kronecker
// sum L_h = I⊗L_x + L_y⊗I + shift·I with Toeplitz tridiagonal L_x, L_y.
//
// L_x = tridiag(s, d, u), s·u > 0, is similar to the symmetric Toeplitz tridiag(√(su), d, √(su))
// through D = diag(ρ^j), ρ = √(s/u); that matrix is diagonalised by the DST-I, so
//   L_x = (D S) diag(e) (S D⁻¹),  S_{jk} = √(2/(n+1)) sin(πjk/(n+1)),  e_k = d + 2√(su) cos(πk/(n+1)).
// W⁻¹ = (S D_y⁻¹) ⊗ (S D_x⁻¹) commutes with the time transform, so P_α⁻¹ in 2D is
//   (I ⊗ W) · [per spatial mode: Γ_α, FFT_t, ÷(λ1_k − λ2_k τ μ), iFFT_t, Γ_α⁻¹] · (I ⊗ W⁻¹)
// (the bracket is K6 in k_timefft.cu).  This file applies one axis of W⁻¹ or W to every line:
//   forward:  ŷ_k = Σ_j sin(πjk/(n+1)) · ρ^{−j} y_j          (unnormalised sine sum)
//   inverse:  y_j = ρ^{j} · 2/(n+1) · Σ_k sin(πjk/(n+1)) ŷ_k
// A DST-I of length n = M−1 (M = n+1 a power of two) is computed as the odd extension of length
// 2M, i.e. a complex FFT of length M of packed pairs plus the real split: FFT_{2M}(e)_k = −2i ŷ_k.
#include "common.cuh"
#include "internal.h"
#include "fft_device.cuh"

// YPASS = false: lines are rows (t, y), elements x contiguous.  YPASS = true: lines are columns
// (t, x), elements y with stride ld.  X lines per CTA.
template <bool YPASS>
__global__ void __launch_bounds__(512) k_dst(const double* __restrict__ in, double* __restrict__ out, int n, int logM,
                                             int64_t ld, int ny, int64_t nlines, int X, int CS,
                                             const double* __restrict__ pre, const double* __restrict__ post,
                                             const double2* __restrict__ tw, int accumulate) {
  double2* const sbuf = fft_smem;
  double* sd = reinterpret_cast<double*>(sbuf);
  const int tid = threadIdx.x, T = blockDim.x;
  const int M = 1 << logM;  // n + 1
  const int64_t slice = (int64_t)ny * ld;
  // line -> base offset, element stride
  auto base_of = [&](int64_t line) -> int64_t {
    if (!YPASS) return line * ld;                 // line = t*ny + y
    const int64_t xt = ld;                        // lines per t for the y pass: ld columns
    const int64_t t = line / xt, x = line - t * xt;
    return t * slice + x;
  };
  const int64_t estride = YPASS ? ld : 1;
  const int64_t line0 = (int64_t)blockIdx.x * X;
  // ---- load + pre-scale + odd extension into packed complex columns: e_0 = e_M = 0,
  //      e_j = p_j y_j (1 <= j <= n), e_{2M−j} = −e_j
  {
    const int total = X * M;  // also zero-fills e_0 / e_M slots
    for (int q = tid; q < total; q += T) {
      int c, j;
      if (YPASS) { j = q / X; c = q - j * X; } else { c = q / M; j = q - c * M; }   // coalesced order
      const int64_t line = line0 + c;
      double v = 0.0;
      if (j < n && line < nlines) {
        v = in[base_of(line) + (int64_t)j * estride];
        if (pre) v *= pre[j];
      }
      double* col = sd + 2 * (c * CS);
      if (j < n) {
        const int e = j + 1;           // extended index
        const int e2 = 2 * M - e;
        col[2 * padi(e >> 1) + (e & 1)] = v;
        col[2 * padi(e2 >> 1) + (e2 & 1)] = -v;
      } else {
        // j == n: zero the e_0 and e_M slots
        col[2 * padi(0) + 0] = 0.0;
        col[2 * padi(M >> 1) + (M & 1)] = 0.0;
      }
    }
  }
  __syncthreads();
  fft_columns<false>(CS, X, logM, tw, tid, T);
  // ---- split: E_k = split_fwd(Z_k, Z_{M−k}, ω_{2M}^k), ŷ_k = −Im(E_k)/2, k = 1..n
  {
    const int total = X * M;
    for (int q = tid; q < total; q += T) {
      int c, j;
      if (YPASS) { j = q / X; c = q - j * X; } else { c = q / M; j = q - c * M; }
      const int64_t line = line0 + c;
      if (line >= nlines) continue;
      const int64_t addr = base_of(line) + (int64_t)j * estride;
      if (j >= n) {
        // x-pass: zero the padding columns [n, ld) of the output row
        if (!YPASS)
          for (int64_t jj = n; jj < ld; ++jj) out[base_of(line) + jj] = accumulate ? out[base_of(line) + jj] : 0.0;
        continue;
      }
      const int k = j + 1;
      const double2* cb = sbuf + c * CS;
      const double2 zk = cb[padi(k & (M - 1))];
      const double2 zm = cb[padi((M - k) & (M - 1))];
      const double2 E = split_fwd(zk, zm, tw[k]);
      double y = -0.5 * E.y;
      if (post) y *= post[j];
      if (accumulate) y += out[addr];
      out[addr] = y;
    }
  }
}

static int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

template <bool YPASS>
static cudaError_t run_dst(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                           int accumulate) {
  const int n = YPASS ? c->ny : c->nx;
  const int M = n + 1;
  const int logM = ilog2(M);
  const int X = 16;
  const int CS = padi_host(M + 1) + 1;
  const int64_t nlines = YPASS ? (int64_t)c->N * c->ld : (int64_t)c->N * c->ny;
  const int per = M >= 16 ? M / 16 : 1;
  int T = X * per;
  if (T < 64) T = 64;
  if (T > 512) T = 512;
  const size_t smem = (size_t)X * CS * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_dst<YPASS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const unsigned grid = (unsigned)((nlines + X - 1) / X);
  const int kid = YPASS ? KID_DST_Y : KID_DST_X;
  cnp_prof_begin(c, kid);
  k_dst<YPASS><<<grid, T, smem, c->stream>>>(in, out, n, logM, c->ld, c->ny, nlines, X, CS, pre, post,
                                            YPASS ? c->d_twy : c->d_twx, accumulate);
  cnp_prof_end(c, kid, (accumulate ? 24.0 : 16.0) * cnp_units(c));
  return cudaGetLastError();
}

cudaError_t launch_dst_x(cnpint_ctx* c, const double* in, double* out, const double* vscale, int inverse) {
  (void)vscale;
  return inverse ? run_dst<false>(c, in, out, nullptr, c->d_dx, 0) : run_dst<false>(c, in, out, c->d_dxi, nullptr, 0);
}
cudaError_t launch_dst_x_acc(cnpint_ctx* c, const double* in, double* out) {
  return run_dst<false>(c, in, out, nullptr, c->d_dx, 1);
}
cudaError_t launch_dst_y(cnpint_ctx* c, const double* in, double* out, int inverse) {
  return inverse ? run_dst<true>(c, in, out, nullptr, c->d_dy, 0) : run_dst<true>(c, in, out, c->d_dyi, nullptr, 0);
}
