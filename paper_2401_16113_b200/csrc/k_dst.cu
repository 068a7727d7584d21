// K5: the spatial fast diagonalisation of the 2D operator ("if 𝓛 = κΔ, the fast
// discrete sine transform (DST) is used in step-(b)"), generalised to the Black–Scholes Kronecker
// sum L_h = I⊗L_x + L_y⊗I + shift·I with Toeplitz tridiagonal L_x, L_y.
//
// L_x = tridiag(s, d, u), s·u > 0, is similar to the symmetric Toeplitz tridiag(√(su), d, √(su))
// through D = diag(ρ^j), ρ = √(s/u); that matrix is diagonalised by the DST-I, so
//   L_x = (D S) diag(e) (S D⁻¹),  S_{jk} = √(2/(n+1)) sin(πjk/(n+1)),  e_k = d + 2√(su) cos(πk/(n+1)).
// W⁻¹ = (S D_y⁻¹) ⊗ (S D_x⁻¹) commutes with the time transform, so P_α⁻¹ in 2D is
//   (I ⊗ W) · [per spatial mode: Γ_α, FFT_t, ÷(λ1_k − λ2_k τ μ), iFFT_t, Γ_α⁻¹] · (I ⊗ W⁻¹)
// (the bracket is K6 in k_tfft.cu).  This file applies one axis of W⁻¹ or W to every line:
//   forward:  ŷ_k = Σ_j sin(πjk/(n+1)) · ρ^{−j} y_j          (unnormalised sine sum)
//   inverse:  y_j = ρ^{j} · 2/(n+1) · Σ_k sin(πjk/(n+1)) ŷ_k
// B200 design: two real lines a, b are packed as one complex line a + i b and embedded as the odd
// extension of length E = 2(n+1) (n+1 a power of two), whose complex FFT gives both sine sums at
// once: FFT(ext a + i ext b)_k = −2i S(a)_k + 2 S(b)_k.  The extension is synthesised inside the
// first butterfly stage (only the n samples live in shared memory), the FFT is the compile-time
// tile machinery of fft_tile.cuh (Stockham radix 8/4/2, per-stage twiddle tables), lines come in by
// cp.async and the CTAs are persistent (tables built once).
//   x pass: a line is a row (t, y) of n contiguous samples; pairs are rows (2p, 2p+1).
//   y pass: a line is a column (t, x) with stride ld; pairs are adjacent columns (x, x+1), so a
//           tile of NC pairs reads 16·NC-byte row segments (128 B for NC = 8).
#include "common.cuh"
#include "internal.h"

#include "fft_tile.cuh"

namespace {

template <int LOGE, int NC>
struct DstLayout {
  static constexpr int E = 1 << LOGE;
  static constexpr int M = E / 2;  // n + 1
  static constexpr int CS = tf_cs(LOGE);
  static constexpr int off_stw = NC * CS;
  static constexpr int off_pre = off_stw + tf_stage_tw(LOGE);  // M+1 doubles (as (M+2)/2 slots)
  static constexpr size_t bytes = (size_t)(off_pre + (M + 2) / 2 + 1) * 16;
};

}  // namespace

template <bool YPASS, int LOGE, int NC>
__global__ void __launch_bounds__(256, 2)
    k_dst(const double* __restrict__ in, double* __restrict__ out, int N, int ny, int64_t ld,
          const double* __restrict__ pre, const double* __restrict__ post, int accumulate, int debug_sign,
          int nx) {
  using LY = DstLayout<LOGE, NC>;
  constexpr int NT = 256;
  constexpr int M = LY::M;
  constexpr int n = M - 1;
  constexpr int CS = LY::CS;
  const int tid = threadIdx.x;
  double2* const buf = tf_smem;
  double2* const stw = tf_smem + LY::off_stw;
  double* const pre_s = reinterpret_cast<double*>(tf_smem + LY::off_pre);  // pre_s[e], e = 0..M
  const int ldi = (int)ld;
  // ---- tables once per CTA: stage twiddles, pre-scaling of the extension (0 at e = 0, M)
  fill_stage_twiddles(stw, LOGE, debug_sign ? -1.0 : 1.0, tid, NT);
  for (int e = tid; e <= M; e += NT) pre_s[e] = (e == 0 || e == M) ? 0.0 : (pre ? pre[e - 1] : 1.0);
  // tiles: x pass — NC row pairs; y pass — NC adjacent column pairs of one time slice
  const int nlines = N * ny;
  const int pairs_per_t = ldi / 2;
  const int tiles_per_t = (pairs_per_t + NC - 1) / NC;
  const int ntiles = YPASS ? N * tiles_per_t : ((nlines + 1) / 2 + NC - 1) / NC;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // ---- load the n samples of each packed line into slots 1..n (cp.async, no staging)
    if (!YPASS) {
      const int line0 = tile * NC * 2;
      for (int q = tid; q < NC * n; q += NT) {
        const int c = q / n, j = q - c * n;
        const int la = line0 + 2 * c, lb = la + 1;
        double* dst = reinterpret_cast<double*>(buf + c * CS + pd(j + 1));
        if (la < nlines) cp_async8(dst, in + (int64_t)la * ld + j);
        else dst[0] = 0.0;
        if (lb < nlines) cp_async8(dst + 1, in + (int64_t)lb * ld + j);
        else dst[1] = 0.0;
      }
    } else {
      const int t = tile / tiles_per_t, p0 = (tile - t * tiles_per_t) * NC;
      for (int q = tid; q < NC * n; q += NT) {
        const int y = q / NC, c = q - y * NC;
        const int p = p0 + c;
        double2* dst = buf + c * CS + pd(y + 1);
        if (p < pairs_per_t) cp_async16(dst, in + ((int64_t)t * ny + y) * ld + 2 * p);
        else *dst = make_double2(0.0, 0.0);
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (pre) {  // pre-scale the n samples in place (D⁻¹ for the forward transform)
      for (int q = tid; q < NC * n; q += NT) {
        const int c = q / n, e = q - c * n + 1;
        double2* p = buf + c * CS + pd(e);
        *p = cscale(*p, pre_s[e]);
      }
      __syncthreads();
    }
    local_fft<false, TF_ODDEXT, LOGE, NC, NT>(buf, stw, TfScale{nullptr, nullptr, 1, 0, 1.0});
    // ---- F_k = −2i S(a)_k + 2 S(b)_k, k = 1..n: S(a) = −Im F/2, S(b) = Re F/2, then post-scale
    if (!YPASS) {
      const int line0 = tile * NC * 2;
      for (int q = tid; q < NC * ldi; q += NT) {
        const int c = q / ldi, x = q - c * ldi;
        const int la = line0 + 2 * c, lb = la + 1;
        double sa = 0.0, sb = 0.0;
        if (x < n) {
          const double2 F = buf[c * CS + pd(x + 1)];
          const double g = post ? post[x] : 1.0;
          sa = -0.5 * F.y * g;
          sb = 0.5 * F.x * g;
        }
        if (la < nlines) {
          double* o = out + (int64_t)la * ld + x;
          *o = accumulate ? *o + sa : sa;
        }
        if (lb < nlines) {
          double* o = out + (int64_t)lb * ld + x;
          *o = accumulate ? *o + sb : sb;
        }
      }
    } else {
      const int t = tile / tiles_per_t, p0 = (tile - t * tiles_per_t) * NC;
      for (int q = tid; q < NC * n; q += NT) {
        const int y = q / NC, c = q - y * NC;
        const int p = p0 + c;
        if (p >= pairs_per_t) continue;
        const double2 F = buf[c * CS + pd(y + 1)];
        const double g = post ? post[y] : 1.0;
        double2 v = make_double2(-0.5 * F.y * g, 0.5 * F.x * g);
        if (2 * p >= nx) v.x = 0.0;      // padding columns stay exactly zero
        if (2 * p + 1 >= nx) v.y = 0.0;
        double2* o = reinterpret_cast<double2*>(out + ((int64_t)t * ny + y) * ld + 2 * p);
        if (accumulate) {
          const double2 w = *o;
          v.x += w.x;
          v.y += w.y;
        }
        stg_cs2(o, v);
      }
    }
    __syncthreads();  // buffer reads done before the next tile's copies land
  }
}

template <bool YPASS, int LOGE>
static cudaError_t run_dst_t(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                             int accumulate) {
  constexpr int NC = LOGE <= 9 ? 8 : LOGE == 10 ? 4 : 2;
  using LY = DstLayout<LOGE, NC>;
  auto kern = k_dst<YPASS, LOGE, NC>;
  static int grid_max = 0;
  if (!grid_max) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LY::bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, LY::bytes);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    grid_max = per_sm * c->num_sms;
  }
  const int n = YPASS ? c->ny : c->nx;
  (void)n;
  const int nlines = c->N * c->ny;
  const int ld = (int)c->ld;
  const int ntiles = YPASS ? c->N * ((ld / 2 + NC - 1) / NC) : ((nlines + 1) / 2 + NC - 1) / NC;
  const int grid = ntiles < grid_max ? ntiles : grid_max;
  kern<<<grid, 256, LY::bytes, c->stream>>>(in, out, c->N, c->ny, c->ld, pre, post, accumulate, c->debug & 1,
                                           c->nx);
  return cudaGetLastError();
}

template <bool YPASS>
static cudaError_t run_dst(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                           int accumulate) {
  const int n = YPASS ? c->ny : c->nx;
  int logE = 0;
  while ((1 << logE) < 2 * (n + 1)) ++logE;
  const int kid = YPASS ? KID_DST_Y : KID_DST_X;
  cnp_prof_begin(c, kid);
  cudaError_t e;
  switch (logE) {
    case 2: e = run_dst_t<YPASS, 2>(c, in, out, pre, post, accumulate); break;
    case 3: e = run_dst_t<YPASS, 3>(c, in, out, pre, post, accumulate); break;
    case 4: e = run_dst_t<YPASS, 4>(c, in, out, pre, post, accumulate); break;
    case 5: e = run_dst_t<YPASS, 5>(c, in, out, pre, post, accumulate); break;
    case 6: e = run_dst_t<YPASS, 6>(c, in, out, pre, post, accumulate); break;
    case 7: e = run_dst_t<YPASS, 7>(c, in, out, pre, post, accumulate); break;
    case 8: e = run_dst_t<YPASS, 8>(c, in, out, pre, post, accumulate); break;
    case 9: e = run_dst_t<YPASS, 9>(c, in, out, pre, post, accumulate); break;
    case 10: e = run_dst_t<YPASS, 10>(c, in, out, pre, post, accumulate); break;
    case 11: e = run_dst_t<YPASS, 11>(c, in, out, pre, post, accumulate); break;
    default: e = cudaErrorInvalidValue; break;
  }
  cnp_prof_end(c, kid, (accumulate ? 24.0 : 16.0) * cnp_units(c));
  return e;
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
