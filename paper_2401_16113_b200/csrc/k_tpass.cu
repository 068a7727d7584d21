// K6 for 2D with N = 256 / 512 (c4, c5 N = 256): the fused time pass of the 2D P_α⁻¹ as register
// FFTs.  Per spatial-mode column pair (PAPER.md:315-316 with Eq. 3.2 steps (a)-(c)):
//   z_t = 1/(N γ_t) · iFFT_k[ FFT_t(γ s v)_k / (λ1_k − λ2_k μ) ],  μ = τ(e_x + e_y) + τ·shift,
// the same operation as k_tfft.cu MODE 2.  A tile is NC = 8 adjacent column pairs × all N rows
// (128-B row segments; 4 pairs at N = 1024); the N-point transforms are three register radix passes, N = R1·R2·R3, with
// two shared-memory exchanges (Cooley–Tukey, n = m + M n1, M = R2 R3; k = k1 + R1 kk,
// kk = k2 + R2 k3 — the scheme of k_dst_r in k_dst.cu), instead of one shared round trip per
// radix-8 stage.  The forward transform leaves frequency k = r + R1R2·k3 in thread r; the inverse
// runs the plan (R3, R2, R1), whose first step takes exactly that assignment, so the only extra
// exchange is the Hermitian partner k ↔ N − k needed to separate the packed pair.
#include "common.cuh"
#include "internal.h"

#include "fft_tile.cuh"

namespace {

template <int A_, int B_, int C_>
struct P3 {
  static constexpr int R1 = A_, R2 = B_, R3 = C_, E = A_ * B_ * C_, M = B_ * C_;
  static constexpr int T1 = M, T2 = A_ * C_, T3 = A_ * B_;
  static constexpr int SB = M;      // B_{k1}[m] at k1·SB + m
  static constexpr int SC = C_ + 1; // C_{k1,k2}[m3] at (k2·R1 + k1)·SC + m3 (odd)
  static constexpr int AREA = R1 * SB > R1 * R2 * SC ? R1 * SB : R1 * R2 * SC;
};

// step 1: thread m holds x[m + M n1] (n1 < R1)
template <class P, bool INV>
CNP_DEV void p3_step1(double2 (&v)[P::R1], double2* area, const double2* twE, int m) {
  dftR<P::R1, INV>(v);
#pragma unroll
  for (int k1 = 0; k1 < P::R1; ++k1) {
    const double2 w = twE[m * k1];
    area[k1 * P::SB + m] = k1 ? (INV ? cmul_conj(v[k1], w) : cmul(v[k1], w)) : v[0];
  }
}
// step 2 (read part): thread r = m3 + R3 k1
template <class P, bool INV>
CNP_DEV void p3_step2_read(double2 (&u)[P::R2], const double2* area, int r) {
  const int m3 = r % P::R3, k1 = r / P::R3;
#pragma unroll
  for (int m2 = 0; m2 < P::R2; ++m2) u[m2] = area[k1 * P::SB + m3 + P::R3 * m2];
  dftR<P::R2, INV>(u);
}
template <class P, bool INV>
CNP_DEV void p3_step2_write(const double2 (&u)[P::R2], double2* area, const double2* twE, int r) {
  const int m3 = r % P::R3, k1 = r / P::R3;
#pragma unroll
  for (int k2 = 0; k2 < P::R2; ++k2) {
    const double2 w = twE[(m3 * k2) * P::R1];  // ω_M^{m3 k2} = ω_E^{m3 k2 R1}
    area[(k2 * P::R1 + k1) * P::SC + m3] = k2 ? (INV ? cmul_conj(u[k2], w) : cmul(u[k2], w)) : u[0];
  }
}
// step 3: thread r = k1 + R1 k2 → X[r + R1 R2 k3], k3 < R3
template <class P, bool INV>
CNP_DEV void p3_step3(double2 (&w)[P::R3], const double2* area, int r) {
  const int k1 = r % P::R1, k2 = r / P::R1;
#pragma unroll
  for (int m3 = 0; m3 < P::R3; ++m3) w[m3] = area[(k2 * P::R1 + k1) * P::SC + m3];
  dftR<P::R3, INV>(w);
}

#ifndef TP_MINB
#define TP_MINB 2
#endif
template <int LOGN>
struct TpPlan {
  static constexpr int N = 1 << LOGN, H = N / 2;
  using F = P3<8, 8, N / 64>;           // forward
  using I = P3<N / 64, 8, 8>;           // inverse (transposed)
  static constexpr int TP = N >= 1024 ? N / 8 : 64;  // max role count of both plans
  static constexpr int NC = 512 / TP;   // column pairs per tile (8: 128-B row segments; 4 at N = 1024)
  static constexpr int MINB = N >= 1024 ? 1 : TP_MINB;
  static constexpr int NT = NC * TP;
  static constexpr int AREA = (F::AREA > I::AREA ? F::AREA : I::AREA) | 1;
  static constexpr int HI = N / 64;
  static constexpr int off_tw = NC * AREA;
  static constexpr int off_lam = off_tw + N;
  static constexpr int off_g = off_lam + 2 * (H + 1);  // doubles ghi[HI] glo[64] ihi[HI] ilo[64]
  static constexpr size_t bytes = (size_t)(off_g + (2 * (HI + 64)) / 2 + 1) * 16;
  static_assert(F::T1 <= TP && F::T2 <= TP && F::T3 <= TP && I::T1 <= TP && I::T2 <= TP && I::T3 <= TP, "roles");
  static_assert(F::T3 == I::T1 && I::R1 == F::R3, "forward output = inverse input assignment");
};

}  // namespace

template <int LOGN>
__global__ void __launch_bounds__(TpPlan<LOGN>::NT, TpPlan<LOGN>::MINB)
    k_tpass_r(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ vscale, int64_t W,
              int ld, int nx, const double* __restrict__ gam, const double* __restrict__ igam,
              const double2* __restrict__ lam1, const double2* __restrict__ lam2, const double* __restrict__ ex,
              const double* __restrict__ ey, double tau, double tau_shift, int debug_sign) {
  using TP = TpPlan<LOGN>;
  using F = typename TP::F;
  using I = typename TP::I;
  constexpr int N = TP::N, H = TP::H, NC = TP::NC;
  const int tid = threadIdx.x;
  const int pr = tid % NC, r = tid / NC;  // pair slot (fastest: 8 pairs = 128-B row segments), role
  double2* const area = tf_smem + pr * TP::AREA;
  double2* const twE = tf_smem + TP::off_tw;
  double2* const l1s = tf_smem + TP::off_lam;
  double2* const l2s = l1s + (H + 1);
  double* const ghi = reinterpret_cast<double*>(tf_smem + TP::off_g);
  double* const glo = ghi + TP::HI;
  double* const ihi = glo + 64;
  double* const ilo = ihi + TP::HI;
  const double sg = debug_sign ? -1.0 : 1.0;
  for (int q = tid; q < N; q += TP::NT) { double2 w = expi_neg(q, N); w.y *= sg; twE[q] = w; }
  for (int q = tid; q <= H; q += TP::NT) { l1s[q] = lam1[q]; l2s[q] = lam2[q]; }
  for (int q = tid; q < TP::HI; q += TP::NT) { ghi[q] = __ldg(gam + q * 64); ihi[q] = __ldg(igam + q * 64); }
  for (int q = tid; q < 64; q += TP::NT) { glo[q] = __ldg(gam + q); ilo[q] = (double)N * __ldg(igam + q); }
  pdl_enter();  // PDL: tables above are create-time constants; the basis scale and the input come from earlier kernels
  const double s = vscale ? *vscale : 1.0;
  __syncthreads();
  const int Wi = (int)W;
  const int npairs = Wi / 2;
  const int ntiles = (npairs + NC - 1) / NC;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int p = tile * NC + pr;
    const bool ok = p < npairs;
    const int col = 2 * p;
    const int xin = col % ld, yy = col / ld;
    const bool padA = xin >= nx, padB = xin + 1 >= nx;
    // ---- forward step 1: thread m loads rows t = m + M n1 of its pair, Γ_α·s on load
    if (r < F::T1) {
      double2 v[F::R1];
#pragma unroll
      for (int n1 = 0; n1 < F::R1; ++n1) {
        const int t = r + F::M * n1;
        v[n1] = ok ? ldg_cs2(reinterpret_cast<const double2*>(in + (int64_t)t * W + col)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int n1 = 0; n1 < F::R1; ++n1) {
        const int t = r + F::M * n1;
        v[n1] = cscale(v[n1], ghi[t >> 6] * glo[t & 63] * s);
      }
      p3_step1<F, false>(v, area, twE, r);
    }
    __syncthreads();
    double2 u[F::R2];
    if (r < F::T2) p3_step2_read<F, false>(u, area, r);
    __syncthreads();
    if (r < F::T2) p3_step2_write<F, false>(u, area, twE, r);
    __syncthreads();
    double2 x[F::R3];
    if (r < F::T3) p3_step3<F, false>(x, area, r);
    __syncthreads();
    // ---- spectrum X_k (k = r + T3 k3) into the area by frequency, then the partner N − k
    if (r < F::T3) {
#pragma unroll
      for (int k3 = 0; k3 < F::R3; ++k3) area[r + F::T3 * k3] = x[k3];
    }
    __syncthreads();
    double2 z[F::R3];
    if (r < F::T3) {
      double mua = 1.0, mub = 1.0;  // padding columns: μ = 1 (α = 1 has λ1_0 = 0; see k_tpass2.cu)
      if (ok && !padA) {
        mua = tau * (ex[xin] + ey[yy]) + tau_shift;
        if (!padB) mub = tau * (ex[xin + 1] + ey[yy]) + tau_shift;
      }
#pragma unroll
      for (int k3 = 0; k3 < F::R3; ++k3) {
        const int k = r + F::T3 * k3;
        const double2 zk = x[k3], zm = area[(N - k) & (N - 1)];
        double2 xa = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        double2 xb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
        const double2 l1 = k <= H ? l1s[k] : cconj(l1s[N - k]);
        const double2 l2 = k <= H ? l2s[k] : cconj(l2s[N - k]);
        xa = cmul(xa, crecip(csub(l1, cscale(l2, mua))));
        xb = cmul(xb, crecip(csub(l1, cscale(l2, mub))));
        z[k3] = (k == 0 || k == H) ? make_double2(xa.x, xb.x) : make_double2(xa.x - xb.y, xa.y + xb.x);
      }
    }
    __syncthreads();  // partner reads done: the area takes the inverse exchanges
    // ---- inverse: plan (R3, R2, R1); thread r holds input index r + T3·k3 = m + M'·n1
    if (r < I::T1) p3_step1<I, true>(z, area, twE, r);
    __syncthreads();
    double2 u2[I::R2];
    if (r < I::T2) p3_step2_read<I, true>(u2, area, r);
    __syncthreads();
    if (r < I::T2) p3_step2_write<I, true>(u2, area, twE, r);
    __syncthreads();
    if (r < I::T3 && ok) {
      double2 y[I::R3];
      p3_step3<I, true>(y, area, r);
#pragma unroll
      for (int k3 = 0; k3 < I::R3; ++k3) {
        const int t = r + I::T3 * k3;
        const double g = ihi[t >> 6] * ilo[t & 63];
        const double2 val = make_double2(padA ? 0.0 : y[k3].x * g, padB ? 0.0 : y[k3].y * g);
        stg_cs2(reinterpret_cast<double2*>(out + (int64_t)t * W + col), val);
      }
    }
    __syncthreads();  // the area is free for the next tile
  }
}

template <int LOGN>
static cudaError_t run_tpass(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  using TP = TpPlan<LOGN>;
  auto kern = k_tpass_r<LOGN>;
  int grid_max = 0;
  cudaError_t ce = cnp_dev_cached((const void*)kern, &grid_max, [&](int* v) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TP::bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TP::NT, TP::bytes);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    *v = per_sm * c->num_sms;
    return cudaSuccess;
  });
  if (ce != cudaSuccess) return ce;
  const int ntiles = (int)((c->slice / 2 + TP::NC - 1) / TP::NC);
  const int grid = ntiles < grid_max ? ntiles : grid_max;
  cnp_launch(c, kern, dim3(grid), dim3(TP::NT), TP::bytes, in, out, vscale, c->slice, (int)c->ld, c->nx,
             (const double*)c->d_gam, (const double*)c->d_igam, (const double2*)c->d_lam1, (const double2*)c->d_lam2,
             (const double*)c->d_ex, (const double*)c->d_ey, c->tau_p, c->tau_p * c->shift, c->debug & 1);
  return cudaGetLastError();
}

// N = 1024 (plan 8·8·16, four pairs per tile, 128 registers) measured slower than the cluster kernel
// (c5 n255: 815 vs 754 µs) and is not routed
bool tpass_ok(const cnpint_ctx* c) { return c->dim == 2 && (c->N == 256 || c->N == 512) && !(c->debug & 64); }

cudaError_t launch_tpass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  cnp_prof_begin(c, KID_TIMEPASS2D);
  cudaError_t e = c->N == 256 ? run_tpass<8>(c, in, out, vscale) : run_tpass<9>(c, in, out, vscale);
  cnp_prof_end(c, KID_TIMEPASS2D, 16.0 * cnp_units(c));
  return e;
}
