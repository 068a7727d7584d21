// K6, lean 2D time pass (round 2): per spatial-mode column pair (PAPER.md:315-316 with Eq. 3.2
// steps (a)-(c); the operation of k_tfft.cu MODE 2 and k_tpass.cu):
//   z_t = 1/(N γ_t) · iFFT_k[ FFT_t(γ s v)_k / (λ1_k − λ2_k μ) ],  μ = τ(e_x + e_y) + τ·shift,
// two real columns packed as one complex column and separated by Hermitian symmetry.
// Built like the lean sine passes (k_dst4.cu / k_dst5.cu): P = 8 column pairs per tile with the threads
// interleaved pair-fastest (every row access is one 128-B segment), TP = 64 threads per pair owning it
// for the whole transform, register radix passes N = R1·R2·R3 (1024 = 8·8·16, 512 = 8·8·8,
// 256 = 8·8·4) with the items a thread owns enumerated so that the forward transform's last step leaves
// exactly the inverse plan's (R3, R2, R1) first-step inputs in the thread — the only exchanges are the
// four radix exchanges and the Hermitian partner k ↔ N − k, in per-pair regions at an odd stride.
#include "common.cuh"
#include "internal.h"

#include "fft_device.cuh"

template <int LOGN>
struct T2Plan {
  static constexpr int N = 1 << LOGN, H = N / 2;
  static constexpr int R1 = 8, R2 = 8, R3 = N / 64;   // forward plan; inverse (R3, R2, R1)
  static constexpr int TP = N >= 512 ? 64 : N / 8;   // threads per column pair
  static constexpr int P = 8;                        // column pairs per tile (128-B row segments)
  static constexpr int NT = P * TP;
  static constexpr int MINB = LOGN >= 10 ? 1 : 2;
  static constexpr int RS = N + 1;                   // region stride (complex), odd
  static constexpr int F1 = (N / R1) / TP, F2 = (N / R2) / TP, F3 = (N / R3) / TP;  // forward items
  static constexpr int B1 = (N / R3) / TP, B2 = (N / R2) / TP, B3 = (N / R1) / TP;  // inverse items
  static constexpr size_t off_tw = (size_t)P * RS * 16;
  static constexpr size_t off_lam = off_tw + (size_t)N * 16;
  static constexpr size_t off_g = off_lam + (size_t)2 * (H + 1) * 16;
  static constexpr size_t bytes = off_g + (size_t)2 * N * 8;
  // GEN 2: per-mode tables f_k = ½/λ2_k (complex) and (c_k = λ1_k/λ2_k, c_k.y², κ_k) instead of λ1, λ2
  static constexpr size_t off_f2 = off_g + (size_t)2 * N * 8;
  static constexpr size_t bytes2 = off_f2 + (size_t)(H + 1) * 16;
  static_assert(F3 == B1, "forward output items = inverse input items");
  static_assert(F1 >= 1 && F2 >= 1 && F3 >= 1 && B2 >= 1 && B3 >= 1, "every step has whole items per thread");
};

template <int LOGN, int GEN>
__global__ void __launch_bounds__(T2Plan<LOGN>::NT, T2Plan<LOGN>::MINB)
    k_tpass2(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ vscale, int64_t W,
             int ld, int nx, const double* __restrict__ gam, const double* __restrict__ igam,
             const double2* __restrict__ lam1, const double2* __restrict__ lam2, const double2* __restrict__ sk,
             const double2* __restrict__ il2, const double* __restrict__ ex, const double* __restrict__ ey,
             double tau, double tau_shift, const double2* __restrict__ twN, int debug_sign, int l2pf) {
  using PL = T2Plan<LOGN>;
  constexpr int N = PL::N, H = PL::H, TP = PL::TP, P = PL::P, NT = PL::NT, RS = PL::RS;
  constexpr int R1 = PL::R1, R2 = PL::R2, R3 = PL::R3;
  char* const smem = reinterpret_cast<char*>(fft_smem);
  double2* const tw = reinterpret_cast<double2*>(smem + PL::off_tw);   // ω_N^q
  double2* const l1s = reinterpret_cast<double2*>(smem + PL::off_lam);  // GEN 1: λ1_k; GEN 2: (c_k.x, c_k.y)
  double2* const l2s = l1s + (H + 1);                                   // GEN 1: λ2_k; GEN 2: (c_k.y², κ_k)
  double* const gs = reinterpret_cast<double*>(smem + PL::off_g);      // γ_t
  double* const igs = gs + N;                                          // 1/(N γ_t)
  double2* const fs = reinterpret_cast<double2*>(smem + PL::off_f2);    // GEN 2: f_k = ½/λ2_k (½/λ1_k if λ2_k = 0)
  const int tid = threadIdx.x, pr = tid % P, r = tid / P;
  double2* const A = reinterpret_cast<double2*>(smem) + pr * RS;
  const double sg = debug_sign ? -1.0 : 1.0;
  for (int q = tid; q < N; q += NT) {
    double2 w = twN[q];
    w.y *= sg;
    tw[q] = w;
    gs[q] = gam[q];
    igs[q] = igam[q];
  }
  for (int q = tid; q <= H; q += NT) {
    if constexpr (GEN == 1) {
      l1s[q] = lam1[q];
      l2s[q] = lam2[q];
    } else {
      // 1/(λ1 − λ2 μ) = (1/λ2)·1/(c − μ), c = λ1/λ2 (host long double); α = 1, k = N/2 has λ2 = 0:
      // there 1/λ1 with c = 1, κ = 0 (no μ term)
      const double2 i2 = il2[q];
      const bool z = i2.x == 0.0 && i2.y == 0.0;
      const double2 cq = z ? make_double2(1.0, 0.0) : sk[q];
      const double2 fq = z ? crecip(lam1[q]) : i2;
      l1s[q] = cq;
      l2s[q] = make_double2(cq.y * cq.y, z ? 0.0 : 1.0);
      fs[q] = cscale(fq, 0.5);
    }
  }
  pdl_enter();  // PDL: tables above are create-time constants; the basis scale and the input come from earlier kernels
  const double s = vscale ? *vscale : 1.0;
  __syncthreads();
  const int npairs = (int)(W / 2);
  const int ntiles = (npairs + P - 1) / P;
  auto twf = [&](int e) { return tw[e & (N - 1)]; };                // ω_N^e
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int p = tile * P + pr;
    const bool ok = p < npairs;
    const int col = 2 * p;
    const int xin = col % ld, yy = col / ld;
    const bool padA = !ok || xin >= nx, padB = !ok || xin + 1 >= nx;
    // ---- forward step 1: item m (rows t = m + (N/R1) n1), Γ_α·s on load, DFT_R1, ω_N^{m k1}
#pragma unroll
    for (int i = 0; i < PL::F1; ++i) {
      const int m = r + i * TP;
      double2 v[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int t = m + (N / R1) * n1;
        const double2 x = ok ? ldg_cs2(reinterpret_cast<const double2*>(in + (int64_t)t * W + col)) : make_double2(0.0, 0.0);
        v[n1] = cscale(x, gs[t] * s);
      }
      dftR<R1, false>(v);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) A[k1 * (N / R1) + m] = k1 ? cmul(v[k1], twf(m * k1)) : v[0];
    }
    // the CTA's next tile (N rows × P pairs = 128 B per row) into L2 while this one computes: its step-1
    // loads then hit L2 (ncu: 25 % of the stall samples were those loads waiting on HBM)
    if (l2pf && tile + (int)gridDim.x < ntiles) {
      const int64_t c2 = 2 * (int64_t)(tile + gridDim.x) * P;
      const unsigned nb = (unsigned)(2 * (npairs - (tile + (int)gridDim.x) * P < P ? npairs - (tile + (int)gridDim.x) * P : P) * 8);
      for (int t = tid; t < N; t += NT) prefetch_l2(in + (int64_t)t * W + c2, nb);
    }
    __syncthreads();
    // ---- forward step 2: item (k1, m3): B[k1][m3 + R3 m2] → DFT_R2 → ω_N^{R1 m3 k2}
    double2 u[PL::F2][R2];
#pragma unroll
    for (int i = 0; i < PL::F2; ++i) {
      const int q = r + i * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
      for (int m2 = 0; m2 < R2; ++m2) u[i][m2] = A[k1 * (N / R1) + m3 + R3 * m2];
      dftR<R2, false>(u[i]);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PL::F2; ++i) {
      const int q = r + i * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) A[(k2 * R1 + k1) * R3 + m3] = k2 ? cmul(u[i][k2], twf(R1 * m3 * k2)) : u[i][k2];
    }
    __syncthreads();
    // ---- forward step 3: item (k1, k2) → Z_k, k = k1 + R1 k2 + R1 R2 k3 (k3 in the thread)
    double2 z[PL::F3][R3];
#pragma unroll
    for (int i = 0; i < PL::F3; ++i) {
      const int q = r + i * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
      for (int m3 = 0; m3 < R3; ++m3) z[i][m3] = A[(k2 * R1 + k1) * R3 + m3];
      dftR<R3, false>(z[i]);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PL::F3; ++i) {
      const int q = r + i * TP;
#pragma unroll
      for (int k3 = 0; k3 < R3; ++k3) {
        if constexpr (GEN >= 2) {
          const int k = q + R1 * R2 * k3;
          const double2 f = k <= H ? fs[k] : cconj(fs[N - k]);
          z[i][k3] = cmul(z[i][k3], f);
        }
        A[q + R1 * R2 * k3] = z[i][k3];
      }
    }
    __syncthreads();
    // ---- Hermitian separation, the per-mode division, re-packing (frequencies k of this thread)
    // padding columns (input and output exactly 0) take μ = 1: with α = 1 the k = 0 mode has λ1 = 0,
    // and μ = 0 there would put 0·∞ = NaN into the partner column of the packed pair
    double mua = 1.0, mub = 1.0;
    if (!padA) mua = tau * (ex[xin] + ey[yy]) + tau_shift;
    if (!padB) mub = tau * (ex[xin + 1] + ey[yy]) + tau_shift;
#pragma unroll
    for (int i = 0; i < PL::F3; ++i) {
      const int q = r + i * TP;
#pragma unroll
      for (int k3 = 0; k3 < R3; ++k3) {
        const int k = q + R1 * R2 * k3;
        const double2 zk = z[i][k3], zm = A[(N - k) & (N - 1)];
        double2 xa, xb;
        if constexpr (GEN == 1) {
          xa = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
          xb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
          const double2 l1 = k <= H ? l1s[k] : cconj(l1s[N - k]);
          const double2 l2 = k <= H ? l2s[k] : cconj(l2s[N - k]);
          // the divide by a Newton-refined reciprocal (no IEEE-division slow path; within an ulp):
          // N = 256 416 → 397 µs at c5 n511, N = 1024 neutral (profiles/r02_div_ab.txt)
          xa = cmul(xa, crecip_nr(csub(l1, cscale(l2, mua))));
          xb = cmul(xb, crecip_nr(csub(l1, cscale(l2, mub))));
        } else {
          // zk, zm already carry ½/λ2 (f_{N−k} = conj f_k), so xa = X_a/λ2; then ÷ (c − κμ):
          // × conj(c − κμ) / |c − κμ|² (12 fp64 per column instead of 17)
          xa = make_double2(zk.x + zm.x, zk.y - zm.y);
          xb = make_double2(zk.y + zm.y, zm.x - zk.x);
          const int kk = k <= H ? k : N - k;
          const double2 cc = l1s[kk], cq = l2s[kk];
          const double cy = k <= H ? cc.y : -cc.y;
          const double ra = fma(-cq.y, mua, cc.x), rb = fma(-cq.y, mub, cc.x);
          const double na = rcp_nr(fma(ra, ra, cq.x)), nb = rcp_nr(fma(rb, rb, cq.x));
          xa = make_double2(fma(xa.x, ra, xa.y * cy) * na, fma(xa.y, ra, -xa.x * cy) * na);
          xb = make_double2(fma(xb.x, rb, xb.y * cy) * nb, fma(xb.y, rb, -xb.x * cy) * nb);
        }
        z[i][k3] = (k == 0 || k == H) ? make_double2(xa.x, xb.x) : make_double2(xa.x - xb.y, xa.y + xb.x);
      }
    }
    __syncthreads();  // partner reads done: the region takes the inverse exchanges
    // ---- inverse, plan (R3, R2, R1): step 1 item m' = q (its inputs k = m' + (N/R3) n1 are z[i][·])
#pragma unroll
    for (int i = 0; i < PL::B1; ++i) {
      const int m = r + i * TP;
      dftR<R3, true>(z[i]);
#pragma unroll
      for (int k1 = 0; k1 < R3; ++k1) {
        const double2 w = twf(m * k1);
        A[k1 * (N / R3) + m] = k1 ? cmul_conj(z[i][k1], w) : z[i][0];
      }
    }
    __syncthreads();
    double2 u2[PL::B2][R2];
#pragma unroll
    for (int i = 0; i < PL::B2; ++i) {
      const int q = r + i * TP, m3 = q % R1, k1 = q / R1;
#pragma unroll
      for (int m2 = 0; m2 < R2; ++m2) u2[i][m2] = A[k1 * (N / R3) + m3 + R1 * m2];
      dftR<R2, true>(u2[i]);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PL::B2; ++i) {
      const int q = r + i * TP, m3 = q % R1, k1 = q / R1;
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) {
        const double2 w = twf(R3 * m3 * k2);
        A[(k2 * R3 + k1) * R1 + m3] = k2 ? cmul_conj(u2[i][k2], w) : u2[i][0];
      }
    }
    __syncthreads();
    // ---- inverse step 3: item (k1, k2) → y_t, t = k1 + R3 k2 + R3 R2 k3; 1/(N γ_t), 16-B stores
#pragma unroll
    for (int i = 0; i < PL::B3; ++i) {
      const int q = r + i * TP, k1 = q % R3, k2 = q / R3;
      double2 y[R1];
#pragma unroll
      for (int m3 = 0; m3 < R1; ++m3) y[m3] = A[(k2 * R3 + k1) * R1 + m3];
      dftR<R1, true>(y);
      if (ok) {
#pragma unroll
        for (int k3 = 0; k3 < R1; ++k3) {
          const int t = q + R3 * R2 * k3;
          const double g = igs[t];
          const double2 val = make_double2(padA ? 0.0 : y[k3].x * g, padB ? 0.0 : y[k3].y * g);
          stg_cs2(reinterpret_cast<double2*>(out + (int64_t)t * W + col), val);
        }
      }
    }
    __syncthreads();  // the region is free for the next tile
  }
}

template <int LOGN, int GEN>
static cudaError_t run_tpass2(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  using PL = T2Plan<LOGN>;
  auto kern = k_tpass2<LOGN, GEN>;
  constexpr size_t bytes = GEN == 1 ? PL::bytes : PL::bytes2;
  int grid_max = 0;
  cudaError_t ce = cnp_dev_cached((const void*)kern, &grid_max, [&](int* v) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PL::NT, bytes);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    *v = per_sm * c->num_sms;
    return cudaSuccess;
  });
  if (ce != cudaSuccess) return ce;
  const int ntiles = (int)((c->slice / 2 + PL::P - 1) / PL::P);
  const int grid = ntiles < grid_max ? ntiles : grid_max;
  return cnp_launch(c, kern, dim3(grid), dim3(PL::NT), bytes, in, out, vscale, c->slice, (int)c->ld, c->nx,
                    (const double*)c->d_gam, (const double*)c->d_igam, (const double2*)c->d_lam1,
                    (const double2*)c->d_lam2, (const double2*)c->d_sk, (const double2*)c->d_il2,
                    (const double*)c->d_ex, (const double*)c->d_ey, c->tau_p, c->tau_p * c->shift,
                    (const double2*)c->d_tw, c->debug & 1, c->l2pf);
}

// 2D time pass through the lean kernel for N ∈ {256, 512, 1024}; else NotSupported.  Debug 262144 keeps the
// first generation (divide by λ1 − λ2μ) instead of GEN 2 (divide through the per-mode tables f_k, c_k:
// c5 n511 N1024 1994 → 1925 µs, N256 388 → 381 µs; profiles/r02_tpass2_gen2_ab.txt).
cudaError_t launch_tpass2(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  if (c->dim != 2) return cudaErrorNotSupported;
  const bool g1 = (c->debug & 262144) != 0;
  switch (c->N) {
    case 256: return g1 ? run_tpass2<8, 1>(c, in, out, vscale) : run_tpass2<8, 2>(c, in, out, vscale);
    case 512: return g1 ? run_tpass2<9, 1>(c, in, out, vscale) : run_tpass2<9, 2>(c, in, out, vscale);
    case 1024: return g1 ? run_tpass2<10, 1>(c, in, out, vscale) : run_tpass2<10, 2>(c, in, out, vscale);
    default: return cudaErrorNotSupported;
  }
}
